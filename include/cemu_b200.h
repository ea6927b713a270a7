/* cemu_b200.h -- C-ABI of the B200-native collective-emulation path.
 *
 * Drop-in boundary.  The reference (arxiv 2405.02969 "NeuronaBox", C++
 * re-creation `cemu`) interposes on collective calls at
 *   cemu::WorkerSession             proj/include/cemu/collective.hpp:50-131
 *     allreduce_async / allgather_async / wait / close
 * and the paper interposes on NCCL itself.  This header
 * exports the NCCL shapes (nccl.h 2.27.3: ncclAllReduce :392-393,
 * ncclAllGather :425-426, ncclReduceScatter :408-410, ncclBroadcast :379,
 * ncclCommInitRank, ncclCommDestroy, ncclCommCount, ncclCommUserRank,
 * ncclGetErrorString, ncclGroupStart/End) under a `cemu` prefix; the
 * communicator's world is JobConfig.world_size (proj/include/cemu/
 * config.hpp:43-62) and its rank must be one of JobConfig.real_ranks.  The
 * job config comes from $CEMU_CONFIG (cemuCommInitRank) or explicit text
 * (cemuCommInitRankConfig), in the reference's key=value format
 * (proj/src/config.cpp:153-262).
 *
 * All collectives are stream-ordered and asynchronous: nothing blocks the
 * host; completion is observed through the stream (this replaces
 * WorkerSession::wait, collective.cpp:223-228).  Buffers are device memory
 * owned by the caller.  Plain pointers and sizes only.
 */
#ifndef CEMU_B200_H_
#define CEMU_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CEMU_B200_VERSION 10000

struct CUstream_st;
typedef struct CUstream_st* cemuStream_t; /* == cudaStream_t */

/* Result codes: same values as ncclResult_t (nccl.h). */
typedef enum {
  cemuSuccess = 0,
  cemuUnhandledCudaError = 1,
  cemuSystemError = 2,
  cemuInternalError = 3,
  cemuInvalidArgument = 4,
  cemuInvalidUsage = 5,
  cemuRemoteError = 6,
  cemuInProgress = 7
} cemuResult_t;

/* Datatypes: same values as ncclDataType_t. */
typedef enum {
  cemuInt8 = 0, cemuUint8 = 1, cemuInt32 = 2, cemuUint32 = 3,
  cemuInt64 = 4, cemuUint64 = 5, cemuFloat16 = 6, cemuFloat32 = 7,
  cemuFloat64 = 8, cemuBfloat16 = 9
} cemuDataType_t;

/* Reduction ops: same values as ncclRedOp_t.  The reference only sums
 * (proj/src/reduce.cpp:7-19); anything but cemuSum is cemuInvalidArgument. */
typedef enum { cemuSum = 0, cemuProd = 1, cemuMax = 2, cemuMin = 3, cemuAvg = 4 } cemuRedOp_t;

#define CEMU_UNIQUE_ID_BYTES 128
typedef struct { char internal[CEMU_UNIQUE_ID_BYTES]; } cemuUniqueId; /* == ncclUniqueId */

typedef struct cemuComm* cemuComm_t;

/* ------------------------------------------------------------------ */
/* Communicator management (ncclGetUniqueId / ncclCommInitRank / ...)  */
/* ------------------------------------------------------------------ */
cemuResult_t cemuGetVersion(int* version);
/* Wraps ncclGetUniqueId when the job places several real ranks on this box;
 * any 128 bytes otherwise. */
cemuResult_t cemuGetUniqueId(cemuUniqueId* uniqueId);
/* ncclCommInitRank shape.  nranks must equal world_size of the config named
 * by $CEMU_CONFIG; rank must be a real rank.  Device = the caller's current
 * CUDA device. */
cemuResult_t cemuCommInitRank(cemuComm_t* comm, int nranks, cemuUniqueId commId, int rank);
/* ncclCommInitAll shape: one process drives `ndev` GPUs (devlist, or
 * 0..ndev-1), which serve the config's real ranks in ascending order.  Call
 * the collectives of all these comms inside cemuGroupStart/End, as with
 * NCCL.  (The fused peer-memory path needs one process per GPU.) */
cemuResult_t cemuCommInitAll(cemuComm_t* comms, int ndev, const int* devlist);
/* Same with the config given as text (reference key=value format). */
cemuResult_t cemuCommInitRankConfig(cemuComm_t* comm, const char* configText,
                                    cemuUniqueId commId, int rank, int cudaDevice);
cemuResult_t cemuCommDestroy(cemuComm_t comm);
cemuResult_t cemuCommCount(const cemuComm_t comm, int* count);      /* world size */
cemuResult_t cemuCommUserRank(const cemuComm_t comm, int* rank);    /* world rank */
cemuResult_t cemuCommCuDevice(const cemuComm_t comm, int* device);
const char* cemuGetErrorString(cemuResult_t result);
/* Last error text of this thread (names the offending field/argument). */
const char* cemuGetLastError(cemuComm_t comm);

/* ------------------------------------------------------------------ */
/* Collectives (NCCL signatures)                                        */
/* ------------------------------------------------------------------ */
/* Ordering (NCCL's semantics; the reference's one-op-in-flight engine,
 * collective.cpp:357-404): a communicator's calls take effect in the order
 * they are issued, also across streams -- a call on another stream than the
 * previous call waits for it on the device (the host never blocks).  As with
 * NCCL, one communicator is driven by one host thread at a time. */
/* replaces WorkerSession::allreduce_async (collective.cpp:213-216) */
cemuResult_t cemuAllReduce(const void* sendbuff, void* recvbuff, size_t count,
                           cemuDataType_t datatype, cemuRedOp_t op, cemuComm_t comm,
                           cemuStream_t stream);
/* replaces WorkerSession::allgather_async (collective.cpp:218-221) */
cemuResult_t cemuAllGather(const void* sendbuff, void* recvbuff, size_t sendcount,
                           cemuDataType_t datatype, cemuComm_t comm, cemuStream_t stream);
/* NEW (absent from the reference, nccl.h:408-410 shape) */
cemuResult_t cemuReduceScatter(const void* sendbuff, void* recvbuff, size_t recvcount,
                               cemuDataType_t datatype, cemuRedOp_t op, cemuComm_t comm,
                               cemuStream_t stream);
/* NEW (absent from the reference, nccl.h:379 shape) */
cemuResult_t cemuBroadcast(const void* sendbuff, void* recvbuff, size_t count,
                           cemuDataType_t datatype, int root, cemuComm_t comm,
                           cemuStream_t stream);
cemuResult_t cemuGroupStart(void);
cemuResult_t cemuGroupEnd(void);

/* Host-buffer forms of allreduce / allgather: `sendbuff`/`recvbuff` are HOST
 * memory, as WorkerSession's spans are (collective.hpp:68-78:
 * allreduce_async(span<uint8_t>, elem_size), allgather_async(span, ...)).
 * Stream-ordered like cudaMemcpyAsync: recvbuff is complete when `stream`
 * reaches the end of the call (cudaStreamSynchronize = WorkerSession::wait).
 * With one real GPU the buffer is pipelined through the device in chunks
 * (H2D, synthesis, D2H overlap; $CEMU_HOST_CHUNK_MIB, default 32); page-
 * locked host memory is needed for the copies to overlap.  Not groupable.
 * Allgather: recvbuff holds world_size blocks of sendcount elements; in
 * place when sendbuff == recvbuff + rank * sendcount. */
cemuResult_t cemuAllReduceHost(const void* sendbuff, void* recvbuff, size_t count,
                               cemuDataType_t datatype, cemuRedOp_t op, cemuComm_t comm,
                               cemuStream_t stream);
cemuResult_t cemuAllGatherHost(const void* sendbuff, void* recvbuff, size_t sendcount,
                               cemuDataType_t datatype, cemuComm_t comm, cemuStream_t stream);

/* Wire mode (interop with a reference `cemu-emulator`).
 * Dials endpoint[successor(rank)] of the comm's config (which must carry
 * endpoint.R keys and the reference's own keys only, so both sides compute
 * the same config digest), performs the HELLO/TOPO handshake with `plan`
 * (transport.hpp:25-40; allgather bytes = per-rank block) and from then on
 * runs cemuAllReduce / cemuAllGather over the CEMU frame protocol exactly
 * as WorkerSession::run_op does (collective.cpp:268-355): outgoing chunks
 * are read from the device buffer, incoming DATA payloads folded on the GPU
 * (int32 lanes when the element size is 4, bytes otherwise).  Calls become
 * host-synchronous; their call record holds the device model's floors and
 * the reference engine's observed release (arrival) times.  Replaces the
 * WorkerSession constructor's dial + handshake (collective.cpp:28-77);
 * detach (or cemuCommDestroy) sends BYE (collective.cpp:406-442). */
typedef struct {
  int32_t coll;     /* 0 allreduce, 1 allgather */
  uint64_t bytes;   /* allreduce: buffer bytes; allgather: per-rank block */
  uint32_t elemSize;
} cemuPlanEntry;
cemuResult_t cemuCommAttachEmulator(cemuComm_t comm, const cemuPlanEntry* plan, size_t nplan,
                                    int timeoutMs);
cemuResult_t cemuCommDetachEmulator(cemuComm_t comm);

/* Symmetric device memory (ncclMemAlloc / window-registration analogue).
 * Collective over the job's real ranks on this box: each allocates `bytes`
 * and maps every peer's allocation (CUDA IPC).  An allreduce whose send and
 * recv lie in such buffers -- at the same offsets on every real rank -- runs
 * as ONE fused kernel over NVLink peer memory instead of NCCL
 * reduce-scatter + synthesis + NCCL allgather.  One real GPU: plain memory. */
cemuResult_t cemuMemAlloc(cemuComm_t comm, size_t bytes, void** ptr);
cemuResult_t cemuMemFree(cemuComm_t comm, void* ptr);
/* Caller memory as a symmetric range: replaces ncclCommRegister /
 * ncclCommDeregister (nccl.h 2.27.3:243-248) and ncclCommWindowRegister /
 * ncclCommWindowDeregister (nccl.h:251-256).  Collective over the job's real
 * ranks on this box: each rank exports the cudaMalloc allocation holding
 * [buff, buff + size) through CUDA IPC and maps every peer's, so
 * collectives whose buffers lie in registered ranges (at the same offsets
 * on every real rank) take the fused NVLink kernels, as with cemuMemAlloc.
 * The caller keeps ownership; deregister before freeing.  Memory that
 * cannot be exported (e.g. cuMem VMM allocations) fails on every rank with
 * cemuInvalidUsage.  One real GPU: bookkeeping only.  A null buffer or zero
 * size registers nothing (*handle = NULL). */
cemuResult_t cemuCommRegister(cemuComm_t comm, void* buff, size_t size, void** handle);
cemuResult_t cemuCommDeregister(cemuComm_t comm, void* handle);
/* Synthesis cache.  The emulated ranks' payloads depend only on
 * (seed, rank, element index), so their per-element sums are the same in
 * every call over the same element range.  A call over a range of >= 1 MiB
 * (or >= 64 KiB when elements x emulated ranks >= 2^21) with >= minPeers
 * emulated ranks writes those sums into a per-communicator
 * cache (2 bytes per element for the byte kinds up to
 * CEMU_SYNTH_CACHE_C16_MAX = 8192 emulated ranks, else 4) and later calls
 * over the range fold from it -- a memory-bound pass
 * instead of issue-bound synthesis, with identical bits.  capBytes bounds
 * each of the two caches (byte kinds / 32-bit integer kinds; default
 * CEMU_SYNTH_CACHE_MB = 4096 MiB, minPeers CEMU_SYNTH_CACHE_MIN_PEERS = 16);
 * capBytes = 0 turns caching off.  Calling this drops every entry. */
cemuResult_t cemuCommSetSynthCache(cemuComm_t comm, size_t capBytes, uint32_t minPeers);
/* Fills (misses that wrote entries) and hits so far, and the device bytes
 * the caches hold. */
cemuResult_t cemuCommSynthCacheStats(cemuComm_t comm, uint64_t* fills, uint64_t* hits, size_t* bytes);

/* Errors raised inside the fused kernel (a peer that never arrived at a
 * barrier within CEMU_FUSED_TIMEOUT_S); synchronous read. */
cemuResult_t cemuCommGetAsyncError(cemuComm_t comm, cemuResult_t* asyncError);

/* ------------------------------------------------------------------ */
/* Emulation observability: the per-call schedule record                */
/* ------------------------------------------------------------------ */
/* Every collective call gets a sequential id (the reference's op_id,
 * collective.cpp:200).  When the delay model is active the device writes
 * the per-step release floors it evaluated (engine.cpp:36-42 semantics,
 * integer us relative to the call start) and the %globaltimer instant each
 * to-real step was released; read them after the stream is synchronized. */
typedef struct {
  uint64_t call_id;
  int32_t coll;          /* 0 allreduce, 1 allgather, 2 reduce-scatter, 3 broadcast */
  int32_t delay_active;  /* 0: no spin kernel was enqueued */
  uint32_t steps;        /* K = to-real messages of the boundary */
  uint32_t world;
  uint64_t model_bytes;  /* m of the delay model */
  int64_t model_latency_us;  /* max_j floor_j (host closed form, A14) */
  int64_t t_start_ns;    /* device %globaltimer at the call's first kernel */
  int64_t t_end_ns;      /* device %globaltimer when the last step released */
  int64_t device_latency_us; /* max_j floor_j as evaluated on the device */
  int64_t t_origin_ns;   /* the schedule's origin: t_start_ns, or the previous
                            call's t_end_ns when queue chaining applied */
  int64_t late_ns;       /* max_j (release_j - (t_origin + floor_j)): > 0 when
                            the emulator's own work (synthesis, NVLink legs)
                            outlasted some step's floor -- that step's release
                            was late even if the call ended on time */
  int64_t overshoot_ns;  /* max(0, t_end - (t_origin + max_j floor_j)): how
                            much longer than modelled the call itself took */
  int64_t stall_ns;      /* the longest interval between two consecutive
                            clock reads of the releasing thread: ~2-4 us (its
                            sleep) normally; a pause of the whole device
                            (nothing of the kernel running, ~1 ms about once
                            a second on the measured boxes) shows here and
                            bounds how late it made a release */
} cemuCallRecord;

/* Delay-model plugin: replaces DelayModelFn / make_delay_model
 * (proj/include/cemu/delay.hpp:52-55, src/delay.cpp:49-53).  The reference's
 * plugin maps (boundary DAG, bytes) to the per-step release offsets; the
 * boundary is closed-form here, so the function receives the collective
 * (0 allreduce, 1 allgather, 2 reduce-scatter, 3 broadcast), the world size,
 * the model bytes and K = the number of to-real steps, and writes K offsets
 * in microseconds from the call's start into offsetsUs (return 0, or
 * non-zero to fail the call with cemuInvalidArgument).  It runs on the host
 * when the call is enqueued; floors = llround(offset) and the head-of-line
 * release are applied on the device exactly as for the built-in models
 * (engine.cpp:36-70).  Setting it activates delay injection on every call;
 * NULL restores the job config's model.  (In a captured CUDA graph the
 * offsets are those of the capture.) */
typedef int (*cemuDelayModelFn)(int coll, uint32_t worldSize, uint64_t bytes, uint32_t k,
                                double* offsetsUs, void* user);
cemuResult_t cemuCommSetDelayModel(cemuComm_t comm, cemuDelayModelFn fn, void* user);
/* Queue chaining (off by default; CEMU_QUEUE_GAP_US sets the default): a
 * delayed call whose first kernel starts within gapUs after the previous
 * delayed call on the same stream ended was queued behind it, and its
 * schedule starts at that end -- an in-order channel starts the next
 * collective when the previous one leaves the wire, without the emulator's
 * own kernel-dispatch gap.  The record keeps both instants (t_start_ns,
 * t_origin_ns).  cemuRunTrainingLoop uses 10 us for its own loop. */
cemuResult_t cemuCommSetQueueChaining(cemuComm_t comm, int64_t gapUs);
/* The real collective's SM footprint.  A real collective's
 * kernel (NCCL: one CTA per channel) occupies SMs for its whole duration,
 * slowing compute that runs beside it on other streams.  With ctas > 0 every
 * delayed call's wait also holds `ctas` CTAs (544 threads, smemBytes of
 * shared memory each) until its modelled end, so that contention is
 * emulated too, and the call's own HBM-bound memory pass (a cached fold, or
 * the synthesis of <= 16 emulated ranks) runs on at most `ctas` CTAs, as the
 * real reduction would.  0 (the default; CEMU_DELAY_HOLD_CTAS / _SMEM)
 * holds one CTA, the schedule's. */
cemuResult_t cemuCommSetDelayFootprint(cemuComm_t comm, int ctas, size_t smemBytes);

cemuResult_t cemuCommLastCallId(cemuComm_t comm, uint64_t* callId);
/* Copies the record (and up to `cap` floors / release times / offsets) of a
 * call still held in the comm's record ring. Synchronous device read. */
cemuResult_t cemuCommCallRecord(cemuComm_t comm, uint64_t callId, cemuCallRecord* rec,
                                int64_t* floorsUs, int64_t* releaseNs, double* offsetsUs,
                                size_t cap);

/* The call's per-step schedule as EventLog lines (proj/include/cemu/
 * trace.hpp:10-34: "<ts_us> <op_id> <event> <direction> <step> <chunk>"):
 * register, from_real / to_real per step, complete -- device %globaltimer
 * times.  Returns the text length, -(needed) if cap is short, -1 on error. */
int cemuCommEventLog(cemuComm_t comm, uint64_t callId, char* out, size_t cap);

/* ------------------------------------------------------------------ */
/* Job config (proj/src/config.cpp) -- bit-compatible render + digest    */
/* ------------------------------------------------------------------ */
typedef struct cemuJobConfig* cemuJobConfig_t;
/* parse_job_config (config.cpp:153-262) + validate (85-149).  On error
 * returns cemuInvalidArgument and writes the ConfigError text (which names
 * the offending field) into err. */
cemuResult_t cemuConfigParse(const char* text, cemuJobConfig_t* cfg, char* err, size_t errcap);
cemuResult_t cemuConfigLoad(const char* path, cemuJobConfig_t* cfg, char* err, size_t errcap);
void cemuConfigFree(cemuJobConfig_t cfg);
/* render_job_config (config.cpp:264-302): returns length, or -(needed). */
int cemuConfigRender(cemuJobConfig_t cfg, char* out, size_t cap);
/* config_digest (config.cpp:304-312): FNV-1a 64 of the render. */
uint64_t cemuConfigDigest(cemuJobConfig_t cfg);
uint32_t cemuConfigWorldSize(cemuJobConfig_t cfg);
/* Writes up to cap real ranks (ascending); returns how many there are. */
uint32_t cemuConfigRealRanks(cemuJobConfig_t cfg, uint32_t* out, size_t cap);

/* synthesize_global_topology (config.cpp:314-331): one node per rank (its
 * node class and whether it is real) and a ring of edges r -> r+1 mod n, each
 * carrying the job's link; the edge structure depends on the world size
 * alone.  Writes up to cap nodes and edges; returns world_size. */
typedef struct {
  int32_t isReal;
  char nodeClass[64]; /* NUL-terminated, truncated to 63 bytes */
} cemuTopoNode;
typedef struct {
  uint32_t src, dst;
  double alphaUs, betaUsPerByte, gammaUsPerByte;
} cemuTopoEdge;
uint32_t cemuConfigTopology(cemuJobConfig_t cfg, cemuTopoNode* nodes, cemuTopoEdge* edges, size_t cap);
/* RingOrder (config.cpp:360-376): ascending ring. */
uint32_t cemuRingSuccessor(uint32_t n, uint32_t rank);
uint32_t cemuRingPredecessor(uint32_t n, uint32_t rank);

/* ------------------------------------------------------------------ */
/* Schedule + delay model (pure host functions, for parity checks)      */
/* ------------------------------------------------------------------ */
/* Delay model parameters: LinkParams + DelayModelParams (config.hpp:18-24,
 * delay.hpp:16-29) plus the new cost-model algorithm selector. */
typedef struct {
  int32_t kind;   /* 0 none, 1 alpha_beta, 2 fixed   (config.hpp:27) */
  int32_t algo;   /* 0 ring (reference), 1 tree, 2 hierarchical (new) */
  double alpha_us, beta_us_per_byte, gamma_us_per_byte;
  double fixed_us, inject_us;
  uint32_t gpus_per_node;          /* hierarchical: ranks per node */
  double intra_alpha_us, intra_beta_us_per_byte;  /* hierarchical intra links */
} cemuDelayModel;

/* dag.cpp:32-46 */
uint64_t cemuChunkBytes(uint32_t n, uint64_t totalBytes, uint32_t elemSize, uint32_t chunk);
uint64_t cemuChunkOffsetBytes(uint32_t n, uint64_t totalBytes, uint32_t elemSize, uint32_t chunk);
/* dag.cpp:73-82; coll 0 allreduce, 1 allgather */
uint32_t cemuPositions(int coll, uint32_t n);
uint32_t cemuSendChunkAt(int coll, uint32_t n, uint32_t rank, uint32_t position);
/* Closed-form project_boundary (dag.cpp:232-338) for one real rank, in the
 * dump_boundary text format (dag.cpp:378-393).  Returns length or -needed. */
int cemuBoundaryDump(int coll, uint32_t n, uint64_t bytes, uint32_t elemSize, uint32_t realRank,
                     char* out, size_t cap);
/* BoundaryDag::count(kToReal) for an arbitrary real set. */
uint32_t cemuToRealCount(int coll, uint32_t n, const uint32_t* real, uint32_t nreal);
/* delay.cpp:5-21 (ring) and the new tree / hierarchical forms. */
double cemuModelTotalUs(const cemuDelayModel* m, int coll, uint32_t n, uint64_t bytes);
/* delay.cpp:23-47 */
int cemuReleaseOffsets(const cemuDelayModel* m, int coll, uint32_t n, uint64_t bytes,
                       uint32_t k, double* out);
/* engine.cpp:36-42 */
int cemuReleaseFloors(const cemuDelayModel* m, int coll, uint32_t n, uint64_t bytes, uint32_t k,
                      int64_t nowUs, int64_t* out);
/* A14 closed form: completion - registration for an instantaneous real node */
int64_t cemuCallLatencyUs(const cemuDelayModel* m, int coll, uint32_t n, uint64_t bytes,
                          uint32_t k);

/* Multi-GPU decomposition of one allreduce over k real GPUs:
 * real GPU li reduce-scatters, synthesises and all-gathers elements
 * [shardOffset, +shardCount); the tail [tailOffset, +tailCount) (< k
 * elements) is all-reduced and synthesised by every real GPU. */
typedef struct {
  uint64_t shardOffset, shardCount, tailOffset, tailCount;
} cemuShardPlan;
void cemuPlanShards(uint64_t count, uint32_t k, uint32_t li, cemuShardPlan* plan);

/* Payload generator (see paper_2405_02969_b200/csrc/payload.cuh). */
uint32_t cemuPayloadKey(uint64_t seed, uint32_t rank);
uint32_t cemuPayloadWord(uint32_t key, uint64_t wordIndex);

/* ------------------------------------------------------------------ */
/* DDP what-if harness (proj/src/harness.cpp)           */
/* ------------------------------------------------------------------ */
typedef struct cemuModelSpec* cemuModelSpec_t;
/* parse_model_spec (harness.cpp:27-101): `layer = fwd_us bwd_us grad_bytes` */
cemuResult_t cemuModelSpecParse(const char* text, cemuModelSpec_t* spec, char* err, size_t errcap);
/* builtin_model (harness.cpp:116-134): bert-like, small, wide */
cemuResult_t cemuModelSpecBuiltin(const char* name, cemuModelSpec_t* spec);
void cemuModelSpecFree(cemuModelSpec_t spec);
int cemuModelSpecRender(cemuModelSpec_t spec, char* out, size_t cap);
uint32_t cemuModelSpecLayers(cemuModelSpec_t spec, int64_t* fwdUs, int64_t* bwdUs, uint64_t* gradBytes,
                             size_t cap, uint32_t* iterations, uint32_t* warmup, int64_t* updateUs);
/* bucketize (harness.cpp:152-175): buckets in issue (reverse layer) order */
uint32_t cemuBucketize(cemuModelSpec_t spec, uint64_t bucketBytes, uint32_t* firstLayer, uint32_t* lastLayer,
                       uint64_t* bytes, size_t cap);
/* run_training_loop (harness.cpp:191-254) on the device: spin-kernel
 * compute on a compute stream, one emulated allreduce (uint8, in order) per
 * filled bucket on a comm stream.  Device-event timestamps in us from the
 * loop's first event: per iteration start/end, per (iteration, bucket)
 * issue/complete (row-major).  cap = iterations the arrays hold. */
cemuResult_t cemuRunTrainingLoop(cemuComm_t comm, cemuModelSpec_t spec, uint64_t bucketBytes,
                                 double* iterStartUs, double* iterEndUs, double* issueUs, double* completeUs,
                                 size_t cap);
/* The ideal timeline of that loop with bucket b's collective taking
 * bucketLatencyUs[b]: iteration time in us. */
double cemuPredictIterationUs(cemuModelSpec_t spec, uint64_t bucketBytes, const double* bucketLatencyUs, size_t n);
/* Modelled latency (A14) of one `coll` call of `bytes` (delay-model bytes) on this comm. */
cemuResult_t cemuCommModelLatencyUs(cemuComm_t comm, int coll, uint64_t bytes, int64_t* latencyUs);
/* Compute emulation (clock.hpp:29-37): a %globaltimer spin of `us` on `stream`. */
cemuResult_t cemuSpinUs(cemuStream_t stream, uint64_t us);
/* Chained compute emulation: `deviceChain` (one int64 in device memory)
 * holds the previous spin's absolute deadline; this spin ends at
 * deadline + us, so launch gaps do not accumulate.  resync != 0 restarts the
 * chain at this kernel's start (use after a cross-stream wait). */
cemuResult_t cemuSpinChainUs(cemuStream_t stream, uint64_t us, int64_t* deviceChain, int resync);
/* The join after a cross-stream wait on a collective: in stream order,
 * *deviceChain = max(*deviceChain, *deviceOther).  With deviceOther = the
 * collective's release end (cemuCommLastReleaseEnd) the compute timeline
 * continues from the later of the two, instead of from the next kernel's
 * start after the event-to-kernel gap (resync). */
cemuResult_t cemuChainJoin(cemuStream_t stream, int64_t* deviceChain, const int64_t* deviceOther);
/* Device word (%globaltimer ns) holding the release end of the last delayed
 * call enqueued on `comm`; *out = NULL when the delay is off.  The word is
 * rewritten 64 calls later (the record ring). */
cemuResult_t cemuCommLastReleaseEnd(cemuComm_t comm, const int64_t** out);

#ifdef __cplusplus
}
#endif
#endif /* CEMU_B200_H_ */
