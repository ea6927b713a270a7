/* oracle/cemu_oracle.h -- TEST INFRASTRUCTURE ONLY (the checker, never the
 * product).  Plain-C restatement of the reference's collective-emulation hot
 * path (arxiv 2405.02969 "NeuronaBox", C++ re-creation `cemu` under
 * /root/reference/proj), plus the payload generator and fold this build
 * defines for the gaps the reference does not cover.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load liboracle.so.
 *
 * Pinning:
 *   - chunking, ring schedule, boundary, delay model, release offsets,
 *     OpState floors, call latency: pinned bit-exactly against the reference
 *     itself (oracle/_ref/libcemu_ref.so built from /root/reference) and its
 *     own golden files / KATs (tests/golden/).
 *   - zero-payload ("ref-dummy") collective results: pinned against the
 *     reference emulator's actual outputs (WorkerSession + EmulatorServer).
 *   - integer hash-payload allreduce/allgather: pinned against the
 *     reference's all-real TCP ring fed the same hash inputs.
 *   - float folds, reduce-scatter, broadcast, tree/hierarchical delay:
 *     "parity unpinned" -- defined here (the reference has no such code).
 */
#ifndef CEMU_ORACLE_H_
#define CEMU_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* collective kinds */
enum { OR_ALLREDUCE = 0, OR_ALLGATHER = 1, OR_REDUCESCATTER = 2, OR_BROADCAST = 3 };
/* delay kinds: config.hpp:27 order (none, alpha_beta, fixed) */
enum { OR_DELAY_NONE = 0, OR_DELAY_ALPHA_BETA = 1, OR_DELAY_FIXED = 2 };
/* cost-model algorithms (ring is the reference's only one) */
enum { OR_ALGO_RING = 0, OR_ALGO_TREE = 1, OR_ALGO_HIER = 2 };
/* dtypes: ncclDataType_t values (nccl.h) */
enum { OR_INT8 = 0, OR_UINT8 = 1, OR_INT32 = 2, OR_UINT32 = 3, OR_INT64 = 4,
       OR_UINT64 = 5, OR_FLOAT16 = 6, OR_FLOAT32 = 7, OR_FLOAT64 = 8,
       OR_BFLOAT16 = 9 };
/* payload modes */
enum { OR_PAYLOAD_HASH = 0, OR_PAYLOAD_ZERO = 1 };

typedef struct {
  int kind;            /* OR_DELAY_* */
  int algo;            /* OR_ALGO_* */
  double alpha_us, beta_us_per_byte, gamma_us_per_byte;
  double fixed_us, inject_us;
  uint32_t gpus_per_node;          /* hierarchical only */
  double intra_alpha_us, intra_beta_us_per_byte;  /* hierarchical only */
} or_delay_model;

/* ---- schedule: proj/src/dag.cpp:32-82 ---------------------------------- */
uint64_t or_chunk_bytes(uint32_t n, uint64_t total, uint32_t elem, uint32_t c);
uint64_t or_chunk_offset_bytes(uint32_t n, uint64_t total, uint32_t elem,
                               uint32_t c);
uint32_t or_positions(int coll, uint32_t n);
uint32_t or_send_chunk_at(int coll, uint32_t n, uint32_t rank, uint32_t p);
/* Closed-form emulated-side boundary for one real rank, rendered in the
 * dump_boundary format (dag.cpp:378-393).  Returns length or -needed. */
int or_dump_boundary_single_real(int coll, uint32_t n, uint64_t bytes,
                                 uint32_t elem, uint32_t real, char* out,
                                 size_t cap);
/* Number of to-real boundary messages for an arbitrary real set. */
uint32_t or_to_real_count(int coll, uint32_t n, const uint32_t* real,
                          uint32_t nreal);

/* ---- delay model: proj/src/delay.cpp:5-47, engine.cpp:36-42 ----------- */
double or_ring_allreduce_delay_us(uint32_t n, uint64_t bytes, double a,
                                  double b, double g);
double or_ring_allgather_delay_us(uint32_t n, uint64_t bytes, double a,
                                  double b);
double or_model_total_us(const or_delay_model* m, int coll, uint32_t n,
                         uint64_t bytes);
int or_release_offsets(const or_delay_model* m, int coll, uint32_t n,
                       uint64_t bytes, uint32_t k, double* out);
int or_release_floors(const or_delay_model* m, int coll, uint32_t n,
                      uint64_t bytes, uint32_t k, int64_t now_us,
                      int64_t* out);
int64_t or_call_latency_us(const or_delay_model* m, int coll, uint32_t n,
                           uint64_t bytes, uint32_t k);

/* ---- payload generator (new; its bits are the spec) ------------------- */
uint32_t or_payload_key(uint64_t seed, uint32_t rank);
uint32_t or_payload_word(uint32_t key, uint64_t word_index);
/* Synthesised contribution of one rank for elements [first, first+count). */
void or_payload(int dtype, uint32_t key, uint64_t first, uint64_t count,
                void* out);

/* ---- collectives (expected outputs) ----------------------------------- */
/* `real` lists the real ranks (ascending), `sends[i]` is real[i]'s buffer.
 * The real part is summed in ascending real-rank order (callers that compare
 * against NCCL use inputs whose real sum is exact). */
int or_allreduce(int dtype, int mode, uint32_t W, const uint32_t* real,
                 uint32_t nreal, uint32_t me, uint64_t seed,
                 const void* const* sends, void* recv, uint64_t count);
int or_allgather(int dtype, int mode, uint32_t W, const uint32_t* real,
                 uint32_t nreal, uint32_t me, uint64_t seed,
                 const void* const* sends, void* recv, uint64_t sendcount);
int or_reducescatter(int dtype, int mode, uint32_t W, const uint32_t* real,
                     uint32_t nreal, uint32_t me, uint64_t seed,
                     const void* const* sends, void* recv, uint64_t recvcount);
int or_broadcast(int dtype, int mode, uint32_t W, const uint32_t* real,
                 uint32_t nreal, uint32_t me, uint32_t root, uint64_t seed,
                 const void* root_send, void* recv, uint64_t count);

/* ---- ring-order fold: proj/tests/oracles.hpp:43-101 ------------------- */
/* Executes the ring schedule over n full input buffers (inputs[r], count
 * elements each) and writes rank `me`'s final buffer.  int32 wraps; float32
 * folds dst = dst + incoming in fp32 exactly in the ring's order. */
int or_ring_execute_allreduce(int dtype, uint32_t n, const void* const* inputs,
                              uint64_t count, uint32_t me, void* out);

/* rounding helpers shared by tests */
uint16_t or_f32_to_bf16(float f);
float or_bf16_to_f32(uint16_t h);
uint16_t or_f32_to_f16(float f);
float or_f16_to_f32(uint16_t h);

#ifdef __cplusplus
}
#endif
#endif
