// comm.cpp -- the NCCL-shaped communicator of the emulated world.
//
// One cemuComm per real rank (one process per GPU).  Its world is the job's
// world_size; the real ranks of the job are the GPUs on this box and share
// an inner NCCL communicator (only created when there are several).  Every
// collective splits into
//   real part      NCCL over NVLink among the local real GPUs (k > 1 only)
//   emulated part  sm_100a kernels synthesising the W-k emulated peers'
//                  payloads and folding them in (kernels.cu)
//   network delay  the device-evaluated alpha-beta model released on
//                  %globaltimer by a spin kernel on the same stream
// replacing WorkerSession::run_op's TCP ring (proj/src/collective.cpp:
// 268-355) and the emulator process (proj/src/emulator.cpp:59-272).
//
// Stream-ordered, asynchronous; the host never blocks.  Argument and usage
// errors map to cemuInvalidArgument / cemuInvalidUsage with a message that
// names the offending argument (cemuGetLastError), as the reference's
// TransportError/ConfigError texts do (collective.cpp:190-205).
//
// Shared declarations: comm_internal.hpp; the host-buffer pipeline lives in
// host_pipe.cpp, wire mode in comm_wire.cpp, symmetric memory and buffer
// registration in symmetric.cpp, the synthesis cache in synth_cache.cpp.
#include "comm_internal.hpp"
#include "harness.hpp"

namespace cemu_b200 {

thread_local std::string g_last_error;

cemuResult_t fail(cemuResult_t code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// ---- NCCL, loaded on demand (only jobs with several real GPUs need it) ----


std::mutex g_nccl_mu;
Nccl g_nccl;
bool g_nccl_tried = false;

const Nccl* nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (!g_nccl_tried) {
    g_nccl_tried = true;
    const char* env = std::getenv("CEMU_NCCL_LIB");
    // an already-loaded libnccl.so.2 (e.g. torch's) is reused by soname
    void* h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("/usr/lib/x86_64-linux-gnu/libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      Nccl n;
      n.h = h;
#define CEMU_SYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name))
      CEMU_SYM(GetUniqueId, "ncclGetUniqueId");
      CEMU_SYM(CommInitRank, "ncclCommInitRank");
      CEMU_SYM(CommInitAll, "ncclCommInitAll");
      CEMU_SYM(CommDestroy, "ncclCommDestroy");
      CEMU_SYM(AllReduce, "ncclAllReduce");
      CEMU_SYM(AllGather, "ncclAllGather");
      CEMU_SYM(ReduceScatter, "ncclReduceScatter");
      CEMU_SYM(Broadcast, "ncclBroadcast");
      CEMU_SYM(Reduce, "ncclReduce");
      CEMU_SYM(GroupStart, "ncclGroupStart");
      CEMU_SYM(GroupEnd, "ncclGroupEnd");
      CEMU_SYM(GetErrorString, "ncclGetErrorString");
#undef CEMU_SYM
      if (n.GetUniqueId && n.CommInitRank && n.AllReduce && n.AllGather && n.ReduceScatter &&
          n.Broadcast && n.Reduce && n.GroupStart && n.GroupEnd && n.CommDestroy) {
        g_nccl = n;
      }
    }
  }
  return g_nccl.h ? &g_nccl : nullptr;
}

size_t dtype_size(int dt) {
  switch (dt) {
    case cemuInt8: case cemuUint8: return 1;
    case cemuFloat16: case cemuBfloat16: return 2;
    case cemuInt32: case cemuUint32: case cemuFloat32: return 4;
    case cemuInt64: case cemuUint64: case cemuFloat64: return 8;
    default: return 0;
  }
}

thread_local int g_group_depth = 0;
thread_local std::vector<GroupOp> g_group_ops;

cemuResult_t grow_buffer(cemuComm* c, void** buf, size_t* have, size_t bytes, const char* what) {
  if (*have >= bytes) return cemuSuccess;
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return fail(cemuUnhandledCudaError, std::string(what) + ": " + cudaGetErrorString(e));
  if (*buf) c->retired.push_back(*buf);  // an enqueued or captured call may still use it
  *buf = p;
  *have = bytes;
  return cemuSuccess;
}

cemuResult_t ensure_scratch(cemuComm* c, size_t bytes) {
  return grow_buffer(c, &c->scratch, &c->scratch_bytes, bytes, "staging buffer");
}

bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone;
}

// CEMU_ORDER=0 removes the ordering (diagnostic: tests/interleave_worker.py
// shows what goes wrong without it)
bool ordering_on() {
  static const bool on = [] {
    const char* e = std::getenv("CEMU_ORDER");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

cemuResult_t order_begin(cemuComm* c, cudaStream_t s) {
  if (!ordering_on() || !c->order_recorded || c->order_stream == s) return cemuSuccess;  // stream order suffices
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  CUDA_OK(cudaStreamGetCaptureInfo(s, &st, &id));
  if (st == cudaStreamCaptureStatusActive) {
    if (c->order_capture == id) {
      CUDA_OK(cudaStreamWaitEvent(s, c->order_ev, 0));  // recorded earlier in this capture
    } else if (c->order_capture == 0) {
      // recorded eagerly: the graph waits, at each launch, for the event's
      // latest record (an external event node)
      CUDA_OK(cudaStreamWaitEvent(s, c->order_ev, cudaEventWaitExternal));
    }
    // recorded inside another capture: that graph's launch orders it
  } else if (c->order_capture == 0) {
    CUDA_OK(cudaStreamWaitEvent(s, c->order_ev, 0));
  }
  return cemuSuccess;
}

cemuResult_t order_end(cemuComm* c, cudaStream_t s) {
  if (!ordering_on()) return cemuSuccess;
  if (!c->order_ev) CUDA_OK(cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming));
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  CUDA_OK(cudaStreamGetCaptureInfo(s, &st, &id));
  CUDA_OK(cudaEventRecord(c->order_ev, s));
  c->order_stream = s;
  c->order_recorded = true;
  c->order_capture = st == cudaStreamCaptureStatusActive ? id : 0;
  return cemuSuccess;
}

// 20-bit signature of a fused call; every real rank must compute the same
uint64_t buf_tag(const cemuComm::Region* r, uint64_t off) { return r ? (r->id << 40) ^ off : 0; }

uint32_t op_sig(int coll, int dt, uint64_t count, uint64_t bufs) {
  uint64_t h = 1469598103934665603ull;
  for (uint64_t v : {static_cast<uint64_t>(coll), static_cast<uint64_t>(dt), count, bufs}) {
    h ^= v;
    h *= 1099511628211ull;
  }
  return static_cast<uint32_t>(h ^ (h >> 32)) & 0xFFFFFu;
}


const cemuComm::Region* find_region(const cemuComm* c, const void* p, size_t bytes) {
  const auto* b = static_cast<const uint8_t*>(p);
  for (const auto& r : c->regions) {
    if (b >= r.base && b + bytes <= r.base + r.bytes) return &r;
  }
  return nullptr;
}

cemuResult_t check_common(cemuComm* c, int dt, const char* what) {
  if (!c) return fail(cemuInvalidArgument, std::string(what) + ": comm is null");
  if (dtype_size(dt) == 0) {
    return fail(cemuInvalidArgument, std::string(what) + ": unsupported datatype " + std::to_string(dt));
  }
  if (cudaSetDevice(c->device) != cudaSuccess) {
    return fail(cemuUnhandledCudaError, std::string(what) + ": cannot select device");
  }
  return cemuSuccess;
}

cemuResult_t check_op(int op, const char* what) {
  if (op != cemuSum) {
    return fail(cemuInvalidArgument,
                std::string(what) + ": only cemuSum is supported (the reference only sums)");
  }
  return cemuSuccess;
}

// `preinit` (cemuCommInitAll): an inner NCCL comm made by ncclCommInitAll in
// this process; the fused path needs one process per GPU (IPC) and is off.
cemuResult_t init_comm(cemuComm_t* out, JobConfig cfg, const cemuUniqueId& id, int rank, int device,
                       ncclComm_t preinit = nullptr) {
  if (!out) return fail(cemuInvalidArgument, "cemuCommInitRank: comm pointer is null");
  if (rank < 0 || static_cast<uint32_t>(rank) >= cfg.world_size) {
    return fail(cemuInvalidArgument, "rank " + std::to_string(rank) + " out of range [0," +
                                         std::to_string(cfg.world_size - 1) + "]");
  }
  if (!cfg.is_real(static_cast<uint32_t>(rank))) {
    return fail(cemuInvalidArgument,
                "rank " + std::to_string(rank) + " is not a real rank in this job");
  }
  auto c = std::make_unique<cemuComm>();
  c->W = cfg.world_size;
  c->rank = static_cast<uint32_t>(rank);
  c->device = device;
  c->real.assign(cfg.real_ranks.begin(), cfg.real_ranks.end());
  c->k = static_cast<uint32_t>(c->real.size());
  c->li = static_cast<uint32_t>(std::find(c->real.begin(), c->real.end(), c->rank) - c->real.begin());
  c->contiguous = c->real.back() - c->real.front() + 1 == c->k;
  c->seed = cfg.payload_seed;
  c->mode = cfg.payload_mode;
  c->delay.kind = static_cast<int32_t>(cfg.delay_kind);
  c->delay.algo = static_cast<int32_t>(cfg.algo());
  c->delay.alpha_us = cfg.link.alpha_us;
  c->delay.beta_us_per_byte = cfg.link.beta_us_per_byte;
  c->delay.gamma_us_per_byte = cfg.link.gamma_us_per_byte;
  c->delay.fixed_us = cfg.delay_fixed_us;
  c->delay.inject_us = cfg.delay_inject_us;
  c->delay.gpus_per_node = cfg.gpus_per_node;
  c->delay.intra_alpha_us = cfg.intra_alpha_us;
  c->delay.intra_beta_us_per_byte = cfg.intra_beta_us_per_byte;
  c->delay_active = cfg.delay_kind != DelayKind::kNone || cfg.delay_inject_us != 0.0;
  c->config_delay_active = c->delay_active;
  c->queue_gap_ns = queue_gap_ns();
  if (const char* h = std::getenv("CEMU_DELAY_HOLD_CTAS")) c->hold_ctas = std::max(0, std::atoi(h));
  if (const char* h = std::getenv("CEMU_DELAY_HOLD_SMEM")) c->hold_smem = std::max(0, std::atoi(h));
  if (const char* h = std::getenv("CEMU_DELAY_HOLD_ACTIVE")) c->hold_active = std::atoi(h) ? 1 : 0;
  {
    const char* mb = std::getenv("CEMU_SYNTH_CACHE_MB");
    c->cache_cap = (mb ? std::strtoull(mb, nullptr, 10) : 4096ull) << 20;
    if (const char* mp = std::getenv("CEMU_SYNTH_CACHE_MIN_PEERS")) {
      c->cache_min_peers = static_cast<uint32_t>(std::max(1, std::atoi(mp)));
    }
  }
  if (c->mode == PayloadMode::kZero && c->k != 1) {
    return fail(cemuInvalidUsage,
                "payload.mode: zero reproduces the reference emulator, which serves exactly "
                "one real rank (emulator.cpp:75-79)");
  }
  std::vector<uint32_t> keys;
  for (uint32_t r = 0; r < c->W; ++r) {
    if (!cfg.is_real(r)) {
      c->virt.push_back(r);
      keys.push_back(payload_key(c->seed, r));
    }
  }
  if (c->virt.size() > kMaxEmulatedPeers) {
    return fail(cemuInvalidArgument, "world_size: " + std::to_string(c->virt.size()) +
                                         " emulated ranks exceed the " + std::to_string(kMaxEmulatedPeers) +
                                         " one GPU can synthesise per call");
  }
  c->cfg = std::move(cfg);
  if (cudaSetDevice(device) != cudaSuccess) return fail(cemuUnhandledCudaError, "cudaSetDevice failed");
  CUDA_OK(cudaMalloc(&c->d_virt_keys, keys.size() * 4));
  CUDA_OK(cudaMalloc(&c->d_virt_ranks, c->virt.size() * 4));
  CUDA_OK(cudaMemcpy(c->d_virt_keys, keys.data(), keys.size() * 4, cudaMemcpyHostToDevice));
  CUDA_OK(cudaMemcpy(c->d_virt_ranks, c->virt.data(), c->virt.size() * 4, cudaMemcpyHostToDevice));
  for (int coll = 0; coll < 4; ++coll) c->kmax = std::max(c->kmax, to_real_count(coll, c->W, c->real));
  CUDA_OK(preload_delay_kernels());
  CUDA_OK(cudaMalloc(&c->d_slots, cemuComm::kSlots * slot_words(c->kmax) * 8));
  CUDA_OK(cudaMemset(c->d_slots, 0, cemuComm::kSlots * slot_words(c->kmax) * 8));
  if (c->k > 1) {
    const Nccl* n = nccl();
    if (!n) {
      return fail(cemuSystemError,
                  "job places " + std::to_string(c->k) +
                      " real ranks on this box but libnccl.so.2 could not be loaded");
    }
    if (preinit) {
      c->inner = preinit;
    } else {
      ncclUniqueId nid;
      static_assert(sizeof(nid) == sizeof(id), "unique id size");
      std::memcpy(&nid, &id, sizeof nid);
      NCCL_OK(n->CommInitRank(&c->inner, static_cast<int>(c->k), nid, static_cast<int>(c->li)));
    }
    const char* fe = std::getenv("CEMU_FUSED");
    c->fused = !preinit && c->k <= static_cast<uint32_t>(kMaxReal) && !(fe && std::string(fe) == "0");
    if (const char* t = std::getenv("CEMU_FUSED_TIMEOUT_S")) c->fused_timeout_ns = std::atoll(t) * 1'000'000'000LL;
    if (const char* ce = std::getenv("CEMU_CE")) c->ce = std::string(ce) == "0" ? 0 : std::string(ce) == "1" ? 1 : 2;
    if (c->fused) {
      CUDA_OK(cudaMalloc(&c->sig, 4096));
      CUDA_OK(cudaMemset(c->sig, 0, 4096));
      if (auto r = map_peers(c.get(), c->sig, 4096, c->peer_sig)) return r;
    }
  }
  *out = c.release();
  return cemuSuccess;
}

// ----------------------------------------------------------------------------
// collective bodies
// ----------------------------------------------------------------------------
// Fused allreduce over `count` elements whose payload indices start at e0
// (a word boundary): this GPU reduces its 1/k of the 16-byte vectors, the
// last GPU also the ragged tail.  src/dst: every real GPU's buffer.
FusedArgs fused_allreduce_args(const cemuComm* c, int dt, uint64_t count, uint64_t e0, uint8_t* const* src,
                               uint8_t* const* dst) {
  FusedArgs a;
  const uint64_t es = dtype_size(dt);
  const uint64_t epv = 16 / es;
  const uint64_t nvec = count / epv;
  const uint64_t per = nvec / c->k;
  a.k = static_cast<int>(c->k);
  a.me = static_cast<int>(c->li);
  a.ndst = a.k;
  a.word_base = (dt == cemuInt32 || dt == cemuUint32) ? e0 : e0 / 4;
  a.v_begin = per * c->li;
  a.v_end = c->li + 1 == c->k ? nvec : per * (c->li + 1);
  a.ntail = c->li + 1 == c->k ? static_cast<uint32_t>(count - nvec * epv) : 0;
  a.tail_e0 = e0 + nvec * epv;
  for (uint32_t g = 0; g < c->k; ++g) {
    a.src[g] = reinterpret_cast<const uint4*>(src[g]);
    a.dst[g] = reinterpret_cast<uint4*>(dst[g]);
  }
  a.keys = c->d_virt_keys;
  a.nkeys = static_cast<uint32_t>(c->virt.size());
  return a;
}

// CEMU_DEBUG=INFO: one stderr line per call naming the path it took (the
// NCCL_DEBUG analogue), so a job can see whether its buffers reach the
// fused kernels.
int debug_level() {  // CEMU_DEBUG: INFO = 1, TRACE = 2
  static const int level = [] {
    const char* e = std::getenv("CEMU_DEBUG");
    return !e ? 0 : std::string(e) == "TRACE" ? 2 : std::string(e) == "INFO" ? 1 : 0;
  }();
  return level;
}

void log_path(const cemuComm* c, const char* coll, uint64_t bytes, const char* path) {
  if (debug_level() >= 1) {
    std::fprintf(stderr, "cemu: rank %u %s %llu B -> %s\n", c->rank, coll, static_cast<unsigned long long>(bytes),
                 path);
  }
}

// Copy-engine allreduce at k = 2 (probe: profiles/
// ce_pipeline_probe.cu): start barrier; per chunk of this GPU's slice the
// copy engine pulls the peer's chunk into staging and the fused kernel in
// fold-only mode adds local + staged (ascending real rank, as the fused
// path) and the emulated ranks, storing into the local recv and the peer's
// -- the peer store only after a successful start barrier; done barrier.
// The pulls leave the SMs, so the NVLink legs run on both the copy engines
// and the SMs.  Bit-identical to the fused kernel (same fold code).  Chosen
// where it measured faster: two real GPUs, >= 512 MiB, a count divisible
// into 16-byte vectors, <= 16 emulated ranks (CEMU_CE=1 forces it,
// CEMU_CE=0 disables it; 1 GiB: fp32 1.547 vs 1.634 ms, bf16 1.567 vs
// 1.680, int32 1.574 vs 1.680 -- profiles/r02_ce_pull_only.txt).
constexpr uint64_t kCeMinBytes = 512ull << 20;

// Chunk of the slice: at most CEMU_CE_CHUNK_MIB (default 256; measured
// 1 GiB k = 2: 256 MiB chunks 1.452 ms, 128 MiB 1.517, one chunk 1.764) and
// at least two chunks, so the pull, the fold and the push overlap.
uint64_t ce_chunk_vecs(uint64_t slice_vecs) {
  static const uint64_t cap = [] {
    const char* e = std::getenv("CEMU_CE_CHUNK_MIB");
    return (e ? std::max<uint64_t>(1, std::strtoull(e, nullptr, 10)) : uint64_t{256}) << 20;
  }() / 16;
  const uint64_t n = std::max<uint64_t>(2, (slice_vecs + cap - 1) / cap);
  return (slice_vecs + n - 1) / n;
}

// Auto mode also needs a cheap synthesis: the pipeline serialises the
// first pull and the last push around the folds, which only pays while the
// NVLink legs dominate (measured 1 GiB k = 2: 14 emulated ranks fp32 1.55 vs
// 1.64 ms fused, bf16 1.11 vs 1.26; 126 emulated ranks bf16 3.19 vs 2.45).
constexpr size_t kCeMaxAutoPeers = 16;

// The larger of the two slices: every rank sizes its staging alike, so the
// capture-time check below agrees across ranks.
// The largest rank's slice (the last rank's: the ragged remainder) in
// 16-byte vectors: every rank sizes its per-peer staging alike, so the
// capture-time check below agrees across ranks.
uint64_t ce_stage_vecs(uint64_t count, size_t es, uint32_t k) {
  const uint64_t nvec = count / (16 / es);
  return nvec - nvec / k * (k - 1);
}

// Every real rank must take the same decision (they meet in the barriers),
// so it only looks at symmetric quantities: the count's ragged tail, not
// this rank's share of it.  Inside a stream capture the staging cannot
// grow (no allocation there), so such a call stays on the fused kernel.
bool ce_allreduce_fits(const cemuComm* c, const FusedArgs& a, uint64_t count, size_t es, cudaStream_t s) {
  const uint64_t bytes = count * es;
  if (!c->ce || c->k < 2 || bytes < kCeMinBytes || count % (16 / es) != 0) return false;
  if (c->ce == 2 && c->k != 2) return false;  // measured faster at two GPUs; CEMU_CE=1 forces it at k > 2
  // many emulated ranks: only while the synthesis cache serves the folds
  // (synthesised folds are issue-bound and the pipeline serialises around
  // them; cached ones are memory-bound: 1 GiB at worlds 32-128, 1.53 vs
  // 1.63 ms fused -- profiles/r02_ce_pull_only.txt)
  if (c->ce == 2 && c->virt.size() > kCeMaxAutoPeers &&
      !(c->cache_cap > 0 && c->virt.size() >= c->cache_min_peers)) {
    return false;
  }
  const uint64_t sv = ce_stage_vecs(count, es, c->k);
  if (c->cep.stage_bytes < (c->k - 1) * sv * 16 && capturing(s)) return false;
  (void)a;
  const uint64_t chunks = (sv + ce_chunk_vecs(sv) - 1) / ce_chunk_vecs(sv);
  return chunks * (c->k - 1) <= cemuComm::CePipe::kEvents - 2;  // the event pool
}

cemuResult_t ce_allreduce(cemuComm* c, int dt, FusedArgs a, uint64_t stage_vecs, cudaStream_t s, Call* call) {
  auto& p = c->cep;
  const uint32_t k = c->k;
  const uint64_t slice = stage_vecs * 16;  // per peer
  for (uint32_t g = 0; g < k; ++g) {
    if (g != c->li && !p.pull[g]) CUDA_OK(cudaStreamCreateWithFlags(&p.pull[g], cudaStreamNonBlocking));
  }
  for (cudaEvent_t& ev : p.ev) {
    if (!ev) CUDA_OK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  if (auto r = grow_buffer(c, &p.stage, &p.stage_bytes, (k - 1) * slice, "copy-engine staging")) return r;
  a.stamp = call->take_stamp();
  CUDA_OK(cache_fused(c, dt, a, s, &call->launches));  // the fold-only chunks inherit it
  CUDA_OK(launch_peer_barrier(a, 0, s, &call->launches));
  cudaEvent_t started = p.ev[0];
  CUDA_OK(cudaEventRecord(started, s));
  // fold-only chunks of the fused kernel: local + every peer's staged data
  // + the emulated ranks, stored into every real GPU's recv -- the peer
  // stores gated on the start barrier's verdict (the comm's error word), so
  // ranks that disagree never write into each other's memory
  FusedArgs f = a;
  f.barriers = 0;
  f.stamp = nullptr;
  f.ndst = static_cast<int>(k);
  f.gate = a.error;
  uintptr_t stage_at[kMaxReal] = {};
  // CEMU_CE_DIRECT = d: the d peers after this GPU in ring order are read by
  // the fold kernels straight from their send buffers over NVLink (SM loads,
  // after the start barrier like the fused kernel's), the others staged by
  // the copy engines -- a split of the incoming NVLink leg between the two
  // engines (at k = 4 concurrent copy-engine pulls from every peer lose)
  static const uint32_t direct_env = [] {
    const char* e = std::getenv("CEMU_CE_DIRECT");
    return e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : 0u;
  }();
  const uint32_t direct = std::min(direct_env, k - 1);
  bool staged[kMaxReal] = {};
  for (uint32_t g = 0, slot = 0; g < k; ++g) {
    if (g == c->li) continue;
    if ((g + k - c->li) % k <= direct) continue;  // read directly: f.src[g] stays the peer's send
    staged[g] = true;
    CUDA_OK(cudaStreamWaitEvent(p.pull[g], started, 0));
    // peer g's staging, indexed like the buffers: vector v at stage[v - v_begin]
    stage_at[g] = reinterpret_cast<uintptr_t>(p.stage) + slot++ * slice - a.v_begin * 16;
    f.src[g] = reinterpret_cast<const uint4*>(stage_at[g]);
  }
  const uint64_t cvec = ce_chunk_vecs(a.v_end - a.v_begin);
  int ev = 2;
  for (uint64_t v0 = a.v_begin; v0 < a.v_end; v0 += cvec) {
    const uint64_t v1 = std::min(a.v_end, v0 + cvec);
    for (uint32_t g = 0; g < k; ++g) {  // every staged peer's chunk on its own copy stream
      if (!staged[g]) continue;
      cudaEvent_t pulled = p.ev[ev++];
      CUDA_OK(cudaMemcpyAsync(reinterpret_cast<void*>(stage_at[g] + v0 * 16), a.src[g] + v0, (v1 - v0) * 16,
                              cudaMemcpyDeviceToDevice, p.pull[g]));
      CUDA_OK(cudaEventRecord(pulled, p.pull[g]));
      CUDA_OK(cudaStreamWaitEvent(s, pulled, 0));
    }
    f.v_begin = v0;
    f.v_end = v1;
    CUDA_OK(launch_fused_allreduce(dt, f, s, &call->launches));
  }
  // done: the peers' stores into my recv are complete, and they no longer
  // read my send
  CUDA_OK(launch_peer_barrier(a, 1, s, &call->launches));
  CUDA_OK(call->finish(kAllReduce));
  return cemuSuccess;
}

cemuResult_t do_allreduce(const void* send, void* recv, size_t count, int dt, cemuComm* c,
                          cudaStream_t s, Phases& ph) {
  const size_t es = dtype_size(dt);
  if (count == 0) return cemuSuccess;
  auto call = std::make_shared<Call>(c, kAllReduce, count * es, s);
  if (!call->error.empty()) return fail(cemuInvalidArgument, call->error);
  const uint32_t nk = static_cast<uint32_t>(c->virt.size());
  if (c->mode == PayloadMode::kZero) ph.push_back([=]() -> cemuResult_t {
    // A10: zero replies; the real rank keeps chunk (rank+1) mod W
    // (test_transport.cpp:129-167), every other chunk is gathered zeros.
    CUDA_OK(call->stamp_now());
    const uint64_t total = count * es;
    const uint32_t keep = (c->rank + 1) % c->W;
    const uint64_t off = chunk_offset_bytes(c->W, total, static_cast<uint32_t>(es), keep);
    const uint64_t len = chunk_bytes(c->W, total, static_cast<uint32_t>(es), keep);
    auto* r8 = static_cast<uint8_t*>(recv);
    if (off) CUDA_OK(cudaMemsetAsync(r8, 0, off, s));
    if (send != recv && len) {
      CUDA_OK(cudaMemcpyAsync(r8 + off, static_cast<const uint8_t*>(send) + off, len,
                              cudaMemcpyDeviceToDevice, s));
    }
    if (total - off - len) CUDA_OK(cudaMemsetAsync(r8 + off + len, 0, total - off - len, s));
    CUDA_OK(call->finish(kAllReduce));
    return cemuSuccess;
  });
  if (c->mode == PayloadMode::kZero) return log_path(c, "allreduce", count * es, "zero payload"), cemuSuccess;
  if (c->k == 1) {
    log_path(c, "allreduce", count * es, "synthesis");
    ph.push_back([=]() -> cemuResult_t {
      CUDA_OK(synth_reduce(c, dt, send, recv, count, 0, call->take_stamp(), s, &call->launches));
      CUDA_OK(call->finish(kAllReduce));
      return cemuSuccess;
    });
    return cemuSuccess;
  }
  // k real GPUs, buffers from cemuMemAlloc: one fused kernel over peer memory
  const cemuComm::Region* rs = c->fused ? find_region(c, send, count * es) : nullptr;
  const cemuComm::Region* rr = c->fused ? find_region(c, recv, count * es) : nullptr;
  if (rs && rr && dtype_size(dt) <= 4 && dt != cemuInt64 && nk > 0) {
    const uint64_t soff = static_cast<const uint8_t*>(send) - rs->base;
    const uint64_t roff = static_cast<uint8_t*>(recv) - rr->base;
    uint8_t* sp[kMaxReal];
    uint8_t* dp[kMaxReal];
    for (uint32_t g = 0; g < c->k; ++g) {
      sp[g] = rs->peer[g] + soff;
      dp[g] = rr->peer[g] + roff;
    }
    FusedArgs a = fused_allreduce_args(c, dt, count, 0, sp, dp);
    const uint64_t tags = buf_tag(rs, soff) * 31 + buf_tag(rr, roff);
    if ((soff | roff) % 16 == 0 && ce_allreduce_fits(c, a, count, es, s)) {
      log_path(c, "allreduce", count * es, "copy-engine pipeline");
      ph.push_back([=]() mutable -> cemuResult_t {
        set_barrier(c, a);
        a.sig = op_sig(kAllReduce, dt, count, tags);
        return ce_allreduce(c, dt, a, ce_stage_vecs(count, es, c->k), s, call.get());
      });
      return cemuSuccess;
    }
    if ((soff | roff) % 16 == 0) log_path(c, "allreduce", count * es, "fused");
    if ((soff | roff) % 16 == 0) ph.push_back([=]() mutable -> cemuResult_t {
      set_barrier(c, a);
      a.sig = op_sig(kAllReduce, dt, count, tags);
      a.ndst = a.k;
      a.stamp = call->take_stamp();
      CUDA_OK(cache_fused(c, dt, a, s, &call->launches));
      CUDA_OK(launch_fused_allreduce(dt, a, s, &call->launches));
      CUDA_OK(call->finish(kAllReduce));
      return cemuSuccess;
    });
    if ((soff | roff) % 16 == 0) return cemuSuccess;
  }
  // k real GPUs: NCCL reduce-scatter of the real part, synthesis on this
  // GPU's 1/k shard only, NCCL allgather.
  log_path(c, "allreduce", count * es, "nccl reduce-scatter + synthesis + nccl allgather");
  const Nccl* n = nccl();
  cemuShardPlan plan;
  cemuPlanShards(count, c->k, c->li, &plan);
  const size_t shard = plan.shardCount;
  const size_t rem = plan.tailCount;
  auto* r8 = static_cast<uint8_t*>(recv);
  const auto* s8 = static_cast<const uint8_t*>(send);
  const auto ndt = static_cast<ncclDataType_t>(dt);
  ph.push_back([=]() -> cemuResult_t {  // phase 0: the real part over NCCL
    CUDA_OK(call->stamp_now());
    if (shard) NCCL_OK(n->ReduceScatter(send, r8 + c->li * shard * es, shard, ndt, ncclSum, c->inner, s));
    if (rem) NCCL_OK(n->AllReduce(s8 + c->k * shard * es, r8 + c->k * shard * es, rem, ndt, ncclSum, c->inner, s));
    return cemuSuccess;
  });
  ph.push_back([=]() -> cemuResult_t {  // phase 1: the emulated part on the own shard
    if (shard) {
      CUDA_OK(synth_reduce(c, dt, r8 + c->li * shard * es, r8 + c->li * shard * es, shard, c->li * shard, nullptr,
                           s, &call->launches));
    }
    if (rem) {
      CUDA_OK(synth_reduce(c, dt, r8 + c->k * shard * es, r8 + c->k * shard * es, rem, c->k * shard, nullptr, s,
                           &call->launches));
    }
    return cemuSuccess;
  });
  ph.push_back([=]() -> cemuResult_t {  // phase 2: everyone's shards
    if (shard) NCCL_OK(n->AllGather(r8 + c->li * shard * es, r8, shard, ndt, c->inner, s));
    return cemuSuccess;
  });
  // phase 3: the delay, after the allgather (in a group NCCL launches it at
  // the phase's ncclGroupEnd, so it must not share a phase with our kernels)
  ph.push_back([=]() -> cemuResult_t {
    CUDA_OK(call->finish(kAllReduce));
    return cemuSuccess;
  });
  return cemuSuccess;
}

cemuResult_t do_allgather(const void* send, void* recv, size_t sc, int dt, cemuComm* c, cudaStream_t s,
                          Phases& ph) {
  const size_t es = dtype_size(dt);
  if (sc == 0) return cemuSuccess;
  auto call = std::make_shared<Call>(c, kAllGather, sc * es, s);
  if (!call->error.empty()) return fail(cemuInvalidArgument, call->error);
  auto* r8 = static_cast<uint8_t*>(recv);
  const uint32_t nvirt = static_cast<uint32_t>(c->virt.size());
  const bool own_in_place = send == r8 + static_cast<uint64_t>(c->rank) * sc * es;
  if (c->mode == PayloadMode::kZero) {
    ph.push_back([=]() -> cemuResult_t {
    // test_transport.cpp:169-182: own block kept, every other block zeros
    CUDA_OK(call->stamp_now());
    const uint64_t blk = sc * es;
    if (c->rank) CUDA_OK(cudaMemsetAsync(r8, 0, c->rank * blk, s));
    if (c->rank + 1 < c->W) CUDA_OK(cudaMemsetAsync(r8 + (c->rank + 1) * blk, 0, (c->W - c->rank - 1) * blk, s));
    if (!own_in_place) CUDA_OK(cudaMemcpyAsync(r8 + c->rank * blk, send, blk, cudaMemcpyDeviceToDevice, s));
    CUDA_OK(call->finish(kAllGather));
    return cemuSuccess;
    });
    return cemuSuccess;
  }
  if (c->k > 1 && c->fused && es <= 4) {
    // fused: push the own block to every real GPU over NVLink, synthesise the
    // emulated blocks locally -- one kernel
    const cemuComm::Region* rr = find_region(c, recv, sc * es * c->W);
    const uint64_t roff = rr ? static_cast<uint64_t>(r8 - rr->base) : 1;
    if (rr && roff % 16 == 0 && (sc * es) % 16 == 0) {  // symmetric conditions only
      log_path(c, "allgather", sc * es, "fused");
      ph.push_back([=]() -> cemuResult_t {
      const void* own_src = send;
      if (reinterpret_cast<uintptr_t>(send) % 16 != 0) {  // local: stage into the own block
        own_src = r8 + static_cast<uint64_t>(c->rank) * sc * es;
        if (own_src != send) CUDA_OK(cudaMemcpyAsync(const_cast<void*>(own_src), send, sc * es, cudaMemcpyDeviceToDevice, s));
      }
      FusedGatherArgs a;
      set_barrier(c, a);
      a.sig = op_sig(kAllGather, dt, sc, buf_tag(rr, roff));
      a.own = static_cast<const uint4*>(own_src);
      for (uint32_t g = 0; g < c->k; ++g) a.dst[g] = reinterpret_cast<uint4*>(rr->peer[g] + roff);
      a.own_block = c->rank;
      a.block_vecs = sc * es / 16;
      a.vranks = c->d_virt_ranks;
      a.vkeys = c->d_virt_keys;
      a.nvirt = nvirt;
      a.stamp = call->take_stamp();
      CUDA_OK(launch_fused_allgather(dt, a, s, &call->launches));
      CUDA_OK(call->finish(kAllGather));
      return cemuSuccess;
      });
      return cemuSuccess;
    }
  }
  log_path(c, "allgather", sc * es, c->k == 1 ? "synthesis" : "synthesis + nccl allgather");
  const void* own = (c->k == 1 && !own_in_place) ? send : nullptr;
  ph.push_back([=]() -> cemuResult_t {  // emulated blocks, written locally
    CUDA_OK(launch_synth_fill(dt, recv, sc, c->d_virt_ranks, c->d_virt_keys, nvirt, 0, 0, own, c->rank,
                              call->take_stamp(), s, &call->launches));
    if (c->k == 1) CUDA_OK(call->finish(kAllGather));
    return cemuSuccess;
  });
  if (c->k > 1) ph.push_back([=]() -> cemuResult_t {  // real blocks over NCCL
    const Nccl* n = nccl();
    const auto ndt = static_cast<ncclDataType_t>(dt);
    if (c->contiguous) {
      NCCL_OK(n->AllGather(send, r8 + static_cast<uint64_t>(c->real[0]) * sc * es, sc, ndt, c->inner, s));
    } else {
      NCCL_OK(n->GroupStart());
      for (uint32_t j = 0; j < c->k; ++j) {
        NCCL_OK(n->Broadcast(send, r8 + static_cast<uint64_t>(c->real[j]) * sc * es, sc, ndt,
                             static_cast<int>(j), c->inner, s));
      }
      NCCL_OK(n->GroupEnd());
    }
    return cemuSuccess;
  });
  if (c->k > 1) ph.push_back([=]() -> cemuResult_t {  // the delay, after the grouped NCCL launch
    CUDA_OK(call->finish(kAllGather));
    return cemuSuccess;
  });
  return cemuSuccess;
}

cemuResult_t do_reducescatter(const void* send, void* recv, size_t rc, int dt, cemuComm* c,
                              cudaStream_t s, Phases& ph) {
  const size_t es = dtype_size(dt);
  if (rc == 0) return cemuSuccess;
  auto call = std::make_shared<Call>(c, kReduceScatter, rc * es * c->W, s);
  if (!call->error.empty()) return fail(cemuInvalidArgument, call->error);
  const auto* s8 = static_cast<const uint8_t*>(send);
  const uint64_t mine = static_cast<uint64_t>(c->rank) * rc;
  if (c->mode == PayloadMode::kZero) {
    ph.push_back([=]() -> cemuResult_t {  // own contribution to chunk `rank` plus zero replies
      CUDA_OK(launch_synth_fill(dt, recv, rc, nullptr, nullptr, 0, 0, 0, s8 + mine * es, 0,
                                call->take_stamp(), s, &call->launches));
      CUDA_OK(call->finish(kReduceScatter));
      return cemuSuccess;
    });
    return cemuSuccess;
  }
  const uint32_t nk = static_cast<uint32_t>(c->virt.size());
  if (c->k == 1) {
    ph.push_back([=]() -> cemuResult_t {
      CUDA_OK(synth_reduce(c, dt, s8 + mine * es, recv, rc, mine,
                                  call->take_stamp(), s, &call->launches));
      CUDA_OK(call->finish(kReduceScatter));
      return cemuSuccess;
    });
    return cemuSuccess;
  }
  // fused: pull this rank's chunk from every real GPU's (symmetric) send over
  // NVLink, add the emulated ranks, write the local recv -- one kernel
  // The decision must be the same on every real rank (they meet in the
  // kernel's barriers), so it only looks at symmetric quantities: the send
  // region offset and the chunk size.  A misaligned local recv is served
  // through an aligned staging buffer instead of changing the decision.
  const cemuComm::Region* rs = c->fused ? find_region(c, send, rc * es * c->W) : nullptr;
  const uint64_t sbase = rs ? static_cast<uint64_t>(s8 - rs->base) : 1;
  if (rs && es <= 4 && nk > 0 && sbase % 16 == 0 && (rc * es) % 16 == 0) {
    log_path(c, "reduce-scatter", rc * es, "fused");
    ph.push_back([=]() -> cemuResult_t {
    const uint64_t soff = sbase + mine * es;
    void* out = recv;
    if (reinterpret_cast<uintptr_t>(recv) % 16 != 0) {
      if (auto r = ensure_scratch(c, rc * es)) return r;
      out = c->scratch;
    }
    FusedArgs a;
    set_barrier(c, a);
    a.sig = op_sig(kReduceScatter, dt, rc, buf_tag(rs, sbase));
    const uint64_t epv = 16 / es;
    a.ndst = 1;
    a.word_base = (dt == cemuInt32 || dt == cemuUint32) ? mine : mine / 4;
    a.v_begin = 0;
    a.v_end = rc / epv;
    a.ntail = static_cast<uint32_t>(rc - a.v_end * epv);
    a.tail_e0 = mine + a.v_end * epv;
    for (uint32_t g = 0; g < c->k; ++g) a.src[g] = reinterpret_cast<const uint4*>(rs->peer[g] + soff);
    a.dst[0] = static_cast<uint4*>(out);
    a.keys = c->d_virt_keys;
    a.nkeys = nk;
    a.stamp = call->take_stamp();
    CUDA_OK(cache_fused(c, dt, a, s, &call->launches));
    CUDA_OK(launch_fused_allreduce(dt, a, s, &call->launches));
    if (out != recv) CUDA_OK(cudaMemcpyAsync(recv, out, rc * es, cudaMemcpyDeviceToDevice, s));
    CUDA_OK(call->finish(kReduceScatter));
    return cemuSuccess;
    });
    return cemuSuccess;
  }
  log_path(c, "reduce-scatter", rc * es, "nccl reduce-scatter + synthesis");
  const Nccl* n = nccl();
  const auto ndt = static_cast<ncclDataType_t>(dt);
  ph.push_back([=]() -> cemuResult_t {  // phase 0: the real part over NCCL
  CUDA_OK(call->stamp_now());
  if (c->contiguous) {
    NCCL_OK(n->ReduceScatter(s8 + static_cast<uint64_t>(c->real[0]) * rc * es, recv, rc, ndt, ncclSum,
                             c->inner, s));
  } else {
    NCCL_OK(n->GroupStart());
    for (uint32_t j = 0; j < c->k; ++j) {
      NCCL_OK(n->Reduce(s8 + static_cast<uint64_t>(c->real[j]) * rc * es, recv, rc, ndt, ncclSum,
                        static_cast<int>(j), c->inner, s));
    }
    NCCL_OK(n->GroupEnd());
  }
  return cemuSuccess;
  });
  ph.push_back([=]() -> cemuResult_t {  // phase 1: the emulated part
    CUDA_OK(synth_reduce(c, dt, recv, recv, rc, mine, nullptr, s, &call->launches));
    CUDA_OK(call->finish(kReduceScatter));
    return cemuSuccess;
  });
  return cemuSuccess;
}

cemuResult_t do_broadcast(const void* send, void* recv, size_t count, int dt, int root, cemuComm* c,
                          cudaStream_t s, Phases& ph) {
  const size_t es = dtype_size(dt);
  if (root < 0 || static_cast<uint32_t>(root) >= c->W) {
    return fail(cemuInvalidArgument, "cemuBroadcast: root " + std::to_string(root) + " out of range [0," +
                                         std::to_string(c->W - 1) + "]");
  }
  if (count == 0) return cemuSuccess;
  auto call = std::make_shared<Call>(c, kBroadcast, count * es, s);
  if (!call->error.empty()) return fail(cemuInvalidArgument, call->error);
  const uint32_t r = static_cast<uint32_t>(root);
  ph.push_back([=]() -> cemuResult_t {
  if (c->cfg.is_real(r)) {
    if (c->k == 1) {
      if (send != recv) {
        CUDA_OK(launch_synth_fill(dt, recv, count, nullptr, nullptr, 0, 0, 0, send, 0, call->take_stamp(), s,
                                  &call->launches));
      }
    } else {
      CUDA_OK(call->stamp_now());
      const int lroot = static_cast<int>(std::find(c->real.begin(), c->real.end(), r) - c->real.begin());
      NCCL_OK(nccl()->Broadcast(send, recv, count, static_cast<ncclDataType_t>(dt), lroot, c->inner, s));
      return cemuSuccess;  // the delay in the next phase (after a grouped NCCL launch)
    }
  } else if (c->mode == PayloadMode::kZero) {
    CUDA_OK(call->stamp_now());
    CUDA_OK(cudaMemsetAsync(recv, 0, count * es, s));
  } else {
    CUDA_OK(launch_synth_fill(dt, recv, count, nullptr, nullptr, 1, 0, payload_key(c->seed, r), nullptr, 0,
                              call->take_stamp(), s, &call->launches));
  }
  CUDA_OK(call->finish(kBroadcast));
  return cemuSuccess;
  });
  if (c->cfg.is_real(r) && c->k > 1) ph.push_back([=]() -> cemuResult_t {
    CUDA_OK(call->finish(kBroadcast));
    return cemuSuccess;
  });
  return cemuSuccess;
}

// A collective is planned into phases (closures); nothing runs at planning
// time.  Alone, its phases run back to back.  In a group, cemuGroupEnd runs
// "rounds" -- the i-th call of every communicator -- phase by phase, each
// phase inside one NCCL group, so a single thread driving several devices
// (cemuCommInitAll) never blocks in a device's NCCL call while another
// device's matching call has not been issued.  Every phase re-selects its
// communicator's device.
// The call's first phase waits for the communicator's previous call when
// that was issued on another stream; a last phase of its own (after any
// grouped NCCL launch of the previous phase) records the order event.
template <typename F>
cemuResult_t run_or_defer(cemuComm* c, cudaStream_t s, F&& plan) {
  auto ops = std::make_shared<Phases>();
  if (auto r = plan(*ops)) return r;
  if (ops->empty()) return cemuSuccess;  // zero-size call: nothing enqueued
  ops->insert(ops->begin(), [c, s]() { return order_begin(c, s); });
  ops->push_back([c, s]() { return order_end(c, s); });
  Phases wrapped;
  int idx = 0;
  for (auto& f : *ops) {
    wrapped.push_back([c, f, idx]() -> cemuResult_t {
      if (cudaSetDevice(c->device) != cudaSuccess) return fail(cemuUnhandledCudaError, "cannot select device");
      // a launch reports cudaGetLastError(): drop an error some earlier,
      // unrelated runtime call left behind (e.g. a destroyed communicator's
      // IPC unmapping) so it cannot fail this call
      const cudaError_t pend = cudaGetLastError();
      if (pend && debug_level() >= 2) {
        std::fprintf(stderr, "cemu: stale error before phase %d: %s\n", idx, cudaGetErrorString(pend));
      }
      return f();
    });
    ++idx;
  }
  if (g_group_depth > 0) {
    g_group_ops.push_back(GroupOp{c, std::move(wrapped)});
    return cemuSuccess;
  }
  for (auto& f : wrapped) {
    if (auto r = f()) return r;
  }
  return cemuSuccess;
}

int64_t exchange_queue_gap_ns(cemuComm_t c, int64_t gap_ns) {
  const int64_t old = c->queue_gap_ns;
  c->queue_gap_ns = gap_ns;
  return old;
}

const int64_t* stream_release_end(cemuComm_t c, cudaStream_t s) {
  return (c && c->last_slot && c->last_stream == s) ? c->last_slot + 1 : nullptr;
}

}  // namespace cemu_b200

// =============================================================================
// C-ABI
// =============================================================================
extern "C" {

void cemuPlanShards(uint64_t count, uint32_t k, uint32_t li, cemuShardPlan* p) {
  // equal shards for NCCL reduce-scatter/allgather; the remainder (< k
  // elements) is all-reduced by NCCL and synthesised by every rank alike
  const uint64_t shard = k ? count / k : count;
  p->shardOffset = shard * li;
  p->shardCount = shard;
  p->tailOffset = shard * k;
  p->tailCount = count - shard * k;
}

cemuResult_t cemuGetVersion(int* version) {
  if (!version) return fail(cemuInvalidArgument, "cemuGetVersion: version is null");
  *version = CEMU_B200_VERSION;
  return cemuSuccess;
}

cemuResult_t cemuGetUniqueId(cemuUniqueId* uid) {
  if (!uid) return fail(cemuInvalidArgument, "cemuGetUniqueId: uniqueId is null");
  if (const Nccl* n = nccl()) {
    ncclUniqueId id;
    NCCL_OK(n->GetUniqueId(&id));
    std::memcpy(uid, &id, sizeof id);
    return cemuSuccess;
  }
  std::random_device rd;
  for (auto& b : uid->internal) b = static_cast<char>(rd());
  return cemuSuccess;
}

cemuResult_t cemuCommInitRankConfig(cemuComm_t* comm, const char* text, cemuUniqueId id, int rank,
                                    int device) {
  if (!text) return fail(cemuInvalidArgument, "cemuCommInitRankConfig: configText is null");
  try {
    return init_comm(comm, parse_job_config(text), id, rank, device);
  } catch (const ConfigError& e) {
    return fail(cemuInvalidArgument, e.what());
  } catch (const std::exception& e) {
    return fail(cemuInternalError, e.what());
  }
}

cemuResult_t cemuCommInitRank(cemuComm_t* comm, int nranks, cemuUniqueId id, int rank) {
  const char* path = std::getenv("CEMU_CONFIG");
  if (!path || !*path) {
    return fail(cemuInvalidUsage, "CEMU_CONFIG: must name the job config file");
  }
  try {
    JobConfig cfg = load_job_config(path);
    if (nranks != static_cast<int>(cfg.world_size)) {
      return fail(cemuInvalidArgument, "nranks " + std::to_string(nranks) +
                                           " does not match world_size " +
                                           std::to_string(cfg.world_size) + " of " + path);
    }
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(cemuUnhandledCudaError, "cudaGetDevice failed");
    return init_comm(comm, std::move(cfg), id, rank, dev);
  } catch (const ConfigError& e) {
    return fail(cemuInvalidArgument, e.what());
  } catch (const std::exception& e) {
    return fail(cemuInternalError, e.what());
  }
}

cemuResult_t cemuCommInitAll(cemuComm_t* comms, int ndev, const int* devlist) {
  const char* path = std::getenv("CEMU_CONFIG");
  if (!comms || ndev < 1) return fail(cemuInvalidArgument, "cemuCommInitAll: bad argument");
  if (!path || !*path) return fail(cemuInvalidUsage, "CEMU_CONFIG: must name the job config file");
  try {
    const JobConfig cfg = load_job_config(path);
    if (cfg.real_ranks.size() != static_cast<size_t>(ndev)) {
      return fail(cemuInvalidArgument, "cemuCommInitAll: " + std::to_string(ndev) + " devices but the job has " +
                                           std::to_string(cfg.real_ranks.size()) + " real ranks");
    }
    std::vector<ncclComm_t> inner(ndev, nullptr);
    if (ndev > 1) {
      const Nccl* n = nccl();
      if (!n || !n->CommInitAll) return fail(cemuSystemError, "cemuCommInitAll: libnccl.so.2 not loadable");
      NCCL_OK(n->CommInitAll(inner.data(), ndev, devlist));
    }
    cemuUniqueId id{};
    int i = 0;
    for (uint32_t r : cfg.real_ranks) {  // device i serves the i-th real rank
      const int dev = devlist ? devlist[i] : i;
      if (auto e = init_comm(&comms[i], cfg, id, static_cast<int>(r), dev, inner[i])) return e;
      ++i;
    }
    if (ndev > 1) {
      // Establish NCCL's connections now, inside one group: a single thread
      // later issuing each device's call in turn must never block in a
      // lazy connection handshake waiting for a device it has not reached.
      const Nccl* n = nccl();
      std::vector<float*> scratch(ndev, nullptr);
      for (int d = 0; d < ndev; ++d) {
        CUDA_OK(cudaSetDevice(comms[d]->device));
        CUDA_OK(cudaMalloc(&scratch[d], 64 * sizeof(float) * ndev));
      }
      for (int op = 0; op < 4; ++op) {
        NCCL_OK(n->GroupStart());
        for (int d = 0; d < ndev; ++d) {
          cudaSetDevice(comms[d]->device);
          float* b = scratch[d];
          switch (op) {
            case 0: NCCL_OK(n->AllReduce(b, b, 64, ncclFloat32, ncclSum, comms[d]->inner, nullptr)); break;
            case 1: NCCL_OK(n->ReduceScatter(b, b, 64, ncclFloat32, ncclSum, comms[d]->inner, nullptr)); break;
            case 2: NCCL_OK(n->AllGather(b, b, 64, ncclFloat32, comms[d]->inner, nullptr)); break;
            default: NCCL_OK(n->Broadcast(b, b, 64, ncclFloat32, 0, comms[d]->inner, nullptr)); break;
          }
        }
        NCCL_OK(n->GroupEnd());
      }
      for (int d = 0; d < ndev; ++d) {
        CUDA_OK(cudaSetDevice(comms[d]->device));
        CUDA_OK(cudaDeviceSynchronize());
        cudaFree(scratch[d]);
      }
    }
    return cemuSuccess;
  } catch (const ConfigError& e) {
    return fail(cemuInvalidArgument, e.what());
  }
}

cemuResult_t cemuCommDestroy(cemuComm_t c) {
  delete c;  // ~cemuComm releases everything (null is a no-op, as ncclCommDestroy(NULL))
  return cemuSuccess;
}

cemuResult_t cemuCommCount(const cemuComm_t c, int* count) {
  if (!c || !count) return fail(cemuInvalidArgument, "cemuCommCount: null argument");
  *count = static_cast<int>(c->W);
  return cemuSuccess;
}

cemuResult_t cemuCommUserRank(const cemuComm_t c, int* rank) {
  if (!c || !rank) return fail(cemuInvalidArgument, "cemuCommUserRank: null argument");
  *rank = static_cast<int>(c->rank);
  return cemuSuccess;
}

cemuResult_t cemuCommCuDevice(const cemuComm_t c, int* device) {
  if (!c || !device) return fail(cemuInvalidArgument, "cemuCommCuDevice: null argument");
  *device = c->device;
  return cemuSuccess;
}

const char* cemuGetErrorString(cemuResult_t r) {
  switch (r) {
    case cemuSuccess: return "no error";
    case cemuUnhandledCudaError: return "unhandled cuda error";
    case cemuSystemError: return "unhandled system error";
    case cemuInternalError: return "internal error";
    case cemuInvalidArgument: return "invalid argument";
    case cemuInvalidUsage: return "invalid usage";
    case cemuRemoteError: return "remote process exited or there was a network error";
    case cemuInProgress: return "operation in progress";
  }
  return "unknown result code";
}

const char* cemuGetLastError(cemuComm_t) { return g_last_error.c_str(); }

cemuResult_t cemuAllReduce(const void* send, void* recv, size_t count, cemuDataType_t dt, cemuRedOp_t op,
                           cemuComm_t c, cemuStream_t stream) {
  if (auto r = check_common(c, dt, "cemuAllReduce")) return r;
  if (auto r = check_op(op, "cemuAllReduce")) return r;
  if (count && (!send || !recv)) return fail(cemuInvalidArgument, "cemuAllReduce: null buffer");
  auto s = reinterpret_cast<cudaStream_t>(stream);
  if (c->wire) {
    if (g_group_depth > 0) return fail(cemuInvalidUsage, "wire mode: collectives cannot be grouped");
    const uint64_t b = static_cast<uint64_t>(count) * dtype_size(dt);
    return wire_call(c, kAllReduce, send, recv, b, b, static_cast<uint32_t>(dtype_size(dt)), s);
  }
  return run_or_defer(c, s, [=](Phases& ph) { return do_allreduce(send, recv, count, dt, c, s, ph); });
}


cemuResult_t cemuAllGather(const void* send, void* recv, size_t sc, cemuDataType_t dt, cemuComm_t c,
                           cemuStream_t stream) {
  if (auto r = check_common(c, dt, "cemuAllGather")) return r;
  if (sc && (!send || !recv)) return fail(cemuInvalidArgument, "cemuAllGather: null buffer");
  auto s = reinterpret_cast<cudaStream_t>(stream);
  if (c->wire) {
    if (g_group_depth > 0) return fail(cemuInvalidUsage, "wire mode: collectives cannot be grouped");
    const uint64_t b = static_cast<uint64_t>(sc) * dtype_size(dt);
    return wire_call(c, kAllGather, send, recv, b * c->W, b, static_cast<uint32_t>(dtype_size(dt)), s);
  }
  return run_or_defer(c, s, [=](Phases& ph) { return do_allgather(send, recv, sc, dt, c, s, ph); });
}

cemuResult_t cemuReduceScatter(const void* send, void* recv, size_t rc, cemuDataType_t dt, cemuRedOp_t op,
                               cemuComm_t c, cemuStream_t stream) {
  if (auto r = check_common(c, dt, "cemuReduceScatter")) return r;
  if (auto r = check_op(op, "cemuReduceScatter")) return r;
  if (rc && (!send || !recv)) return fail(cemuInvalidArgument, "cemuReduceScatter: null buffer");
  if (c->wire) return fail(cemuInvalidUsage, "wire mode: the CEMU protocol has allreduce and allgather only");
  auto s = reinterpret_cast<cudaStream_t>(stream);
  return run_or_defer(c, s, [=](Phases& ph) { return do_reducescatter(send, recv, rc, dt, c, s, ph); });
}

cemuResult_t cemuBroadcast(const void* send, void* recv, size_t count, cemuDataType_t dt, int root,
                           cemuComm_t c, cemuStream_t stream) {
  if (auto r = check_common(c, dt, "cemuBroadcast")) return r;
  if (count && !recv) return fail(cemuInvalidArgument, "cemuBroadcast: null recvbuff");
  if (c->wire) return fail(cemuInvalidUsage, "wire mode: the CEMU protocol has allreduce and allgather only");
  auto s = reinterpret_cast<cudaStream_t>(stream);
  return run_or_defer(c, s, [=](Phases& ph) { return do_broadcast(send, recv, count, dt, root, c, s, ph); });
}

cemuResult_t cemuGroupStart(void) {
  ++g_group_depth;
  return cemuSuccess;
}

cemuResult_t cemuGroupEnd(void) {
  if (g_group_depth == 0) return fail(cemuInvalidUsage, "cemuGroupEnd: not in a group");
  if (--g_group_depth > 0) return cemuSuccess;
  std::vector<GroupOp> ops;
  ops.swap(g_group_ops);
  // round r = the r-th call of every communicator, in issue order
  std::vector<std::vector<GroupOp*>> rounds;
  std::map<cemuComm*, size_t> calls_of;
  for (auto& op : ops) {
    const size_t r = calls_of[op.c]++;
    if (rounds.size() <= r) rounds.resize(r + 1);
    rounds[r].push_back(&op);
  }
  const Nccl* n = nccl();
  for (auto& round : rounds) {
    size_t nph = 0;
    for (auto* op : round) nph = std::max(nph, op->phases.size());
    for (size_t p = 0; p < nph; ++p) {
      if (n) n->GroupStart();
      cemuResult_t err = cemuSuccess;
      for (auto* op : round) {
        if (p < op->phases.size() && !err) err = op->phases[p]();
      }
      if (n && n->GroupEnd() != ncclSuccess && !err) err = fail(cemuInternalError, "ncclGroupEnd failed");
      if (err) return err;
    }
  }
  return cemuSuccess;
}

cemuResult_t cemuCommLastCallId(cemuComm_t c, uint64_t* id) {
  if (!c || !id) return fail(cemuInvalidArgument, "cemuCommLastCallId: null argument");
  if (c->calls == 0) return fail(cemuInvalidUsage, "cemuCommLastCallId: no call issued yet");
  *id = c->calls - 1;
  return cemuSuccess;
}

cemuResult_t cemuCommCallRecord(cemuComm_t c, uint64_t id, cemuCallRecord* rec, int64_t* floors,
                                int64_t* release, double* offsets, size_t cap) {
  if (!c || !rec) return fail(cemuInvalidArgument, "cemuCommCallRecord: null argument");
  const uint32_t i = static_cast<uint32_t>(id % cemuComm::kSlots);
  const auto& m = c->meta[i];
  if (m.call_id != id) {
    return fail(cemuInvalidArgument, "cemuCommCallRecord: call " + std::to_string(id) +
                                         " is no longer held (ring of " +
                                         std::to_string(cemuComm::kSlots) + ")");
  }
  std::memset(rec, 0, sizeof *rec);
  rec->call_id = id;
  rec->coll = m.coll;
  rec->delay_active = m.delay ? 1 : 0;
  rec->steps = m.k;
  rec->world = c->W;
  rec->model_bytes = m.bytes;
  rec->model_latency_us = m.latency;
  if (!m.delay) return cemuSuccess;
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(cemuUnhandledCudaError, "cudaSetDevice");
  std::vector<int64_t> h(slot_words(c->kmax));
  CUDA_OK(cudaMemcpy(h.data(), c->d_slots + i * slot_words(c->kmax), h.size() * 8, cudaMemcpyDeviceToHost));
  rec->t_start_ns = h[0];
  rec->t_end_ns = h[1];
  rec->device_latency_us = h[2];
  rec->t_origin_ns = h[4];
  rec->late_ns = h[5];
  rec->overshoot_ns = h[6];
  rec->stall_ns = h[3];
  const size_t n = std::min<size_t>(cap, m.k);
  if (floors) std::memcpy(floors, h.data() + kSlotHeader, n * 8);
  if (release) std::memcpy(release, h.data() + kSlotHeader + c->kmax, n * 8);
  if (offsets) std::memcpy(offsets, h.data() + kSlotHeader + 2 * c->kmax, n * 8);
  return cemuSuccess;
}

cemuResult_t cemuCommGetAsyncError(cemuComm_t c, cemuResult_t* err) {
  if (!c || !err) return fail(cemuInvalidArgument, "cemuCommGetAsyncError: null argument");
  *err = cemuSuccess;
  if (!c->sig) return cemuSuccess;
  uint32_t e = 0;
  cudaSetDevice(c->device);
  CUDA_OK(cudaMemcpy(&e, c->sig + 260, 4, cudaMemcpyDeviceToHost));
  if (e) {
    *err = cemuRemoteError;
    g_last_error = e == 1   ? "fused collective: a peer never started (start barrier timed out)"
                   : e == 2 ? "fused collective: a peer never finished (done barrier timed out)"
                            : "fused collective: real ranks disagree on the call (collective, dtype or count)";
  }
  return cemuSuccess;
}

cemuResult_t cemuCommModelLatencyUs(cemuComm_t c, int coll, uint64_t bytes, int64_t* out) {
  if (!c || !out || coll < 0 || coll > 3) return fail(cemuInvalidArgument, "cemuCommModelLatencyUs: bad argument");
  const uint32_t k = to_real_count(coll, c->W, c->real);
  if (c->delay_fn) {
    std::vector<double> offs(k, 0.0);
    if (const int rc = c->delay_fn(coll, c->W, bytes, k, offs.data(), c->delay_user)) {
      return fail(cemuInvalidArgument, "delay model plugin returned " + std::to_string(rc));
    }
    int64_t lat = 0;
    for (double o : offs) lat = std::max<int64_t>(lat, std::llround(o));
    *out = lat;
    return cemuSuccess;
  }
  *out = c->delay_active ? call_latency_us(c->delay, coll, c->W, bytes, k) : 0;
  return cemuSuccess;
}

cemuResult_t cemuCommSetDelayFootprint(cemuComm_t c, int ctas, size_t smem_bytes) {
  if (!c || ctas < 0 || ctas > 4096 || smem_bytes > 227 * 1024) {
    return fail(cemuInvalidArgument, "cemuCommSetDelayFootprint: ctas in [0, 4096], smem <= 227 KB");
  }
  c->hold_ctas = ctas;
  c->hold_smem = static_cast<int32_t>(smem_bytes);
  return cemuSuccess;
}

cemuResult_t cemuCommSetQueueChaining(cemuComm_t c, int64_t gap_us) {
  if (!c || gap_us < 0) return fail(cemuInvalidArgument, "cemuCommSetQueueChaining: bad argument");
  c->queue_gap_ns = gap_us * 1000;
  return cemuSuccess;
}

cemuResult_t cemuCommSetDelayModel(cemuComm_t c, cemuDelayModelFn fn, void* user) {
  if (!c) return fail(cemuInvalidArgument, "cemuCommSetDelayModel: comm is null");
  if (fn && !c->h_offsets) {
    if (cudaSetDevice(c->device) != cudaSuccess) return fail(cemuUnhandledCudaError, "cudaSetDevice");
    CUDA_OK(cudaMallocHost(&c->h_offsets, static_cast<size_t>(cemuComm::kSlots) * c->kmax * sizeof(double)));
  }
  c->delay_fn = fn;
  c->delay_user = user;
  c->delay_active = fn ? true : c->config_delay_active;
  return cemuSuccess;
}

// EventLog lines (trace.hpp:10-34: "<ts_us> <op_id> <event> <direction>
// <step> <chunk>") of one call, as the reference emulator would log them:
// register, the real node's from_real sends (an instantaneous real node
// sends step p when step p-1's reply was released), every to_real release
// at its device %globaltimer instant, complete.  Chunks are given for a
// single real rank (ring schedule, dag.cpp:73-82), "-" otherwise.
int cemuCommEventLog(cemuComm_t c, uint64_t id, char* out, size_t cap) {
  cemuCallRecord rec;
  std::vector<int64_t> floors, rel;
  if (!c) return -1;
  const uint32_t i = static_cast<uint32_t>(id % cemuComm::kSlots);
  const uint32_t k = c->meta[i].k;
  floors.resize(k ? k : 1);
  rel.resize(k ? k : 1);
  if (cemuCommCallRecord(c, id, &rec, floors.data(), rel.data(), nullptr, k) != cemuSuccess) return -1;
  if (!rec.delay_active) return fail(cemuInvalidUsage, "cemuCommEventLog: call ran without the delay model"), -1;
  const bool single = c->k == 1;
  const int coll = rec.coll == kReduceScatter || rec.coll == kBroadcast ? -1 : rec.coll;
  const uint32_t W = c->W, R = c->rank, prev = (R + W - 1) % W;
  std::string s;
  char line[160];
  auto emit = [&](int64_t ns, const char* ev, const char* dir, int64_t step, int64_t chunk) {
    char st[24], ch[24];
    if (step >= 0) std::snprintf(st, sizeof st, "%lld", static_cast<long long>(step)); else std::snprintf(st, sizeof st, "-");
    if (chunk >= 0) std::snprintf(ch, sizeof ch, "%lld", static_cast<long long>(chunk)); else std::snprintf(ch, sizeof ch, "-");
    std::snprintf(line, sizeof line, "%lld %llu %s %s %s %s\n", static_cast<long long>(ns / 1000),
                  static_cast<unsigned long long>(id), ev, dir, st, ch);
    s += line;
  };
  emit(rec.t_start_ns, "register", "-", -1, -1);
  for (uint32_t j = 0; j < k; ++j) {
    // the real node's send of step j (forwarding what arrived at step j-1)
    const int64_t t_fr = j == 0 ? rec.t_start_ns : rel[j - 1];
    emit(t_fr, "recv", "from_real", j, single && coll >= 0 ? send_chunk_at(coll, W, R, j) : -1);
    emit(rel[j], "send", "to_real", j, single && coll >= 0 ? send_chunk_at(coll, W, prev, j) : -1);
  }
  emit(rec.t_end_ns, "complete", "-", -1, -1);
  if (!out || s.size() + 1 > cap) return -static_cast<int>(s.size() + 1);
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

}  // extern "C"

// launch counter for bench.py's gpu_launches (not part of the public header)

extern "C" uint64_t cemuCommKernelLaunches(cemuComm_t c) { return c ? c->launches : 0; }

extern "C" cemuResult_t cemuCommLastReleaseEnd(cemuComm_t c, const int64_t** out) {
  if (!c || !out) return cemuInvalidArgument;
  *out = c->last_slot ? c->last_slot + 1 : nullptr;
  return cemuSuccess;
}
