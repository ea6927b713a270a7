// comm_internal.hpp -- what the communicator's translation units share
// (comm.cpp: lifecycle, collective bodies, the C-ABI; symmetric.cpp:
// symmetric memory and registration; synth_cache.cpp: the synthesis cache;
// host_pipe.cpp: the host-buffer pipeline; comm_wire.cpp: wire mode).  Not
// part of the C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "cemu_b200.h"
#include "config.hpp"
#include "delay_math.cuh"
#include "kernels.hpp"
#include "payload.cuh"
#include "schedule.hpp"
#include "wire.hpp"

namespace cemu_b200 {

// cemuGetLastError's text: the last failure on this thread
extern thread_local std::string g_last_error;
cemuResult_t fail(cemuResult_t code, const std::string& msg);

// ---- NCCL, loaded on demand (only jobs with several real GPUs need it) ----
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int,
                         ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
const Nccl* nccl();

size_t dtype_size(int dt);

// Deferred calls between cemuGroupStart/End (NCCL group semantics: nothing
// needs to start before ncclGroupEnd).  The composite ops chain NCCL calls
// with our kernels, so they are replayed in order at GroupEnd.
using Phases = std::vector<std::function<cemuResult_t()>>;
struct GroupOp {
  cemuComm* c;
  Phases phases;
};
extern thread_local int g_group_depth;
extern thread_local std::vector<GroupOp> g_group_ops;

}  // namespace cemu_b200

// The communicator is the C-ABI's opaque cemuComm (a global name); its
// members use the library's types.  This header is private to the three
// communicator translation units.
using namespace cemu_b200;

struct cemuComm {
  JobConfig cfg;
  uint32_t W = 0, rank = 0;
  int device = 0;
  std::vector<uint32_t> real;  // ascending world ranks of the real GPUs
  uint32_t k = 1, li = 0;      // number of real ranks, my index among them
  bool contiguous = true;      // real ranks form one block [real[0], real[0]+k)
  cemuDelayModel delay{};
  bool delay_active = false;
  // delay-model plugin (cemuCommSetDelayModel): offsets per call from the
  // user's function, staged through pinned memory into the record slot
  cemuDelayModelFn delay_fn = nullptr;
  void* delay_user = nullptr;
  bool config_delay_active = false;
  double* h_offsets = nullptr;            // pinned, kSlots x kmax
  cudaEvent_t offsets_copied[64] = {};    // per slot: the staging may be rewritten
  uint64_t seed = 1;
  PayloadMode mode = PayloadMode::kHash;
  std::vector<uint32_t> virt;  // emulated ranks, ascending
  uint32_t* d_virt_keys = nullptr;
  uint32_t* d_virt_ranks = nullptr;
  // per-call record ring
  static constexpr uint32_t kSlots = 64;
  uint32_t kmax = 1;
  int64_t* d_slots = nullptr;
  struct Meta {
    uint64_t call_id = ~0ull;
    int32_t coll = 0;
    bool delay = false;
    uint32_t k = 0;
    uint64_t bytes = 0;
    int64_t latency = 0;
  } meta[kSlots];
  uint64_t calls = 0;
  // the previous delayed call's record slot and stream: a call queued right
  // behind it on the same stream starts when it ended (queue_gap_ns())
  int64_t* last_slot = nullptr;
  cudaStream_t last_stream = nullptr;
  int64_t queue_gap_ns = 0;  // cemuCommSetQueueChaining (0: every call's schedule starts at its own start)
  int32_t hold_ctas = 0, hold_smem = 0, hold_active = 0;  // cemuCommSetDelayFootprint
  // the footprint's side stream, forked from the call's stream at its start
  // and joined back at its end
  cudaStream_t hold_stream = nullptr;
  cudaEvent_t hold_fork = nullptr, hold_join = nullptr;
  ncclComm_t inner = nullptr;
  uint64_t launches = 0;
  // fused multi-GPU path (k > 1): IPC-mapped signal areas and symmetric buffers
  uint8_t* sig = nullptr;  // local: flags[16] u64 | counter u32 @256 | error u32 @260 | epoch u64 @264
  uint8_t* peer_sig[kMaxReal] = {};       // every real GPU's area (own = sig)
  bool fused = true;
  int64_t fused_timeout_ns = 30'000'000'000LL;
  // A symmetric range: mapped on every real GPU, so fused kernels reach the
  // peers' copies over NVLink.  cemuMemAlloc allocations (owned), the host
  // pipe's buffers (owned) and caller memory registered with
  // cemuCommRegister (ncclCommRegister / ncclCommWindowRegister; not owned).
  struct Region {
    uint8_t* base = nullptr;
    size_t bytes = 0;
    uint8_t* peer[kMaxReal] = {};      // every real GPU's copy of `base` (own = base)
    uint8_t* peer_map[kMaxReal] = {};  // the IPC mapping each peer[g] lies in (closed on release)
    bool owned = true;                 // base is a cudaMalloc of this communicator
    uint64_t id = 0;                   // registration handle (cemuCommRegister)
  };
  std::vector<Region> regions;
  uint64_t next_region_id = 1;
  // IPC mappings opened in this process, shared by every region inside the
  // same peer allocation (a handle is opened once): key = peer index + handle
  struct IpcMap {
    void* ptr = nullptr;
    int refs = 0;
  };
  std::map<std::string, IpcMap> ipc_maps;
  void* scratch = nullptr;  // aligned staging for misaligned local outputs
  size_t scratch_bytes = 0;
  // Device buffers superseded by a larger one (scratch, copy-engine
  // staging).  An enqueued call -- or a captured graph -- may still use them,
  // so they are released only when the communicator is destroyed, never by
  // a device-wide synchronize on the enqueue path.
  std::vector<void*> retired;
  // Per-communicator call order across streams (NCCL's semantics; the
  // reference runs a session's ops strictly in order, one in flight:
  // collective.hpp:43-47, collective.cpp:357-404).  Every call records
  // order_ev on its stream when it is enqueued; a call on another stream
  // first waits for it.  Fused multi-GPU kernels spin on peer flags, so two
  // of them in flight at once would share the signal area's epoch and CTA
  // counter -- and could deadlock on SM occupancy -- without this.
  // Synthesis cache (kernels.hpp CacheRef): the emulated
  // peers' per-element sums, written by the first call over an element
  // range and folded from by every later call within it.  One cache for the
  // byte kinds (u8/i8/fp16/bf16/fp32 share byte_r(e)), one for the 32-bit
  // integer kinds; each a list of segments sized to exactly the ranges seen
  // (a reduce-scatter chunk at a high rank costs its own size, not its
  // offset).  Nothing is allocated or filled inside a stream capture.
  struct SynthCache {
    struct Segment {
      uint64_t b, e;  // element range [b, e) whose entries it holds
      void* ptr;
      size_t bytes;
      bool captured;  // a captured graph reads it: never reused, only retired
      // centred entries (kCacheCentered16): the fill's escape count (mapped
      // host memory), the event after the fill, and once that event has
      // completed whether the range holds escapes (-1 = not known yet)
      uint32_t* esc_h = nullptr;
      uint32_t* esc_d = nullptr;
      cudaEvent_t filled = nullptr;
      int esc_state = -1;
    };
    std::vector<Segment> segs;
    std::vector<std::pair<void*, size_t>> spare;  // dropped, never-captured segments: reusable
    size_t bytes = 0;
    int kind = kNoCache;
  };
  SynthCache cache_bytes, cache_words;
  // escape counters of the centred segments: blocks of 1024 mapped pinned
  // words, one word per segment ever created; and the segments' fill events
  std::vector<uint32_t*> esc_blocks;
  size_t esc_used = 0;
  std::vector<cudaEvent_t> seg_events;
  size_t cache_cap = 0;           // bytes per cache (CEMU_SYNTH_CACHE_MB; 0 = off)
  uint32_t cache_min_peers = 16;  // CEMU_SYNTH_CACHE_MIN_PEERS
  uint64_t cache_fills = 0, cache_hits = 0;
  cudaEvent_t order_ev = nullptr;
  cudaStream_t order_stream = nullptr;
  bool order_recorded = false;
  unsigned long long order_capture = 0;  // capture id of the last record (0: recorded eagerly)
  // host-buffer collectives (cemuAllReduceHost / cemuAllGatherHost): chunks
  // ride a 3-stage pipeline -- H2D copy engine, synthesis kernel, D2H copy
  // engine -- over kPipeBufs rotating device buffers, so both PCIe
  // directions and the SMs work at once
  static constexpr int kPipeBufs = 4;
  struct HostPipe {
    bool ready = false;
    size_t chunk = 0;                 // bytes per chunk (multiple of 1 MiB)
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    cudaEvent_t start = nullptr;
    cudaEvent_t loaded[kPipeBufs] = {}, done[kPipeBufs] = {}, drained[kPipeBufs] = {};
    void* buf[kPipeBufs] = {};
    bool symmetric = false;            // k > 1: buffers are regions mapped on every real GPU
    uint8_t* peer[kPipeBufs][kMaxReal] = {};
  } pipe;
  // wire mode (cemuCommAttachEmulator): collectives travel the CEMU protocol
  // to a reference emulator instead of being synthesised
  std::unique_ptr<WireSession> wire;
  void* wire_buf = nullptr;  // device staging of one received DATA payload
  size_t wire_buf_bytes = 0;
  // copy-engine allreduce (k = 2, large symmetric buffers):
  // the NVLink legs ride the copy engines, the fold + synthesis the SMs
  int ce = 2;  // CEMU_CE: 0 off, 1 forced, 2 (default) auto -- see ce_allreduce_fits
  struct CePipe {
    static constexpr int kEvents = 2 * 64 + 2;
    cudaStream_t pull[kMaxReal] = {};  // per peer: its send chunks into this GPU's staging
    cudaEvent_t ev[kEvents] = {};
    void* stage = nullptr;
    size_t stage_bytes = 0;
  } cep;

  // Releases every resource held, in dependency order; also runs when
  // initialisation fails half way (init_comm owns the comm in a unique_ptr).
  ~cemuComm() {
    cudaSetDevice(device);
    wire.reset();  // BYE to the emulator
    auto& p = pipe;
    // every internal stream drains before any mapping is closed or memory freed
    for (cudaStream_t st : {p.h2d, p.comp, p.d2h, hold_stream}) {
      if (st) cudaStreamSynchronize(st);
    }
    for (cudaStream_t st : cep.pull) {
      if (st) cudaStreamSynchronize(st);
    }
    if (order_ev) cudaEventSynchronize(order_ev);
    for (int b = 0; b < kPipeBufs; ++b) {
      if (!p.symmetric && p.buf[b]) cudaFree(p.buf[b]);  // symmetric buffers are regions (below)
      for (cudaEvent_t ev : {p.loaded[b], p.done[b], p.drained[b]}) {
        if (ev) cudaEventDestroy(ev);
      }
    }
    if (p.start) cudaEventDestroy(p.start);
    for (cudaStream_t st : {p.h2d, p.comp, p.d2h}) {
      if (st) cudaStreamDestroy(st);
    }
    for (auto& r : regions) {
      if (r.owned) cudaFree(r.base);
    }
    for (auto& m : ipc_maps) {
      if (m.second.ptr) cudaIpcCloseMemHandle(m.second.ptr);
    }
    for (cudaStream_t st : cep.pull) {
      if (st) cudaStreamDestroy(st);
    }
    if (order_ev) cudaEventDestroy(order_ev);
    if (hold_stream) cudaStreamDestroy(hold_stream);
    for (cudaEvent_t ev : {hold_fork, hold_join}) {
      if (ev) cudaEventDestroy(ev);
    }
    for (void* r : retired) cudaFree(r);
    for (cudaEvent_t ev : seg_events) cudaEventDestroy(ev);
    for (uint32_t* b : esc_blocks) cudaFreeHost(b);
    for (const auto* sc : {&cache_bytes, &cache_words}) {
      for (const auto& g : sc->segs) cudaFree(g.ptr);
      for (const auto& g : sc->spare) cudaFree(g.first);
    }
    for (cudaEvent_t ev : cep.ev) {
      if (ev) cudaEventDestroy(ev);
    }
    cudaFree(cep.stage);
    cudaFree(sig);
    cudaFree(scratch);
    cudaFree(wire_buf);
    if (inner) {
      if (const Nccl* n = nccl()) n->CommDestroy(inner);
    }
    for (cudaEvent_t ev : offsets_copied) {
      if (ev) cudaEventDestroy(ev);
    }
    if (h_offsets) cudaFreeHost(h_offsets);
    cudaFree(d_virt_keys);
    cudaFree(d_virt_ranks);
    cudaFree(d_slots);
    cudaGetLastError();  // a destructor reports nothing: leave no stale error behind
  }
};

namespace cemu_b200 {

struct Call {
  cemuComm* c;
  int64_t* slot = nullptr;
  bool stamped = false;
  int launches = 0;
  cudaStream_t s;

  uint32_t i = 0;  // record slot of this call
  std::vector<double> plugin;  // a delay-model plugin's offsets for this call
  std::string error;           // set when the plugin failed: the call must not run

  Call(cemuComm* comm, int coll, uint64_t model_bytes, cudaStream_t stream) : c(comm), s(stream) {
    const uint64_t id = c->calls++;
    i = static_cast<uint32_t>(id % cemuComm::kSlots);
    auto& m = c->meta[i];
    m.call_id = id;
    m.coll = coll;
    m.delay = c->delay_active;
    m.k = to_real_count(coll, c->W, c->real);
    m.bytes = model_bytes;
    if (c->delay_fn) {
      // DelayModelFn(boundary, bytes) -> offsets (delay.hpp:52-55): the
      // boundary is closed-form here, so the plugin sees (coll, n, bytes, K)
      plugin.assign(m.k, 0.0);
      const int rc = c->delay_fn(coll, c->W, model_bytes, m.k, plugin.data(), c->delay_user);
      if (rc != 0) {
        error = "delay model plugin returned " + std::to_string(rc) + " for call " + std::to_string(id);
      }
      int64_t lat = 0;
      for (double o : plugin) lat = std::max<int64_t>(lat, std::llround(o));
      m.latency = lat;
    } else {
      m.latency = c->delay_active ? call_latency_us(c->delay, coll, c->W, model_bytes, m.k) : 0;
    }
    if (c->delay_active) slot = c->d_slots + i * slot_words(c->kmax);
  }
  // pointer the first kernel of the call writes t_start into (or null)
  int64_t* take_stamp() {
    if (!slot || stamped) return nullptr;
    stamped = true;
    footprint_err = begin_footprint();
    return slot;
  }
  cudaError_t stamp_now() {
    if (!slot || stamped) return cudaSuccess;
    stamped = true;
    if (const cudaError_t e = begin_footprint()) return e;
    return launch_stamp(slot, s, &launches);
  }
  // The real collective's SM footprint (cemuCommSetDelayFootprint): forked
  // from the call's stream as its first kernel is enqueued, joined at the end.
  bool footprint = false;
  cudaError_t footprint_err = cudaSuccess;
  cudaError_t begin_footprint() {
    if (footprint || !slot || c->hold_ctas <= 0 || c->meta[i].latency <= 0) return cudaSuccess;
    if (!c->hold_stream) {
      if (const cudaError_t e = cudaStreamCreateWithFlags(&c->hold_stream, cudaStreamNonBlocking)) return e;
    }
    for (cudaEvent_t* ev : {&c->hold_fork, &c->hold_join}) {
      if (!*ev) {
        if (const cudaError_t e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) return e;
      }
    }
    if (const cudaError_t e = cudaEventRecord(c->hold_fork, s)) return e;
    if (const cudaError_t e = cudaStreamWaitEvent(c->hold_stream, c->hold_fork, 0)) return e;
    footprint = true;
    return launch_footprint(reinterpret_cast<unsigned long long*>(slot + 7), c->meta[i].latency * 1000,
                            c->hold_ctas, c->hold_smem, c->hold_active, c->hold_stream, &launches);
  }
  cudaError_t finish(int coll) {
    if (slot && !stamped) {
      if (const cudaError_t e = begin_footprint()) return e;  // the spin kernel is the call's first
    }
    if (footprint_err) return footprint_err;
    c->launches += launches;
    if (!slot) {
      c->last_slot = nullptr;  // nothing to chain to / join with
      return cudaSuccess;
    }
    if (footprint) {  // the call ends when its footprint does too
      const cudaError_t e = launch_delay_and_join(coll);
      return e;
    }
    return launch_delay(coll);
  }
  cudaError_t launch_delay_and_join(int coll) {
    const cudaError_t e = launch_delay(coll);
    if (e) return e;
    if (const cudaError_t r = cudaEventRecord(c->hold_join, c->hold_stream)) return r;
    return cudaStreamWaitEvent(s, c->hold_join, 0);
  }
  cudaError_t launch_delay(int coll) {
    const auto& m = c->meta[i];
    DelayLaunch d;
    d.model = c->delay;
    d.coll = coll;
    d.n = c->W;
    d.bytes = m.bytes;
    d.k = m.k;
    d.kmax = c->kmax;
    d.self_stamp = stamped ? 0 : 1;
    d.preloaded = 0;
    d.prev_end = (c->last_slot && c->last_stream == s) ? c->last_slot + 1 : nullptr;
    d.queue_gap_ns = c->queue_gap_ns;
    if (!plugin.empty() && plugin.size() <= static_cast<size_t>(kInlineOffsets)) {
      // the offsets ride in the spin kernel's parameter block: nothing on
      // the host to recycle, no host wait, graph-capture safe
      auto offs = std::make_unique<InlineOffsets>();
      std::memcpy(offs->us, plugin.data(), plugin.size() * sizeof(double));
      int l = 0;
      const cudaError_t e = launch_delay_spin(d, slot, s, &l, offs.get());
      c->launches += l;
      c->last_slot = slot;
      c->last_stream = s;
      return e;
    }
    if (!plugin.empty()) {
      // larger worlds: stage the plugin's offsets into the slot's offsets
      // region, in stream order; the pinned staging of slot i is reused 64
      // calls later (its previous copy has long completed in practice)
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      if (const cudaError_t e = cudaStreamIsCapturing(s, &cap)) return e;
      if (cap != cudaStreamCaptureStatusNone) return cudaErrorStreamCaptureUnsupported;  // > 2048 steps
      cudaEvent_t& ev = c->offsets_copied[i];
      if (!ev) {
        if (const cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) return e;
      } else if (const cudaError_t e = cudaEventSynchronize(ev)) {
        return e;
      }
      double* h = c->h_offsets + static_cast<size_t>(i) * c->kmax;
      std::memcpy(h, plugin.data(), plugin.size() * sizeof(double));
      auto* dev_offs = reinterpret_cast<double*>(slot + kSlotHeader + 2 * static_cast<size_t>(c->kmax));
      if (const cudaError_t e = cudaMemcpyAsync(dev_offs, h, plugin.size() * sizeof(double),
                                                cudaMemcpyHostToDevice, s)) {
        return e;
      }
      if (const cudaError_t e = cudaEventRecord(ev, s)) return e;
      d.preloaded = 1;
    }
    int l = 0;
    const cudaError_t e = launch_delay_spin(d, slot, s, &l);
    c->launches += l;
    c->last_slot = slot;
    c->last_stream = s;
    return e;
  }
};

#define CUDA_OK(expr)                                                                   \
  do {                                                                                  \
    const cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess)                                                              \
      return fail(cemuUnhandledCudaError, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define NCCL_OK(expr)                                                                       \
  do {                                                                                      \
    const ncclResult_t r_ = (expr);                                                         \
    if (r_ != ncclSuccess)                                                                  \
      return fail(static_cast<cemuResult_t>(r_),                                            \
                  std::string(#expr) + ": " +                                               \
                      (nccl()->GetErrorString ? nccl()->GetErrorString(r_) : "nccl error")); \
  } while (0)

// ---- shared helpers (comm.cpp) ----
// Maps every real GPU's allocation `local` (collectively) into this process.
cemuResult_t map_peers(cemuComm* c, void* local, size_t bytes, uint8_t** peers, uint8_t** peer_maps = nullptr);
// Drops the region's peer mappings (every real rank collectively: no peer
// still maps this GPU's memory when the call returns).
void unmap_region(cemuComm* c, cemuComm::Region& r);
cemuResult_t ensure_scratch(cemuComm* c, size_t bytes);
// True while `s` is being captured into a CUDA graph.
bool capturing(cudaStream_t s);
// All-gather `rec` (bytes each) among the k real GPUs over the inner NCCL
// comm; synchronous -- setup and registration only (symmetric.cpp).
cudaError_t exchange_records(cemuComm* c, const void* rec, size_t bytes, std::vector<uint8_t>* all, ncclResult_t* nr);
// Grows *buf to >= bytes; the superseded buffer goes to c->retired.
cemuResult_t grow_buffer(cemuComm* c, void** buf, size_t* have, size_t bytes, const char* what);
// Call order across streams (see cemuComm::order_ev): before the call's
// first enqueue / after its last one, on the call's stream.
cemuResult_t order_begin(cemuComm* c, cudaStream_t s);
cemuResult_t order_end(cemuComm* c, cudaStream_t s);
// 20-bit signature of a fused call; every real rank must compute the same
// `bufs`: the symmetric buffers' identity (region id, offset) -- ranks that
// pass different buffers disagree too, and must abort before any transfer
uint32_t op_sig(int coll, int dt, uint64_t count, uint64_t bufs = 0);
uint64_t buf_tag(const cemuComm::Region* r, uint64_t off);
const cemuComm::Region* find_region(const cemuComm* c, const void* p, size_t bytes);
cemuResult_t check_common(cemuComm* c, int dt, const char* what);
cemuResult_t check_op(int op, const char* what);
FusedArgs fused_allreduce_args(const cemuComm* c, int dt, uint64_t count, uint64_t e0, uint8_t* const* src,
                               uint8_t* const* dst);
cemuResult_t do_allreduce(const void* send, void* recv, size_t count, int dt, cemuComm* c, cudaStream_t s,
                          Phases& ph);
cemuResult_t do_allgather(const void* send, void* recv, size_t sc, int dt, cemuComm* c, cudaStream_t s,
                          Phases& ph);

template <typename A>
void set_barrier(cemuComm* c, A& a) {
  for (uint32_t g = 0; g < c->k; ++g) a.peer_flags[g] = reinterpret_cast<uint64_t*>(c->peer_sig[g]);
  a.k = static_cast<int>(c->k);
  a.me = static_cast<int>(c->li);
  a.flags = reinterpret_cast<uint64_t*>(c->sig);
  a.counter = reinterpret_cast<uint32_t*>(c->sig + 256);
  a.error = reinterpret_cast<uint32_t*>(c->sig + 260);
  a.epoch = reinterpret_cast<uint64_t*>(c->sig + 264);
  a.timeout_ns = c->fused_timeout_ns;
}

// Synthesis through the cache where it applies (else plain synthesis):
// launch_synth_reduce's arguments; fills the cache first on a miss.
cudaError_t synth_reduce(cemuComm* c, int dt, const void* src, void* dst, uint64_t count, uint64_t e0,
                         int64_t* stamp, cudaStream_t s, int* launches);
// The fused kernel's slice through the cache (sets a.cache / a.cache_kind,
// launches the fill on a miss).
cudaError_t cache_fused(cemuComm* c, int dt, FusedArgs& a, cudaStream_t s, int* launches);

// ---- host_pipe.cpp ----
cemuResult_t host_allreduce(const void* send, void* recv, size_t count, int dt, cemuComm* c, cudaStream_t s);
cemuResult_t host_allgather(const void* send, void* recv, size_t sc, int dt, cemuComm* c, cudaStream_t s);

// ---- comm_wire.cpp ----
cemuResult_t wire_call(cemuComm* c, int coll, const void* send, void* recv, uint64_t buf_bytes,
                       uint64_t model_bytes, uint32_t es, cudaStream_t s);

}  // namespace cemu_b200
