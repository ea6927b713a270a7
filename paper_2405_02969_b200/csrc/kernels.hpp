// kernels.hpp -- launch API of the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cemu_b200.h"

namespace cemu_b200 {

// Per-call record slot in device memory (int64 words):
//   [0] t_start_ns (the call's first kernel)  [1] t_end_ns  [2] device max
//   floor (us)  [3] K  [4] schedule origin (= [0] unless queue-chained)
//   [5] late_ns: max over steps of release - (origin + floor)
//   [6] overshoot_ns: max(0, t_end - (origin + max floor))  [7] reserved
//   [8 .. 8+kmax)            floors_us[j]
//   [8+kmax .. 8+2kmax)      release_ns[j]   (%globaltimer at release)
//   [8+2kmax .. 8+3kmax)     offsets_us[j]   (double bits)
// Emulated peers one call can synthesise (the kernels' shared-memory key
// table: 8 B per peer, up to the 227 KB a block can opt into).
constexpr uint32_t kMaxEmulatedPeers = 28 * 1024;
constexpr int kSlotHeader = 8;
inline size_t slot_words(uint32_t kmax) { return kSlotHeader + 3 * static_cast<size_t>(kmax); }

struct DelayLaunch {
  cemuDelayModel model;
  int32_t coll;
  uint32_t n;
  uint64_t bytes;
  uint32_t k;
  uint32_t kmax;
  int32_t self_stamp;  // 1: this kernel records t_start itself
  int32_t preloaded;   // 1: the K offsets are already in the slot (a delay-model plugin's)
  // Back-to-back calls on one stream: the end time (slot[1]) of the previous
  // delayed call on this stream, or null.  A call whose start lies within
  // queue_gap_ns after it was queued behind that call, and its network time
  // starts at that end rather than after the emulator's own kernel-dispatch
  // gap (an in-order channel starts the next collective when the previous
  // one leaves the wire).
  const int64_t* prev_end;
  int64_t queue_gap_ns;
};
// The real collective's SM footprint for one call (cemuCommSetDelayFootprint):
// `ctas` CTAs of 544 threads with `smem` bytes each, from the first
// holder's start for lat_ns; `active` = busy-poll instead of sleeping.
// *start (a device word) is zeroed in stream order before the launch.
cudaError_t launch_footprint(unsigned long long* start, int64_t lat_ns, int ctas, int smem, int active,
                             cudaStream_t stream, int* launches);

// *chain = max(*chain, *other) in stream order (one 1-thread kernel).
cudaError_t launch_chain_join(int64_t* chain, const int64_t* other, cudaStream_t stream, int* launches);

// CEMU_QUEUE_GAP_US: the communicators' default queue-chaining gap
// (default 0 = off; cemuCommSetQueueChaining sets it per communicator)
int64_t queue_gap_ns();

// Synthesis cache (kernels.cu, "synthesis cache"): the emulated peers'
// contribution depends only on (seed, rank, element index), never on the
// call, so a communicator may keep it per element and fold repeat calls
// from it.  Entries, indexed by absolute payload element e:
//   kCacheLanes16  byte kinds (u8/i8/fp16/bf16/fp32), <= 256 peers: uint16
//                  t_e = sum over peers of byte_r(e)
//   kCacheWide32   byte kinds, > CEMU_SYNTH_CACHE_C16_MAX peers: uint32 t_e;
//                  32-bit integer kinds: uint32 wrapping sum of word_r(e)
//   kCacheCentered16  byte kinds, 257..CEMU_SYNTH_CACHE_C16_MAX (8192) peers:
//                  uint16 u_e = t_e - c16_offset(n) (mod 2^32) when it lies in
//                  [1, 65535], else 0 -- an escape: the fold recomputes t_e
//                  exactly from the keys.  t_e has mean 127.5 n and standard
//                  deviation 73.9 sqrt(n), so u_e is centred on 32768 and an
//                  escape needs a 6.9-sigma sum at n = 4096 (4.8 at 8192)
enum CacheKind { kNoCache = 0, kCacheLanes16 = 1, kCacheWide32 = 2, kCacheCentered16 = 3 };
// floor(127.5 n) - 32768 (mod 2^32): the centred entries' offset
inline constexpr uint32_t c16_offset(uint32_t n) { return n * 255u / 2u - 32768u; }
struct CacheRef {
  void* ptr = nullptr;  // entry 0 = payload element 0
  int kind = kNoCache;
  // centred entries: `clean` = the range is known to hold no escape (its
  // fill has completed and counted none), so the fold may skip the escape
  // test; `esc` = where a fill counts its escapes (mapped host memory)
  bool clean = false;
  uint32_t* esc = nullptr;
};
// Cache entries of one element range need this many bytes per element.
inline size_t cache_entry_bytes(int kind) { return kind == kCacheWide32 ? 4 : 2; }

// dst[i] = src[i] (+) sum over `nkeys` emulated peers of their payload at
// element elem_base + i.  src may equal dst.  Returns the number of kernel
// launches issued through *launches.  With a cache (whose entries cover
// [elem_base, elem_base + count)) the sums are read instead of synthesised:
// same bits.  Cached calls need 16-byte aligned src/dst and elem_base % 4 == 0.
cudaError_t launch_synth_reduce(int dtype, const void* src, void* dst, uint64_t count,
                                uint64_t elem_base, const uint32_t* d_keys, uint32_t nkeys,
                                int64_t* stamp, cudaStream_t stream, int* launches, CacheRef cache = {},
                                uint32_t grid_cap = 0);
// grid_cap > 0: at most that many CTAs (grid-stride) -- an emulated call
// with a delay footprint keeps its own memory work on about as many SMs as
// the real collective's kernel would use (cemuCommSetDelayFootprint).
// launch_synth_reduce that also writes the cache entries of
// [elem_base, elem_base + count) in the same pass (the first call over a
// range): <= 256 emulated peers for the byte kinds (uint16 entries) or the
// 32-bit integer kinds; a ragged tail's entries by a small fill.
cudaError_t launch_synth_reduce_filling(int dtype, const void* src, void* dst, uint64_t count, uint64_t elem_base,
                                        const uint32_t* d_keys, uint32_t nkeys, int64_t* stamp, cudaStream_t stream,
                                        int* launches, CacheRef cache, uint32_t grid_cap = 0);
// Writes the cache entries of elements [elem_base, elem_base + count)
// (byte kinds: whole payload words, i.e. rounded out to multiples of 4).
// `words`: the 32-bit integer kinds' entries.
cudaError_t launch_synth_cache_fill(bool words, uint64_t elem_base, uint64_t count, const uint32_t* d_keys,
                                    uint32_t nkeys, CacheRef cache, cudaStream_t stream, int* launches);

// Writes whole per-rank blocks: for b in [0, nblocks) block dst_index[b]
// (elements [dst_index[b]*block_elems, +block_elems) of dst) is filled with
// the payload of key[b]; if own_src != nullptr, block own_index is copied
// from own_src.  d_index/d_keys may be null when nblocks == 1, then
// index0/key0 are used.  Payload element indices start at elem_base (the
// block holds elements [elem_base, elem_base + block_elems) of the rank's
// payload; one block per launch then).
cudaError_t launch_synth_fill(int dtype, void* dst, uint64_t block_elems,
                              const uint32_t* d_index, const uint32_t* d_keys, uint32_t nblocks,
                              uint32_t index0, uint32_t key0, const void* own_src,
                              uint32_t own_index, int64_t* stamp, cudaStream_t stream,
                              int* launches, uint64_t elem_base = 0);

// One-kernel multi-GPU allreduce over peer memory (see kernels.cu).
constexpr int kMaxReal = 8;
struct FusedArgs {
  const uint4* src[kMaxReal];  // real GPUs' send buffers, ascending real rank (own = local)
  uint4* dst[kMaxReal];        // real GPUs' recv buffers
  int k = 0, me = 0;
  int ndst = 0;                     // k (allreduce: push to every GPU) or 1 (reduce-scatter)
  uint64_t word_base = 0;           // payload word of vector 0 (reduce-scatter: own chunk)
  uint64_t v_begin = 0, v_end = 0;  // 16-byte vectors this GPU reduces
  uint32_t ntail = 0;               // ragged elements after the last vector (last GPU only)
  uint64_t tail_e0 = 0;
  const uint32_t* keys = nullptr;   // emulated ranks' payload keys
  uint32_t nkeys = 0;
  uint64_t* flags = nullptr;        // local signals: [0,8) start, [8,16) done
  uint64_t* peer_flags[kMaxReal];   // every real GPU's signal area (own = local)
  uint32_t* counter = nullptr;      // local CTA-completion counter
  uint32_t* error = nullptr;        // set on barrier timeout
  uint64_t* epoch = nullptr;       // local device counter: this call is *epoch + 1 (graph-replay safe)
  uint32_t sig = 0;                 // op signature (coll, dtype, count): must agree across ranks
  int64_t* stamp = nullptr;
  int64_t timeout_ns = 0;
  // 0: fold only -- no start / done barrier, epoch untouched (one chunk of
  // the copy-engine pipeline, whose barriers are launch_peer_barrier's)
  int barriers = 1;
  // synthesis cache covering this GPU's slice (and tail), or none
  const void* cache = nullptr;
  int cache_kind = kNoCache;
  bool cache_clean = false;  // centred entries without escapes (CacheRef::clean)
  // fold-only chunks: when *gate != 0 (the start barrier failed) only
  // dst[me] (local) is written
  const uint32_t* gate = nullptr;
};
// Returns cudaErrorNotSupported for datatypes without a vector path.
cudaError_t launch_fused_allreduce(int dtype, const FusedArgs& a, cudaStream_t stream, int* launches);
// The fused kernel's start (phase 0: announce + wait, stamps a.stamp) or
// done (phase 1: announce + wait, then the epoch advances) barrier alone, as
// a one-warp kernel: brackets a copy-engine allreduce.
cudaError_t launch_peer_barrier(const FusedArgs& a, int phase, cudaStream_t stream, int* launches);


// One-kernel multi-GPU allgather: push the own block to every real GPU over
// NVLink while the same launch synthesises the emulated blocks locally.
struct FusedGatherArgs {
  const uint4* own = nullptr;   // local send block
  uint4* dst[kMaxReal];         // every real GPU's recv buffer (own = local)
  int k = 0, me = 0;
  uint32_t own_block = 0;       // world rank of this GPU
  uint64_t block_vecs = 0;      // 16-byte vectors per block
  const uint32_t* vranks = nullptr;  // emulated ranks (block indices) and keys
  const uint32_t* vkeys = nullptr;
  uint32_t nvirt = 0;
  uint64_t* flags = nullptr;
  uint64_t* peer_flags[kMaxReal];
  uint32_t* counter = nullptr;
  uint32_t* error = nullptr;
  uint64_t* epoch = nullptr;       // local device counter: this call is *epoch + 1 (graph-replay safe)
  uint32_t sig = 0;
  int64_t* stamp = nullptr;
  int64_t timeout_ns = 0;
};
cudaError_t launch_fused_allgather(int dtype, const FusedGatherArgs& a, cudaStream_t stream, int* launches);

// wire mode: dst += src as int32 lanes (words) or bytes, wrapping
cudaError_t launch_wire_fold(void* dst, const void* src, uint64_t bytes, bool words, cudaStream_t stream,
                             int* launches);
cudaError_t launch_stamp(int64_t* slot, cudaStream_t stream, int* launches);
// chain: device int64 holding the previous spin's absolute deadline (or null)
cudaError_t launch_spin_ns(int64_t ns, cudaStream_t stream, int* launches, int64_t* chain = nullptr,
                           bool resync = false);
// A delay-model plugin's offsets passed by value in the launch (16 KB of
// the 32 KB kernel-parameter space): up to kInlineOffsets steps.
constexpr int kInlineOffsets = 2048;
struct InlineOffsets {
  double us[kInlineOffsets];
};
cudaError_t launch_delay_spin(const DelayLaunch& d, int64_t* slot, cudaStream_t stream,
                              int* launches, const InlineOffsets* offs = nullptr);
cudaError_t preload_delay_kernels();

}  // namespace cemu_b200
