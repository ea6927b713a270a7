// synth_cache.cpp -- the synthesis cache: per element range,
// the emulated ranks' sums, written by the first call over the range and
// folded from by every later call within it.
#include "comm_internal.hpp"

namespace cemu_b200 {

// ---- synthesis cache ----------------------------------------------------
namespace {
bool cacheable_dtype(int dt) {
  return dt == cemuFloat32 || dt == cemuBfloat16 || dt == cemuFloat16 || dt == cemuUint8 || dt == cemuInt8 ||
         dt == cemuInt32 || dt == cemuUint32;
}

// The cache to use for elements [b, e) of dtype dt, or none.  *fill: the
// entries must be written first (this call's own pass fills them).
CacheRef cache_for(cemuComm* c, int dt, uint64_t b, uint64_t e, cudaStream_t s, bool* fill) {
  *fill = false;
  if (c->mode != PayloadMode::kHash || c->cache_cap == 0 || c->virt.size() < c->cache_min_peers ||
      !cacheable_dtype(dt) || b % 4 != 0 || e <= b) {
    return {};
  }
  // small calls are launch-bound either way: not worth an entry -- unless
  // the world makes even a small range's synthesis long (>= 2^27 peer-
  // elements: e.g. a 1024-rank FSDP reduce-scatter chunk of ~0.4 MB)
  const uint64_t bytes = (e - b) * dtype_size(dt);
  const bool heavy = (e - b) * static_cast<uint64_t>(c->virt.size()) >= (1ull << 27) && bytes >= (64u << 10);
  if (bytes < (1u << 20) && !heavy) return {};
  const bool words = dt == cemuInt32 || dt == cemuUint32;
  auto& sc = words ? c->cache_words : c->cache_bytes;
  if (sc.kind == kNoCache) sc.kind = (words || c->virt.size() > 256) ? kCacheWide32 : kCacheLanes16;
  const size_t entry = cache_entry_bytes(sc.kind);
  const uint64_t end = words ? e : (e + 3) / 4 * 4;  // the fill writes whole payload words
  // entry 0 of the returned pointer is element 0's: a segment's base moved
  // back by its first element (only indices inside the segment are read)
  auto ref = [&](const cemuComm::SynthCache::Segment& g) {
    return CacheRef{reinterpret_cast<void*>(reinterpret_cast<uintptr_t>(g.ptr) - g.b * entry), sc.kind};
  };
  const bool cap = capturing(s);
  for (auto& g : sc.segs) {
    if (g.b <= b && end <= g.e) {  // written by an earlier call, which every later call is ordered after
      g.captured |= cap;
      ++c->cache_hits;
      return ref(g);
    }
  }
  // a new segment holding exactly this range's entries
  const size_t need = (end - b) * entry;
  if (cap || sc.bytes + need > c->cache_cap) return {};  // no allocation / fill in a capture
  void* p = nullptr;
  size_t have = need;
  // a dropped segment no captured graph reads is free once the calls before
  // this one are done -- and this call is ordered after all of them
  auto best = sc.spare.end();
  for (auto it = sc.spare.begin(); it != sc.spare.end(); ++it) {
    if (it->second >= need && (best == sc.spare.end() || it->second < best->second)) best = it;
  }
  if (best != sc.spare.end()) {
    p = best->first;
    have = best->second;
    sc.spare.erase(best);
  } else if (cudaMalloc(&p, need) != cudaSuccess) {
    cudaGetLastError();
    return {};
  }
  sc.segs.push_back({b, end, p, have, false});
  sc.bytes += have;
  ++c->cache_fills;
  *fill = true;
  return ref(sc.segs.back());
}
}  // namespace

cudaError_t synth_reduce(cemuComm* c, int dt, const void* src, void* dst, uint64_t count, uint64_t e0,
                         int64_t* stamp, cudaStream_t s, int* launches) {
  const uint32_t nk = static_cast<uint32_t>(c->virt.size());
  const bool al = (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16 == 0;
  bool fill = false;
  const CacheRef cr = al ? cache_for(c, dt, e0, e0 + count, s, &fill) : CacheRef{};
  if (!cr.ptr) return launch_synth_reduce(dt, src, dst, count, e0, c->d_virt_keys, nk, stamp, s, launches);
  if (fill && (cr.kind == kCacheWide32) == (dt == cemuInt32 || dt == cemuUint32)) {
    // one pass synthesises, folds and writes the entries (+ the tail's)
    return launch_synth_reduce_filling(dt, src, dst, count, e0, c->d_virt_keys, nk, stamp, s, launches, cr);
  }
  if (fill) {  // > 256 emulated ranks of a byte kind: fill, then the cached fold
    if (stamp) {  // the call starts with the fill
      if (const cudaError_t e = launch_stamp(stamp, s, launches)) return e;
      stamp = nullptr;
    }
    const bool words = dt == cemuInt32 || dt == cemuUint32;
    if (const cudaError_t e = launch_synth_cache_fill(words, e0, count, c->d_virt_keys, nk, cr, s, launches)) return e;
  }
  return launch_synth_reduce(dt, src, dst, count, e0, c->d_virt_keys, nk, stamp, s, launches, cr);
}

cudaError_t cache_fused(cemuComm* c, int dt, FusedArgs& a, cudaStream_t s, int* launches) {
  const bool words = dt == cemuInt32 || dt == cemuUint32;
  const uint64_t epv = 16 / dtype_size(dt);
  auto elem_of = [&](uint64_t v) { return words ? a.word_base + v * 4 : (a.word_base + v * (epv / 4)) * 4; };
  const uint64_t b = elem_of(a.v_begin), e = elem_of(a.v_end) + a.ntail;
  bool fill = false;
  const CacheRef cr = cache_for(c, dt, b, e, s, &fill);
  if (!cr.ptr) return cudaSuccess;
  if (fill) {
    if (a.stamp) {
      if (const cudaError_t r = launch_stamp(a.stamp, s, launches)) return r;
      a.stamp = nullptr;
    }
    if (const cudaError_t r = launch_synth_cache_fill(words, b, e - b, a.keys, a.nkeys, cr, s, launches)) return r;
  }
  a.cache = cr.ptr;
  a.cache_kind = cr.kind;
  return cudaSuccess;
}

}  // namespace cemu_b200

extern "C" {

cemuResult_t cemuCommSetSynthCache(cemuComm_t c, size_t cap, uint32_t min_peers) {
  if (!c) return fail(cemuInvalidArgument, "cemuCommSetSynthCache: comm is null");
  if (min_peers == 0) return fail(cemuInvalidArgument, "cemuCommSetSynthCache: minPeers must be >= 1");
  c->cache_cap = cap;
  c->cache_min_peers = min_peers;
  for (auto* sc : {&c->cache_bytes, &c->cache_words}) {
    for (const auto& g : sc->segs) {
      if (g.captured) {
        c->retired.push_back(g.ptr);  // a captured graph may still read it
      } else {
        sc->spare.emplace_back(g.ptr, g.bytes);  // reusable by a later fill (calls are ordered)
      }
    }
    sc->segs.clear();
    sc->bytes = 0;
    if (cap == 0) {  // caching off: give the memory back once the calls that may read it are done
      if (c->order_ev) cudaEventSynchronize(c->order_ev);
      for (const auto& g : sc->spare) cudaFree(g.first);
      sc->spare.clear();
    }
  }
  return cemuSuccess;
}

cemuResult_t cemuCommSynthCacheStats(cemuComm_t c, uint64_t* fills, uint64_t* hits, size_t* bytes) {
  if (!c) return fail(cemuInvalidArgument, "cemuCommSynthCacheStats: comm is null");
  if (fills) *fills = c->cache_fills;
  if (hits) *hits = c->cache_hits;
  if (bytes) *bytes = c->cache_bytes.bytes + c->cache_words.bytes;
  return cemuSuccess;
}

}  // extern "C"
