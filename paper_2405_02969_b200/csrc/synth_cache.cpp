// synth_cache.cpp -- the synthesis cache: per element range,
// the emulated ranks' sums, written by the first call over the range and
// folded from by every later call within it.
#include "comm_internal.hpp"

namespace cemu_b200 {

// ---- synthesis cache ----------------------------------------------------
namespace {
// The largest emulated world cached with centred 16-bit entries
// (CEMU_SYNTH_CACHE_C16_MAX, default 8192: escapes need a 4.8-sigma byte sum
// there; beyond it uint32 entries).
uint32_t c16_max_peers() {
  static const uint32_t v = [] {
    const char* e = std::getenv("CEMU_SYNTH_CACHE_C16_MAX");
    return e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : 8192u;
  }();
  return v;
}

bool cacheable_dtype(int dt) {
  return dt == cemuFloat32 || dt == cemuBfloat16 || dt == cemuFloat16 || dt == cemuUint8 || dt == cemuInt8 ||
         dt == cemuInt32 || dt == cemuUint32;
}

// A centred segment's escape counter (zeroed) and fill event.
bool esc_slot(cemuComm* c, cemuComm::SynthCache::Segment* g) {
  constexpr size_t kBlock = 1024;
  if (c->esc_used % kBlock == 0) {
    void* blk = nullptr;
    if (cudaHostAlloc(&blk, kBlock * sizeof(uint32_t), cudaHostAllocMapped) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    c->esc_blocks.push_back(static_cast<uint32_t*>(blk));
  }
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  c->seg_events.push_back(ev);
  g->esc_h = c->esc_blocks.back() + c->esc_used++ % kBlock;
  *g->esc_h = 0;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, g->esc_h, 0) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  g->esc_d = static_cast<uint32_t*>(d);
  g->filled = ev;
  return true;
}

// The fill event of the segment a fill just wrote (centred entries only).
void note_filled(cemuComm* c, const CacheRef& cr, cudaStream_t s) {
  if (cr.kind != kCacheCentered16) return;
  for (const auto& g : c->cache_bytes.segs) {
    if (g.esc_d == cr.esc && g.filled) {
      cudaEventRecord(g.filled, s);
      return;
    }
  }
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
  // the world makes even a small range's synthesis longer than the launch
  // (>= 2^21 peer-elements: at world 64 from 128 KiB of fp32, where the
  // synthesis alone took 2.3-2.9 us per call against ~1.6 us cached)
  const uint64_t bytes = (e - b) * dtype_size(dt);
  const bool heavy = (e - b) * static_cast<uint64_t>(c->virt.size()) >= (1ull << 21) && bytes >= (64u << 10);
  if (bytes < (1u << 20) && !heavy) return {};
  const bool words = dt == cemuInt32 || dt == cemuUint32;
  auto& sc = words ? c->cache_words : c->cache_bytes;
  if (sc.kind == kNoCache) {
    const size_t n = c->virt.size();
    sc.kind = words ? kCacheWide32 : n <= 256 ? kCacheLanes16 : n <= c16_max_peers() ? kCacheCentered16 : kCacheWide32;
  }
  const size_t entry = cache_entry_bytes(sc.kind);
  const uint64_t end = words ? e : (e + 3) / 4 * 4;  // the fill writes whole payload words
  // entry 0 of the returned pointer is element 0's: a segment's base moved
  // back by its first element (only indices inside the segment are read)
  auto ref = [&](const cemuComm::SynthCache::Segment& g) {
    return CacheRef{reinterpret_cast<void*>(reinterpret_cast<uintptr_t>(g.ptr) - g.b * entry), sc.kind,
                    g.esc_state == 0, g.esc_d};
  };
  const bool cap = capturing(s);
  for (auto& g : sc.segs) {
    if (g.b <= b && end <= g.e) {  // written by an earlier call, which every later call is ordered after
      g.captured |= cap;
      ++c->cache_hits;
      // a centred range's escape count is known once its fill has run (no
      // wait: until then, and inside a capture, the fold tests for escapes)
      if (g.esc_state < 0 && g.filled && !cap && cudaEventQuery(g.filled) == cudaSuccess) {
        g.esc_state = *reinterpret_cast<volatile uint32_t*>(g.esc_h) != 0 ? 1 : 0;
      }
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
  cemuComm::SynthCache::Segment g{b, end, p, have, false};
  if (sc.kind == kCacheCentered16 && !esc_slot(c, &g)) {
    sc.spare.emplace_back(p, have);
    return {};
  }
  sc.segs.push_back(g);
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
  // a delay footprint stands for the real collective's kernel: the emulated
  // call's own memory pass -- a cached fold, or the synthesis of <= 16
  // emulated ranks, both HBM-bound like the real reduction -- stays within
  // as many CTAs instead of briefly taking every SM from the job's compute
  // (DESIGN §6c).  Issue-bound synthesis (more ranks, a cache fill) keeps
  // the whole machine: on a few CTAs it would outlast the modelled delay.
  const uint32_t fp = (c->hold_ctas > 0 && (c->delay_active || c->delay_fn)) ? static_cast<uint32_t>(c->hold_ctas) : 0;
  const uint32_t cap = nk <= 16 ? fp : 0;
  bool fill = false;
  const CacheRef cr = al ? cache_for(c, dt, e0, e0 + count, s, &fill) : CacheRef{};
  if (!cr.ptr) return launch_synth_reduce(dt, src, dst, count, e0, c->d_virt_keys, nk, stamp, s, launches, {}, cap);
  if (fill && cr.kind == ((dt == cemuInt32 || dt == cemuUint32) ? kCacheWide32 : kCacheLanes16)) {
    // one pass synthesises, folds and writes the entries (+ the tail's)
    return launch_synth_reduce_filling(dt, src, dst, count, e0, c->d_virt_keys, nk, stamp, s, launches, cr, 0);
  }
  if (fill) {  // > 256 emulated ranks of a byte kind (centred or uint32 entries): fill, then the cached fold
    if (stamp) {  // the call starts with the fill
      if (const cudaError_t e = launch_stamp(stamp, s, launches)) return e;
      stamp = nullptr;
    }
    const bool words = dt == cemuInt32 || dt == cemuUint32;
    if (const cudaError_t e = launch_synth_cache_fill(words, e0, count, c->d_virt_keys, nk, cr, s, launches)) return e;
    note_filled(c, cr, s);
  }
  return launch_synth_reduce(dt, src, dst, count, e0, c->d_virt_keys, nk, stamp, s, launches, cr, fp);
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
    note_filled(c, cr, s);
  }
  a.cache = cr.ptr;
  a.cache_kind = cr.kind;
  a.cache_clean = cr.clean;
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
