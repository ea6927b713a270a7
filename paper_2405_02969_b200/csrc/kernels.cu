// kernels.cu -- sm_100a kernels of the emulated collective.
//
// synth_reduce_vec   THE hot kernel.  One streaming pass over the real
//                    rank's buffer: 128-bit non-allocating loads, the
//                    emulated peers' contributions synthesised in registers
//                    from the counter-based hash (payload.cuh) and summed in
//                    SWAR 16-bit lanes, one fused add with the local value,
//                    128-bit streaming stores.  HBM traffic is exactly the
//                    algorithmic 2S bytes: synthesised peers cost no bytes.
//                    Replaces, per call, the reference's 2(n-1) TCP frames,
//                    FrameReader copies and reduce_add_i32/u8
//                    (proj/src/collective.cpp:268-355, reduce.cpp:42-60).
// synth_fill_vec     write-only synthesis of whole emulated blocks
//                    (allgather blocks, a broadcast from an emulated root).
// delay_spin_kernel  evaluates the alpha-beta model on the device
//                    (delay_math.cuh, bit-exact with delay.cpp:5-47 and the
//                    llround floors of engine.cpp:36-42), then releases the
//                    K to-real steps in order on %globaltimer -- the device
//                    analogue of the emulator's poller (emulator.cpp:165-191)
//                    enqueued on the collective's stream.
// *_scalar           element-wise fallbacks (misaligned pointers, 64-bit
//                    types, tails).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "delay_math.cuh"
#include "kernels.hpp"
#include "payload.cuh"


namespace cemu_b200 {
namespace {

constexpr int kThreads = 256;
constexpr uint32_t kMaxKeys = kMaxEmulatedPeers;  // kernels.hpp

__device__ __forceinline__ int64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<int64_t>(t);
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ uint2 ld_stream64(const uint2* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void st_stream(uint4* p, const uint4& v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// bytewise (mod 256) add of two packed words
__device__ __forceinline__ uint32_t add_bytes(uint32_t a, uint32_t b) {
  return ((a & 0x7F7F7F7Fu) + (b & 0x7F7F7F7Fu)) ^ ((a ^ b) & 0x80808080u);
}

__device__ __forceinline__ float f32_of(uint32_t u) { return __uint_as_float(u); }
__device__ __forceinline__ uint32_t u32_of(float f) { return __float_as_uint(f); }

// x (+) s * 2^-7 with a single rounding in fp32 (s*2^-7 is exact).
__device__ __forceinline__ float fold_f32(float x, int32_t s) {
  return __fadd_rn(x, __int2float_rn(s) * kDyadicScale);
}

// a + b per element of packed 16-bit pairs: fp32 add, one rounding to T
__device__ __forceinline__ uint32_t fold_bf16x2_add(uint32_t a, uint32_t b) {
  __nv_bfloat162 va = *reinterpret_cast<__nv_bfloat162*>(&a);
  __nv_bfloat162 vb = *reinterpret_cast<__nv_bfloat162*>(&b);
  __nv_bfloat162 r;
  r.x = __float2bfloat16_rn(__fadd_rn(__bfloat162float(va.x), __bfloat162float(vb.x)));
  r.y = __float2bfloat16_rn(__fadd_rn(__bfloat162float(va.y), __bfloat162float(vb.y)));
  return *reinterpret_cast<uint32_t*>(&r);
}

__device__ __forceinline__ uint32_t fold_f16x2_add(uint32_t a, uint32_t b) {
  __half2 va = *reinterpret_cast<__half2*>(&a);
  __half2 vb = *reinterpret_cast<__half2*>(&b);
  __half2 r;
  r.x = __float2half_rn(__fadd_rn(__half2float(va.x), __half2float(vb.x)));
  r.y = __float2half_rn(__fadd_rn(__half2float(va.y), __half2float(vb.y)));
  return *reinterpret_cast<uint32_t*>(&r);
}

// ---------------------------------------------------------------------------
// vector kinds
// ---------------------------------------------------------------------------
enum VKind { kF32 = 0, kF16 = 1, kBF16 = 2, kU8 = 3, kI32 = 4 };

template <int K>
struct VT;
// EPV elements per 16-byte vector, WPV payload words per vector.
template <> struct VT<kF32>  { static constexpr int EPV = 4,  WPV = 1; static constexpr bool kWords = false; };
template <> struct VT<kF16>  { static constexpr int EPV = 8,  WPV = 2; static constexpr bool kWords = false; };
template <> struct VT<kBF16> { static constexpr int EPV = 8,  WPV = 2; static constexpr bool kWords = false; };
template <> struct VT<kU8>   { static constexpr int EPV = 16, WPV = 4; static constexpr bool kWords = false; };
template <> struct VT<kI32>  { static constexpr int EPV = 4,  WPV = 4; static constexpr bool kWords = true; };

// ---------------------------------------------------------------------------
// generic per-element path (all 10 datatypes)
// ---------------------------------------------------------------------------
// per-peer hash constants live in shared memory as (k1, km) pairs
__device__ __forceinline__ uint32_t pword(uint2 k, uint64_t j) { return payload_mix(k.x, k.y, payload_c1(j)); }

__device__ __forceinline__ uint32_t pbyte(uint2 k, uint64_t e) {
  return (pword(k, e >> 2) >> (8 * (e & 3))) & 0xFFu;
}

__device__ __forceinline__ uint2 peer_consts(uint32_t key) {
  return make_uint2(payload_k1(key), payload_km(key));
}

template <int DT>
__device__ void elem_reduce(const void* src, void* dst, uint64_t i, uint64_t e,
                            const uint2* keys, uint32_t nkeys) {
  if constexpr (DT == cemuInt8 || DT == cemuUint8) {
    uint32_t acc = static_cast<const uint8_t*>(src)[i];
    for (uint32_t q = 0; q < nkeys; ++q) acc += pbyte(keys[q], e);
    static_cast<uint8_t*>(dst)[i] = static_cast<uint8_t>(acc);
  } else if constexpr (DT == cemuInt32 || DT == cemuUint32) {
    uint32_t acc = static_cast<const uint32_t*>(src)[i];
    for (uint32_t q = 0; q < nkeys; ++q) acc += pword(keys[q], e);
    static_cast<uint32_t*>(dst)[i] = acc;
  } else if constexpr (DT == cemuInt64 || DT == cemuUint64) {
    uint64_t acc = static_cast<const uint64_t*>(src)[i];
    for (uint32_t q = 0; q < nkeys; ++q) {
      acc += static_cast<uint64_t>(pword(keys[q], 2 * e)) |
             (static_cast<uint64_t>(pword(keys[q], 2 * e + 1)) << 32);
    }
    static_cast<uint64_t*>(dst)[i] = acc;
  } else {
    int32_t s = 0;
    for (uint32_t q = 0; q < nkeys; ++q) s += static_cast<int32_t>(pbyte(keys[q], e)) - 128;
    if constexpr (DT == cemuFloat64) {
      static_cast<double*>(dst)[i] =
          __dadd_rn(static_cast<const double*>(src)[i], static_cast<double>(s) * 0.0078125);
    } else if constexpr (DT == cemuFloat32) {
      static_cast<float*>(dst)[i] = fold_f32(static_cast<const float*>(src)[i], s);
    } else if constexpr (DT == cemuFloat16) {
      const __half x = static_cast<const __half*>(src)[i];
      static_cast<__half*>(dst)[i] = __float2half_rn(fold_f32(__half2float(x), s));
    } else {
      const __nv_bfloat16 x = static_cast<const __nv_bfloat16*>(src)[i];
      static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(fold_f32(__bfloat162float(x), s));
    }
  }
}

// Exact byte sums t_b = sum over the peers of byte b of payload word j, from
// the raw keys in global memory: a centred cache entry's escape (kernels.hpp
// kCacheCentered16) -- rare by construction, so it stays out of line.
__device__ __noinline__ uint4 exact_byte_sums(const uint32_t* __restrict__ keys, uint32_t nkeys, uint64_t j) {
  const uint32_t c1 = payload_c1(j);
  uint4 t = make_uint4(0, 0, 0, 0);
  for (uint32_t q = 0; q < nkeys; ++q) {
    const uint32_t key = keys[q];
    const uint32_t w = payload_mix(payload_k1(key), payload_km(key), c1);
    t.x += w & 0xFFu;
    t.y += (w >> 8) & 0xFFu;
    t.z += (w >> 16) & 0xFFu;
    t.w += w >> 24;
  }
  return t;
}

// elem_reduce from the synthesis cache: t = the peers' byte sum (or word
// sum) of element e, so s = t - 128 n is elem_reduce's dyadic sum exactly.
// `kind` is the cache's CacheKind; `keys` (global) serve centred escapes.
template <int DT>
__device__ void elem_fold_cached(const void* src, void* dst, uint64_t i, uint64_t e, const void* cache, int kind,
                                 uint32_t nkeys, const uint32_t* keys) {
  if constexpr (DT == cemuInt32 || DT == cemuUint32) {
    static_cast<uint32_t*>(dst)[i] = static_cast<const uint32_t*>(src)[i] + static_cast<const uint32_t*>(cache)[e];
  } else if constexpr (DT == cemuInt64 || DT == cemuUint64 || DT == cemuFloat64) {
    __trap();  // never cached (scalar path only)
  } else {
    uint32_t t;
    if (kind == kCacheWide32) {
      t = static_cast<const uint32_t*>(cache)[e];
    } else {
      t = static_cast<const uint16_t*>(cache)[e];
      if (kind == kCacheCentered16) {
        if (t == 0) {
          const uint4 x = exact_byte_sums(keys, nkeys, e >> 2);
          const uint32_t b = static_cast<uint32_t>(e & 3);
          t = b == 0 ? x.x : (b == 1 ? x.y : (b == 2 ? x.z : x.w));
        } else {
          t += c16_offset(nkeys);
        }
      }
    }
    if constexpr (DT == cemuInt8 || DT == cemuUint8) {
      static_cast<uint8_t*>(dst)[i] = static_cast<uint8_t>(static_cast<const uint8_t*>(src)[i] + t);
    } else {
      const int32_t sum = static_cast<int32_t>(t) - 128 * static_cast<int32_t>(nkeys);
      if constexpr (DT == cemuFloat32) {
        static_cast<float*>(dst)[i] = fold_f32(static_cast<const float*>(src)[i], sum);
      } else if constexpr (DT == cemuFloat16) {
        const __half x = static_cast<const __half*>(src)[i];
        static_cast<__half*>(dst)[i] = __float2half_rn(fold_f32(__half2float(x), sum));
      } else {
        const __nv_bfloat16 x = static_cast<const __nv_bfloat16*>(src)[i];
        static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(fold_f32(__bfloat162float(x), sum));
      }
    }
  }
}

template <int DT>
__device__ void elem_fill(void* dst, uint64_t i, uint64_t e, uint32_t raw_key) {
  const uint2 key = peer_consts(raw_key);
  if constexpr (DT == cemuInt8 || DT == cemuUint8) {
    static_cast<uint8_t*>(dst)[i] = static_cast<uint8_t>(pbyte(key, e));
  } else if constexpr (DT == cemuInt32 || DT == cemuUint32) {
    static_cast<uint32_t*>(dst)[i] = pword(key, e);
  } else if constexpr (DT == cemuInt64 || DT == cemuUint64) {
    static_cast<uint64_t*>(dst)[i] = static_cast<uint64_t>(pword(key, 2 * e)) |
                                     (static_cast<uint64_t>(pword(key, 2 * e + 1)) << 32);
  } else {
    const int32_t s = static_cast<int32_t>(pbyte(key, e)) - 128;
    if constexpr (DT == cemuFloat64) {
      static_cast<double*>(dst)[i] = static_cast<double>(s) * 0.0078125;
    } else if constexpr (DT == cemuFloat32) {
      static_cast<float*>(dst)[i] = __int2float_rn(s) * kDyadicScale;
    } else if constexpr (DT == cemuFloat16) {
      static_cast<__half*>(dst)[i] = __float2half_rn(__int2float_rn(s) * kDyadicScale);
    } else {
      static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(__int2float_rn(s) * kDyadicScale);
    }
  }
}

__device__ __forceinline__ void load_keys(uint2* skeys, const uint32_t* keys, uint32_t nkeys,
                                          uint32_t shift = 0) {
  for (uint32_t i = threadIdx.x; i < nkeys; i += blockDim.x) skeys[i + shift] = peer_consts(keys[i]);
  __syncthreads();
}

// How the vector kernels walk the emulated peers (a template parameter so
// every variant keeps 16-byte-aligned LDS.128 loads of key pairs):
//   kSeed1   odd peer count: peer 0 seeds the sums, the rest go in pairs;
//            keys sit one slot up in shared memory (key q at skeys[q + 1])
//            so the pairs start on a 16-byte boundary
//   kSeed2   even peer count: peers 0 and 1 seed the sums, pairs after
//   kGroups  > 256 byte-kind peers: 256-peer groups, lanes flushed per group
//   kCache16 no synthesis: the peers' per-element byte sums t (<= 256
//            peers, uint16 lanes) are read from the communicator's synthesis
//            cache (synth_cache_fill wrote them; see "synthesis cache" below)
//   kCache32 the same with uint32 entries: byte sums of > 8192 peers, or the
//            wrapping word sums of the 32-bit integer kinds
//   kCacheC16 the same with centred uint16 entries (257..8192 peers; an
//            entry 0 is an escape recomputed from the keys, kernels.hpp)
//   kCacheC16F centred entries of a range known to hold no escape (its fill
//            counted none): the kCache16 fold with the centred constants
enum PeerMode { kSeed1 = 0, kSeed2 = 1, kGroups = 2, kCache16 = 3, kCache32 = 4, kCacheC16 = 5, kCacheC16F = 6 };
__host__ __device__ constexpr uint32_t key_shift(int mode) { return mode == kSeed1 ? 1u : 0u; }
__host__ __device__ constexpr bool cached(int mode) { return mode >= kCache16; }
__host__ __device__ constexpr int cache_kind_of(int mode) {
  return mode == kCache16 ? kCacheLanes16 : (mode == kCacheC16 || mode == kCacheC16F ? kCacheCentered16 : kCacheWide32);
}
inline int peer_mode(bool words, uint32_t nkeys) {
  if (!words && nkeys > 256) return kGroups;  // 16-bit lanes hold <= 257 bytes
  return (nkeys & 1) ? kSeed1 : kSeed2;
}

template <int DT>
__global__ void __launch_bounds__(kThreads) synth_reduce_scalar(const void* src, void* dst,
                                                                uint64_t count, uint64_t elem_base,
                                                                const uint32_t* keys,
                                                                uint32_t nkeys, int64_t* stamp) {
  extern __shared__ uint2 skeys[];
  if (stamp && blockIdx.x == 0 && threadIdx.x == 0) *stamp = globaltimer_ns();
  load_keys(skeys, keys, nkeys);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += stride) {
    elem_reduce<DT>(src, dst, i, elem_base + i, skeys, nkeys);
  }
}

// ---------------------------------------------------------------------------
// the hot kernel
// ---------------------------------------------------------------------------
// acc + a on the FMA pipe: `one` is a runtime 1 (kernel argument), so ptxas
// keeps an IMAD instead of folding it into an ALU-pipe IADD3.  The hash and
// the byte extraction already saturate the ALU pipe (ncu: 93% ALU / 17% FMA
// at 63 peers before this split).
__device__ __forceinline__ uint32_t mad_add(uint32_t a, uint32_t one, uint32_t acc) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(one), "r"(acc));
  return d;
}

// Per-word byte sums from the two accumulators of one peer group (<= 257
// peers): A = sum of whole words (mod 2^32), H = sum of odd bytes in 16-bit
// lanes (S1, S3).  The even-byte lanes follow exactly:
//   S0 + S2 * 2^16 = A - S1 * 2^8 - S3 * 2^24 = A - H * 2^8  (mod 2^32)
// so the mask of the even bytes is never computed per peer.
__device__ __forceinline__ uint32_t even_lanes(uint32_t a, uint32_t h) { return a - (h << 8); }

__device__ __forceinline__ void decode_byte_sums(uint32_t a, uint32_t h, uint32_t s[4]) {
  const uint32_t even = even_lanes(a, h);
  s[0] = even & 0xFFFFu;
  s[1] = h & 0xFFFFu;
  s[2] = even >> 16;
  s[3] = h >> 16;
}

// A 16-bit lane t dropped into the mantissa of 1.5 * 2^16 (one PRMT) is the
// float 98304 + t * 2^-7 exactly (ulp 2^-7 in [2^16, 2^17)); subtracting
// 98304 + n (n peers, each biased by 128) is exact too (same binade), so
//   lane_delta = (t - 128 n) * 2^-7
// costs PRMT + FADD instead of IADD + I2F + FMUL.
constexpr uint32_t kLaneMagic = 0x47C00000u;  // 98304.0f
// (the magic is materialised opaquely so ptxas keeps it in a register and
// the selector as the PRMT immediate, not the other way round)
__device__ __forceinline__ uint32_t lane_magic() {
  uint32_t m;
  asm("mov.b32 %0, %1;" : "=r"(m) : "n"(kLaneMagic));
  return m;
}
__device__ __forceinline__ float lane_float(uint32_t w, uint32_t sel) {
  return __uint_as_float(__byte_perm(w, lane_magic(), sel));
}

// 98304 + byte_e(w) * 2^-7, exactly (byte e of w into the magic's mantissa)
__device__ __forceinline__ float byte_float(uint32_t w, int e) {
  return __uint_as_float(__byte_perm(w, lane_magic(), 0x7650 | static_cast<uint32_t>(e)));
}

// sm_100 packed fp32 pair add (FADD2): two lanes per instruction
__device__ __forceinline__ uint64_t pack_f32x2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 add_f32x2(float a0, float a1, float b0, float b1) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pack_f32x2(a0, a1)), "l"(pack_f32x2(b0, b1)));
  float2 f;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(f.x), "=f"(f.y) : "l"(r));
  return f;
}

// c1 of every payload word of one thread-tile: word j = j0 + u*kThreads*W + w
// with j0 = word_base + (tile base + thread) * W.  Within a tile the high
// half of j almost never changes, so c1 = ((lo*Weyl) ^ (hi*WeylHi)) * M1 is
// one add and one xor per word off a per-tile base (the M1 multiply folds
// into the peer loop's first IMAD); a tile straddling 2^32 words takes the
// general form.
template <int W, int U>
__device__ __forceinline__ void tile_ctrs(uint64_t j0, uint32_t* ctr) {
  constexpr uint32_t kSpan = (U - 1) * kThreads * W + W - 1;
  const uint32_t lo = static_cast<uint32_t>(j0);
  if (lo <= 0xFFFFFFFFu - kSpan) {
    const uint32_t lw = lo * kWeyl;
    const uint32_t hx = static_cast<uint32_t>(j0 >> 32) * kWeylHi;
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        ctr[u * W + w] = ((lw + static_cast<uint32_t>(u * kThreads * W + w) * kWeyl) ^ hx) * kMul1;
      }
    }
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int w = 0; w < W; ++w) ctr[u * W + w] = payload_c1(j0 + static_cast<uint64_t>(u) * kThreads * W + w);
    }
  }
}

// One payload word's byte-kind lanes from its single-group accumulators
// (A, H over n <= 257 peers): u8 -> the packed byte sums mod 256 in r[0];
// float kinds -> the four exact dyadic deltas (t - 128 n) * 2^-7 in r[0..3].
template <int K>
__device__ __forceinline__ void ah_to_lanes(uint32_t a, uint32_t h, uint32_t n, uint32_t* r) {
  const uint32_t even = even_lanes(a, h);
  if constexpr (K == kU8) {  // bytes wrap: low byte of each lane
    r[0] = __byte_perm(even, h, 0x6240);
  } else {
    const float c = -(98304.0f + static_cast<float>(n));
    const float2 d01 = add_f32x2(lane_float(even, 0x7610), lane_float(h, 0x7610), c, c);
    const float2 d23 = add_f32x2(lane_float(even, 0x7632), lane_float(h, 0x7632), c, c);
    r[0] = __float_as_uint(d01.x);
    r[1] = __float_as_uint(d01.y);
    r[2] = __float_as_uint(d23.x);
    r[3] = __float_as_uint(d23.y);
  }
}

// The same lanes from cached byte sums: t16 = the word's four uint16 lane
// sums packed as (t0 | t1 << 16, t2 | t3 << 16) -- exactly the values
// ah_to_lanes decodes from (A, H), so the result is bit-identical.
// kC: centred entries u = t - c16_offset(n): t - 128 n = u - (32768 +
// ceil(n / 2)), so the magic's constant moves by (32768 + ceil(n/2)) * 2^-7
// -- still exact (<= 98560 + 112 in the same binade); bytes add the offset's
// low byte back.
template <int K, bool kC = false>
__device__ __forceinline__ void t16_to_lanes(uint32_t w01, uint32_t w23, uint32_t n, uint32_t* r) {
  if constexpr (K == kU8) {
    r[0] = __byte_perm(w01, w23, 0x6420);  // low byte of each lane sum
    if constexpr (kC) r[0] = add_bytes(r[0], (c16_offset(n) & 0xFFu) * 0x01010101u);
  } else {
    const float c = kC ? -(98560.0f + static_cast<float>((n + 1) / 2) * kDyadicScale)
                       : -(98304.0f + static_cast<float>(n));
    const float2 d01 = add_f32x2(lane_float(w01, 0x7610), lane_float(w01, 0x7632), c, c);
    const float2 d23 = add_f32x2(lane_float(w23, 0x7610), lane_float(w23, 0x7632), c, c);
    r[0] = __float_as_uint(d01.x);
    r[1] = __float_as_uint(d01.y);
    r[2] = __float_as_uint(d23.x);
    r[3] = __float_as_uint(d23.y);
  }
}

// nonzero iff some 16-bit lane of x is 0 (a centred entry's escape)
__device__ __forceinline__ uint32_t zero_lane16(uint32_t x) { return (x - 0x00010001u) & ~x & 0x80008000u; }

// ... and from uint32 byte sums T_e (> 256 peers: centred escapes, uint32
// entries beyond 8192 peers): the kGroups flush below
// computes the same integers (sum over groups of t - 128 * group size).
template <int K>
__device__ __forceinline__ void t32_to_lanes(const uint4& t, uint32_t n, uint32_t* r) {
  if constexpr (K == kU8) {
    r[0] = (t.x & 0xFFu) | ((t.y & 0xFFu) << 8) | ((t.z & 0xFFu) << 16) | (t.w << 24);
  } else {
    const int32_t b = 128 * static_cast<int32_t>(n);
    r[0] = __float_as_uint(__int2float_rn(static_cast<int32_t>(t.x) - b) * kDyadicScale);
    r[1] = __float_as_uint(__int2float_rn(static_cast<int32_t>(t.y) - b) * kDyadicScale);
    r[2] = __float_as_uint(__int2float_rn(static_cast<int32_t>(t.z) - b) * kDyadicScale);
    r[3] = __float_as_uint(__int2float_rn(static_cast<int32_t>(t.w) - b) * kDyadicScale);
  }
}

// Emulated-peer contribution of the U vectors of one thread-tile, as lanes
// r[] ready for fold_vec:
//   float kinds  r[4i + e] = float bits of (sum over peers of byte e of
//                word i, each minus 128) * 2^-7   (exact)
//   u8           r[4i]     = the four byte sums of word i, mod 256, packed
//   word kinds   r[i]      = wrapping sum of word i
// ctr[] holds the hoisted c1 values; nkeys >= 1 (launchers route 0 peers
// elsewhere) and, for kSeed2, even.  Cached modes read the sums of words
// j0 + u * kThreads * W + w from `cache` instead (ctr, skeys unused).
template <int K, int U, int kMode, bool kEnt = false>
__device__ __forceinline__ void peer_sums(const uint32_t* ctr, const uint2* skeys, uint32_t nkeys,
                                          uint32_t one, uint32_t* r, const void* cache = nullptr,
                                          uint64_t j0 = 0, uint32_t* ent = nullptr,
                                          const uint32_t* gkeys = nullptr, uint64_t jlim = ~0ull) {
  using T = VT<K>;
  constexpr int NW = U * T::WPV;
  if constexpr (kMode == kCacheC16) {
    // centred entries: every load of the tile first (an escape test between
    // two loads would serialise them), then decode; escapes out of line
    constexpr int W = T::WPV;
    uint2 c[U * W];
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        // the last tile's idle vectors read the range's last word instead of
        // words past it (the segment may end right before an unmapped page);
        // their lanes are never stored
        const uint64_t j = min(j0 + static_cast<uint64_t>(u) * kThreads * W, jlim - W) + w;
        c[u * W + w] = ld_stream64(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(cache) + 4 * j));
      }
    }
#pragma unroll
    for (int i = 0; i < U * W; ++i) t16_to_lanes<K, true>(c[i].x, c[i].y, nkeys, r + 4 * i);
    uint32_t esc = 0;
#pragma unroll
    for (int i = 0; i < U * W; ++i) esc |= zero_lane16(c[i].x) | zero_lane16(c[i].y);
    if (esc) {  // (unrolled: r stays in registers)
#pragma unroll
      for (int i = 0; i < U * W; ++i) {
        if (zero_lane16(c[i].x) | zero_lane16(c[i].y)) {
          const uint64_t j = j0 + static_cast<uint64_t>(i / W) * kThreads * W + (i % W);
          t32_to_lanes<K>(exact_byte_sums(gkeys, nkeys, j), nkeys, r + 4 * i);
        }
      }
    }
    return;
  }
  if constexpr (cached(kMode)) {
    constexpr int W = T::WPV;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // the last tile's idle vectors read the range's last vector's entries,
      // not entries past the range (the segment may end right before an
      // unmapped page); their lanes are never stored
      const uint64_t jv = min(j0 + static_cast<uint64_t>(u) * kThreads * W, jlim - W);
      if constexpr (T::kWords) {  // four words = four elements: one 16-byte entry
        const uint4 c = ld_stream(reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(cache) + jv));
        r[u * 4 + 0] = c.x;
        r[u * 4 + 1] = c.y;
        r[u * 4 + 2] = c.z;
        r[u * 4 + 3] = c.w;
      } else if constexpr (kMode == kCache16 || kMode == kCacheC16F) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const uint2 c = ld_stream64(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(cache) + 4 * (jv + w)));
          t16_to_lanes<K, kMode == kCacheC16F>(c.x, c.y, nkeys, r + 4 * (u * W + w));
        }
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const uint4 c = ld_stream(reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(cache) + 4 * (jv + w)));
          t32_to_lanes<K>(c, nkeys, r + 4 * (u * W + w));
        }
      }
    }
    return;
  }
  constexpr bool kMulti = kMode == kGroups;
  constexpr uint32_t kShift = key_shift(kMode);
  constexpr uint32_t kSeed = kMode == kSeed1 ? 1 : 2;  // peers folded in before the pair loop
  if constexpr (T::kWords) {
    {
      const uint2 k0 = skeys[kShift];
#pragma unroll
      for (int i = 0; i < NW; ++i) r[i] = payload_mix(k0.x, k0.y, ctr[i]);
      if constexpr (kSeed == 2) {
        const uint2 k1 = skeys[1];
#pragma unroll
        for (int i = 0; i < NW; ++i) r[i] = mad_add(payload_mix(k1.x, k1.y, ctr[i]), one, r[i]);
      }
    }
#pragma unroll 2
    for (uint32_t q = kSeed; q < nkeys; ++q) {
      const uint2 key = skeys[q + kShift];
#pragma unroll
      for (int i = 0; i < NW; ++i) r[i] = mad_add(payload_mix(key.x, key.y, ctr[i]), one, r[i]);
    }
    if constexpr (kEnt) {  // synthesis-cache entries: the word sums themselves
#pragma unroll
      for (int i = 0; i < NW; ++i) ent[i] = r[i];
    }
  } else {
    const uint32_t groups = kMulti ? (nkeys + 255) / 256 : 1;
    int32_t s[kMulti ? NW * 4 : 1];
    if constexpr (kMulti) {
#pragma unroll
      for (int i = 0; i < NW * 4; ++i) s[i] = 0;
    }
    for (uint32_t g = 0; g < groups; ++g) {
      const uint32_t q0 = g * 256;
      const uint32_t q1 = kMulti ? min(nkeys, q0 + 256) : nkeys;
      uint32_t a[NW], h[NW];
      if constexpr (kMulti) {
#pragma unroll
        for (int i = 0; i < NW; ++i) a[i] = h[i] = 0;
      } else {
        const uint2 k0 = skeys[kShift];
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          a[i] = payload_mix(k0.x, k0.y, ctr[i]);
          h[i] = __byte_perm(a[i], 0u, 0x4341);
        }
        if constexpr (kSeed == 2) {
          const uint2 k1 = skeys[1];
#pragma unroll
          for (int i = 0; i < NW; ++i) {
            const uint32_t w = payload_mix(k1.x, k1.y, ctr[i]);
            a[i] = mad_add(w, one, a[i]);
            h[i] = mad_add(__byte_perm(w, 0u, 0x4341), one, h[i]);
          }
        }
      }
#pragma unroll 2
      for (uint32_t q = kMulti ? q0 : kSeed; q < q1; ++q) {
        const uint2 key = skeys[q + kShift];
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          const uint32_t w = payload_mix(key.x, key.y, ctr[i]);
          a[i] = mad_add(w, one, a[i]);
          h[i] = mad_add(__byte_perm(w, 0u, 0x4341), one, h[i]);
        }
      }
      if constexpr (!kMulti) {
#pragma unroll
        for (int i = 0; i < NW; ++i) ah_to_lanes<K>(a[i], h[i], nkeys, r + 4 * i);
        if constexpr (kEnt) {  // synthesis-cache entries: the packed uint16 lane sums
#pragma unroll
          for (int i = 0; i < NW; ++i) {
            const uint32_t even = even_lanes(a[i], h[i]);
            ent[2 * i] = __byte_perm(even, h[i], 0x5410);      // t0 | t1 << 16
            ent[2 * i + 1] = __byte_perm(even, h[i], 0x7632);  // t2 | t3 << 16
          }
        }
      } else {
        // float kinds carry the -128 offset of the dyadic value; bytes wrap
        const int32_t bias = K == kU8 ? 0 : 128 * static_cast<int32_t>(q1 - q0);
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          uint32_t t[4];
          decode_byte_sums(a[i], h[i], t);
#pragma unroll
          for (int e = 0; e < 4; ++e) s[i * 4 + e] += static_cast<int32_t>(t[e]) - bias;
        }
      }
    }
    if constexpr (kMulti) {
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        const int32_t* t = s + 4 * i;
        if constexpr (K == kU8) {
          r[4 * i] = (static_cast<uint32_t>(t[0]) & 0xFFu) | ((static_cast<uint32_t>(t[1]) & 0xFFu) << 8) |
                     ((static_cast<uint32_t>(t[2]) & 0xFFu) << 16) | (static_cast<uint32_t>(t[3]) << 24);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) r[4 * i + e] = __float_as_uint(__int2float_rn(t[e]) * kDyadicScale);
        }
      }
    }
  }
}

// x + d in fp32 (one rounding) with x a 16-bit half of a packed pair: the
// sm_100 mixed-precision add reads the half in place (FHADD.BF16 .H0/.H1),
// so there is no unpack.
__device__ __forceinline__ uint32_t bf16x2_fold(uint32_t p, uint32_t dlo, uint32_t dhi) {
  float lo, hi;
  asm("{ .reg .b16 l, h; mov.b32 {l, h}, %2;\n"
      "  add.rn.f32.bf16 %0, l, %3;\n  add.rn.f32.bf16 %1, h, %4; }"
      : "=f"(lo), "=f"(hi) : "r"(p), "f"(__uint_as_float(dlo)), "f"(__uint_as_float(dhi)));
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ uint32_t f16x2_fold(uint32_t p, uint32_t dlo, uint32_t dhi) {
  float lo, hi;
  asm("{ .reg .b16 l, h; mov.b32 {l, h}, %2;\n"
      "  add.rn.f32.f16 %0, l, %3;\n  add.rn.f32.f16 %1, h, %4; }"
      : "=f"(lo), "=f"(hi) : "r"(p), "f"(__uint_as_float(dlo)), "f"(__uint_as_float(dhi)));
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// One rounding per element: x (+) delta in fp32, then to the element type
// (floats); x + sum (integers).  `r` points at this vector's lanes.
template <int K>
__device__ __forceinline__ uint4 fold_vec(const uint4& x, const uint32_t* r) {
  uint4 y;
  if constexpr (VT<K>::kWords) {
    y.x = x.x + r[0];
    y.y = x.y + r[1];
    y.z = x.z + r[2];
    y.w = x.w + r[3];
  } else if constexpr (K == kF32) {
    const float2 a = add_f32x2(f32_of(x.x), f32_of(x.y), f32_of(r[0]), f32_of(r[1]));
    const float2 b = add_f32x2(f32_of(x.z), f32_of(x.w), f32_of(r[2]), f32_of(r[3]));
    y.x = u32_of(a.x);
    y.y = u32_of(a.y);
    y.z = u32_of(b.x);
    y.w = u32_of(b.y);
  } else if constexpr (K == kBF16) {  // words 0 (elements 0..3) and 1 (4..7)
    y.x = bf16x2_fold(x.x, r[0], r[1]);
    y.y = bf16x2_fold(x.y, r[2], r[3]);
    y.z = bf16x2_fold(x.z, r[4], r[5]);
    y.w = bf16x2_fold(x.w, r[6], r[7]);
  } else if constexpr (K == kF16) {
    y.x = f16x2_fold(x.x, r[0], r[1]);
    y.y = f16x2_fold(x.y, r[2], r[3]);
    y.z = f16x2_fold(x.z, r[4], r[5]);
    y.w = f16x2_fold(x.w, r[6], r[7]);
  } else {  // kU8: packed byte sums of word i at r[4i]
    y.x = add_bytes(x.x, r[0]);
    y.y = add_bytes(x.y, r[4]);
    y.z = add_bytes(x.z, r[8]);
    y.w = add_bytes(x.w, r[12]);
  }
  return y;
}

// kFill: also write the synthesis cache's entries of the tile's payload
// words (single-group modes: <= 256 byte-kind peers, or the word kinds) --
// the first call over a range fills the cache in its own synthesis pass.
template <int K, int DT, int U, int kMode, bool kFill = false>
__global__ void __launch_bounds__(kThreads) synth_reduce_vec(
    const uint4* __restrict__ src, uint4* dst, uint64_t nvec, uint64_t word_base,
    const uint32_t* __restrict__ keys, uint32_t nkeys, int64_t* stamp, const void* tail_src,
    void* tail_dst, uint32_t ntail, uint64_t tail_e0, uint32_t one, const void* __restrict__ cache) {
  using T = VT<K>;
  constexpr int W = T::WPV, NW = U * W;
  extern __shared__ uint2 skeys[];
  if (stamp && blockIdx.x == 0 && threadIdx.x == 0) *stamp = globaltimer_ns();
  if constexpr (!cached(kMode)) load_keys(skeys, keys, nkeys, key_shift(kMode));

  const uint64_t tile = static_cast<uint64_t>(kThreads) * U;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * tile; base < nvec;
       base += static_cast<uint64_t>(gridDim.x) * tile) {
    // 1. issue every load of the tile first: synthesis below never depends
    //    on them, so the whole peer loop hides the HBM latency.
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t v = base + static_cast<uint64_t>(u) * kThreads + threadIdx.x;
      if (v < nvec) x[u] = ld_stream(src + v);
    }
    const uint64_t j0 = word_base + (base + threadIdx.x) * W;
    uint32_t ctr[NW];
    if constexpr (!cached(kMode)) tile_ctrs<W, U>(j0, ctr);
    // 2. the emulated peers' sums (registers only; or the cached sums),
    // 3. fold + stream out
    uint32_t r[T::kWords ? NW : NW * 4];
    uint32_t ent[kFill ? (T::kWords ? NW : 2 * NW) : 1];
    peer_sums<K, U, kMode, kFill>(ctr, skeys, nkeys, one, r, cache, j0, ent, keys, word_base + nvec * W);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t v = base + static_cast<uint64_t>(u) * kThreads + threadIdx.x;
      if (v < nvec) st_stream(dst + v, fold_vec<K>(x[u], r + u * W * (T::kWords ? 1 : 4)));
      if constexpr (kFill) {
        if (v < nvec) {
          const uint64_t jv = j0 + static_cast<uint64_t>(u) * kThreads * W;
          if constexpr (T::kWords) {  // `cache` is the (writable) entry array in fill mode
            st_stream(reinterpret_cast<uint4*>(const_cast<uint32_t*>(static_cast<const uint32_t*>(cache)) + jv),
                      make_uint4(ent[u * 4], ent[u * 4 + 1], ent[u * 4 + 2], ent[u * 4 + 3]));
          } else {
#pragma unroll
            for (int w = 0; w < W; ++w) {
              reinterpret_cast<uint2*>(const_cast<void*>(cache))[jv + w] =
                  make_uint2(ent[2 * (u * W + w)], ent[2 * (u * W + w) + 1]);
            }
          }
        }
      }
    }
  }
  // ragged tail (< one vector): the last block's first threads
  if (ntail && blockIdx.x == gridDim.x - 1 && threadIdx.x < ntail) {
    if constexpr (cached(kMode)) {
      elem_fold_cached<DT>(tail_src, tail_dst, threadIdx.x, tail_e0 + threadIdx.x, cache, cache_kind_of(kMode),
                           nkeys, keys);
    } else {
      elem_reduce<DT>(tail_src, tail_dst, threadIdx.x, tail_e0 + threadIdx.x, skeys + key_shift(kMode), nkeys);
    }
  }
}


// Small buffers: P threads share one vector's peers (peer q goes to lane
// q mod P), each accumulating A/H (or word sums) over its share; the P
// partial sums -- plain wrapping adds, so the lane bounds are those of the
// whole peer set -- are combined with warp shuffles and the group's first
// lane folds and stores.  Used when one thread per vector would leave most
// of the machine idle (a 4 KiB call at 63 peers is 8 blocks instead of 1).
template <int K, int DT, int P>
__global__ void __launch_bounds__(kThreads) synth_reduce_split(
    const uint4* __restrict__ src, uint4* dst, uint64_t nvec, uint64_t word_base,
    const uint32_t* __restrict__ keys, uint32_t nkeys, int64_t* stamp, const void* tail_src,
    void* tail_dst, uint32_t ntail, uint64_t tail_e0, uint32_t one) {
  using T = VT<K>;
  constexpr int W = T::WPV;
  static_assert(P >= 2 && P <= 32 && (P & (P - 1)) == 0, "P: power of two within a warp");
  extern __shared__ uint2 skeys[];
  if (stamp && blockIdx.x == 0 && threadIdx.x == 0) *stamp = globaltimer_ns();
  load_keys(skeys, keys, nkeys);
  const uint32_t part = threadIdx.x % P;
  const uint64_t v = static_cast<uint64_t>(blockIdx.x) * (kThreads / P) + threadIdx.x / P;
  const bool live = v < nvec;
  uint4 x = make_uint4(0, 0, 0, 0);
  if (live && part == 0) x = ld_stream(src + v);
  uint32_t ctr[W], a[W], h[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    ctr[w] = payload_c1(word_base + v * W + w);
    a[w] = h[w] = 0;
  }
  for (uint32_t q = part; q < nkeys; q += P) {
    const uint2 key = skeys[q];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t wv = payload_mix(key.x, key.y, ctr[w]);
      a[w] = mad_add(wv, one, a[w]);
      if constexpr (!T::kWords) h[w] = mad_add(__byte_perm(wv, 0u, 0x4341), one, h[w]);
    }
  }
#pragma unroll
  for (int o = P / 2; o > 0; o >>= 1) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      a[w] += __shfl_xor_sync(0xffffffffu, a[w], o);
      if constexpr (!T::kWords) h[w] += __shfl_xor_sync(0xffffffffu, h[w], o);
    }
  }
  if (live && part == 0) {
    uint32_t r[T::kWords ? W : W * 4];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      if constexpr (T::kWords) {
        r[w] = a[w];
      } else {
        ah_to_lanes<K>(a[w], h[w], nkeys, r + 4 * w);
      }
    }
    st_stream(dst + v, fold_vec<K>(x, r));
  }
  if (ntail && blockIdx.x == gridDim.x - 1 && threadIdx.x < ntail) {
    elem_reduce<DT>(tail_src, tail_dst, threadIdx.x, tail_e0 + threadIdx.x, skeys, nkeys);
  }
}

// ---------------------------------------------------------------------------
// synthesis cache
// ---------------------------------------------------------------------------
// The emulated peers' contribution to element e depends only on (seed,
// rank, e), never on the call (payload.cuh).  A communicator that sees the
// same element range again -- a training loop all-reduces the same buckets
// every step -- folds it from a per-element cache of the peers' sums instead
// of synthesising W-k payloads again: at >= 16 emulated peers synthesis is
// issue-bound (8 issue slots per peer-word), the cached fold is a 3-stream
// HBM pass (read x, read the entry, write y).  This kernel writes the
// entries of payload words [word_begin, word_end) with the hot kernel's own
// arithmetic (A = sum of words, H = sum of odd bytes, even lanes = A - H<<8),
// so a cached fold is bit-identical to a synthesised one.
//   kEntry 0: uint16 lane sums t0..t3 of each word, packed (t0|t1<<16, t2|t3<<16)
//          1: uint32 byte sums (> 256 peers: 256-peer groups, summed exactly)
//          2: uint32 wrapping word sums (32-bit integer kinds; word = element)
//          3: centred uint16 byte sums, packed as 0 (257..8192 peers: t as in
//             1, then u = t - c16_offset(n) or the escape 0, kernels.hpp)
template <int U, int kEntry>
__global__ void __launch_bounds__(kThreads) synth_cache_fill(uint64_t word_begin, uint64_t word_end,
                                                             const uint32_t* __restrict__ keys, uint32_t nkeys,
                                                             void* cache, uint32_t one, uint32_t* esc) {
  constexpr int W = 4, NW = U * W;
  extern __shared__ uint2 skeys[];
  load_keys(skeys, keys, nkeys);
  const uint64_t j0 = word_begin + (static_cast<uint64_t>(blockIdx.x) * kThreads * U + threadIdx.x) * W;
  uint32_t ctr[NW];
  tile_ctrs<W, U>(j0, ctr);
  auto word_of = [&](int i) { return j0 + static_cast<uint64_t>(i / W) * kThreads * W + (i % W); };
  if constexpr (kEntry == 2) {
    uint32_t sum[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) sum[i] = 0;
#pragma unroll 2
    for (uint32_t q = 0; q < nkeys; ++q) {
      const uint2 key = skeys[q];
#pragma unroll
      for (int i = 0; i < NW; ++i) sum[i] = mad_add(payload_mix(key.x, key.y, ctr[i]), one, sum[i]);
    }
    auto* out = static_cast<uint32_t*>(cache);
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      if (word_of(i) < word_end) out[word_of(i)] = sum[i];
    }
  } else {
    constexpr bool kWide = kEntry == 1 || kEntry == 3;
    uint32_t tw[kWide ? NW * 4 : NW * 2];
    if constexpr (kWide) {
#pragma unroll
      for (int i = 0; i < NW * 4; ++i) tw[i] = 0;
    }
    const uint32_t groups = kWide ? (nkeys + 255) / 256 : 1;
    for (uint32_t g = 0; g < groups; ++g) {
      const uint32_t q0 = g * 256, q1 = kWide ? min(nkeys, q0 + 256) : nkeys;
      uint32_t a[NW], h[NW];
#pragma unroll
      for (int i = 0; i < NW; ++i) a[i] = h[i] = 0;
#pragma unroll 2
      for (uint32_t q = q0; q < q1; ++q) {
        const uint2 key = skeys[q];
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          const uint32_t w = payload_mix(key.x, key.y, ctr[i]);
          a[i] = mad_add(w, one, a[i]);
          h[i] = mad_add(__byte_perm(w, 0u, 0x4341), one, h[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        const uint32_t even = even_lanes(a[i], h[i]);
        if constexpr (kWide) {
          uint32_t t[4];
          decode_byte_sums(a[i], h[i], t);
#pragma unroll
          for (int e = 0; e < 4; ++e) tw[4 * i + e] += t[e];
        } else {
          tw[2 * i] = __byte_perm(even, h[i], 0x5410);      // t0 | t1 << 16
          tw[2 * i + 1] = __byte_perm(even, h[i], 0x7632);  // t2 | t3 << 16
        }
      }
    }
    uint32_t nesc = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const uint64_t j = word_of(i);
      if (j >= word_end) continue;
      if constexpr (kEntry == 3) {
        const uint32_t off = c16_offset(nkeys);
        uint32_t u[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          u[e] = tw[4 * i + e] - off;
          if (u[e] - 1u >= 0xFFFFu) {  // outside [1, 65535]: escape
            u[e] = 0;
            ++nesc;
          }
        }
        reinterpret_cast<uint2*>(cache)[j] = make_uint2(u[0] | (u[1] << 16), u[2] | (u[3] << 16));
      } else if constexpr (kWide) {
        reinterpret_cast<uint4*>(cache)[j] = make_uint4(tw[4 * i], tw[4 * i + 1], tw[4 * i + 2], tw[4 * i + 3]);
      } else {
        reinterpret_cast<uint2*>(cache)[j] = make_uint2(tw[2 * i], tw[2 * i + 1]);
      }
    }
    if (kEntry == 3 && nesc && esc) atomicAdd_system(esc, nesc);  // rare: mapped host memory
  }
}

// ---------------------------------------------------------------------------
// fused multi-GPU allreduce over peer memory
// ---------------------------------------------------------------------------
// With k real GPUs on the box, GPU `me` owns 1/k of the vectors: it pulls
// that slice from every real GPU's send buffer over NVLink (P2P loads), sums
// the real contributions in ascending real-rank order, adds the W-k emulated
// ranks' synthesised payloads in the same pass, and pushes the result into
// every real GPU's recv buffer (P2P stores).  One launch replaces NCCL
// reduce-scatter + synthesis + NCCL allgather; every byte crosses NVLink
// once each way, overlapped with the synthesis.  Cross-GPU ordering uses
// epoch flags in IPC-mapped memory (release/acquire at system scope):
//   start: each GPU's first CTA tells every peer "my kernel started" (so its
//          stream's earlier writes to send are complete); every CTA waits
//          for all peers' start flags before its first remote load;
//   done:  the last CTA to finish on each GPU tells every peer "my writes
//          into your recv are done" and waits for the same from all peers,
//          so the kernel ends only when its recv buffer is complete.
// Every wait has a %globaltimer timeout that sets `error` instead of hanging.
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Flags hold (epoch << 20) | signature.  A start flag of the same epoch with
// another signature means the ranks disagree on the call (error 3).
constexpr int kSigBits = 20;
__device__ __forceinline__ uint64_t flag_word(uint64_t epoch, uint32_t sig) {
  return (epoch << kSigBits) | (sig & ((1u << kSigBits) - 1));
}

// 0 = arrived, 1 = timed out, 3 = signature mismatch
__device__ __forceinline__ int wait_flag(const uint64_t* f, uint64_t epoch, uint32_t sig, bool check_sig,
                                         int64_t t0, int64_t timeout) {
  uint64_t v;
  while (((v = ld_acquire_sys(f)) >> kSigBits) < epoch) {
    if (globaltimer_ns() - t0 > timeout) return 1;
    __nanosleep(64);
  }
  if (check_sig && (v >> kSigBits) == epoch && (v & ((1u << kSigBits) - 1)) != (sig & ((1u << kSigBits) - 1))) {
    return 3;
  }
  return 0;
}

// real-part fold in the datatype's own arithmetic (the oracle's real_sum)
template <int K>
__device__ __forceinline__ uint4 add_real(const uint4& a, const uint4& b) {
  uint4 r;
  if constexpr (K == kF32) {
    r.x = u32_of(__fadd_rn(f32_of(a.x), f32_of(b.x)));
    r.y = u32_of(__fadd_rn(f32_of(a.y), f32_of(b.y)));
    r.z = u32_of(__fadd_rn(f32_of(a.z), f32_of(b.z)));
    r.w = u32_of(__fadd_rn(f32_of(a.w), f32_of(b.w)));
  } else if constexpr (K == kBF16) {
    r.x = fold_bf16x2_add(a.x, b.x);
    r.y = fold_bf16x2_add(a.y, b.y);
    r.z = fold_bf16x2_add(a.z, b.z);
    r.w = fold_bf16x2_add(a.w, b.w);
  } else if constexpr (K == kF16) {
    r.x = fold_f16x2_add(a.x, b.x);
    r.y = fold_f16x2_add(a.y, b.y);
    r.z = fold_f16x2_add(a.z, b.z);
    r.w = fold_f16x2_add(a.w, b.w);
  } else if constexpr (K == kU8) {
    r.x = add_bytes(a.x, b.x);
    r.y = add_bytes(a.y, b.y);
    r.z = add_bytes(a.z, b.z);
    r.w = add_bytes(a.w, b.w);
  } else {
    r.x = a.x + b.x;
    r.y = a.y + b.y;
    r.z = a.z + b.z;
    r.w = a.w + b.w;
  }
  return r;
}

// ragged elements after the last full vector: same fold, one element
template <int DT, int kMode>
__device__ void fused_tail_elem(const FusedArgs& a, uint32_t i, const uint2* skeys, int ndst) {
  using S = typename std::conditional<
      DT == cemuInt8 || DT == cemuUint8, uint8_t,
      typename std::conditional<DT == cemuFloat16 || DT == cemuBfloat16, uint16_t, uint32_t>::type>::type;
  S acc = reinterpret_cast<const S*>(a.src[0] + a.v_end)[i];
  for (int g = 1; g < a.k; ++g) {
    const S b = reinterpret_cast<const S*>(a.src[g] + a.v_end)[i];
    if constexpr (DT == cemuFloat32) {
      acc = u32_of(__fadd_rn(f32_of(acc), f32_of(b)));
    } else if constexpr (DT == cemuBfloat16) {
      const uint32_t r = fold_bf16x2_add(static_cast<uint32_t>(acc), static_cast<uint32_t>(b));
      acc = static_cast<S>(r & 0xFFFFu);
    } else if constexpr (DT == cemuFloat16) {
      const uint32_t r = fold_f16x2_add(static_cast<uint32_t>(acc), static_cast<uint32_t>(b));
      acc = static_cast<S>(r & 0xFFFFu);
    } else {
      acc = static_cast<S>(acc + b);
    }
  }
  S out;
  if constexpr (cached(kMode)) {
    elem_fold_cached<DT>(&acc, &out, 0, a.tail_e0 + i, a.cache, cache_kind_of(kMode), a.nkeys, a.keys);
  } else {
    elem_reduce<DT>(&acc, &out, 0, a.tail_e0 + i, skeys, a.nkeys);
  }
  if (ndst == 0) {  // gated: the local copy only
    reinterpret_cast<S*>(a.dst[a.me] + a.v_end)[i] = out;
    return;
  }
  for (int g = 0; g < ndst; ++g) reinterpret_cast<S*>(a.dst[g] + a.v_end)[i] = out;
}

template <int K, int DT, int KMAX, int U, int kMode>
__global__ void __launch_bounds__(kThreads) fused_allreduce_vec(const __grid_constant__ FusedArgs a) {
  using T = VT<K>;
  constexpr int W = T::WPV, NW = U * W;
  extern __shared__ uint2 skeys[];
  __shared__ int abort_s, ndst_s;
  const int64_t t0 = globaltimer_ns();
  // every real GPU runs the same fused calls in the same order, so the local
  // counters agree; the last CTA advances it when the call is complete
  const uint64_t epoch = *a.epoch + 1;
  if (a.stamp && blockIdx.x == 0 && threadIdx.x == 0) *a.stamp = t0;
  // start barrier: announce, then wait for every peer's announcement
  if (a.barriers && blockIdx.x == 0 && threadIdx.x < a.k && static_cast<int>(threadIdx.x) != a.me) {
    st_release_sys(a.peer_flags[threadIdx.x] + a.me, flag_word(epoch, a.sig));
  }
  if (threadIdx.x == 0) {
    abort_s = 0;
    // a fold-only chunk after a failed start barrier (the comm's error word
    // set) keeps its result local (dst[me]): no store reaches a peer's memory
    ndst_s = (a.gate && *reinterpret_cast<volatile const uint32_t*>(a.gate) != 0) ? 0 : a.ndst;
  }
  if constexpr (!cached(kMode)) {
    load_keys(skeys, a.keys, a.nkeys, key_shift(kMode));
  } else {
    __syncthreads();  // abort_s initialised before any thread may set it
  }
  if (a.barriers && threadIdx.x < a.k && static_cast<int>(threadIdx.x) != a.me) {
    const int w = wait_flag(a.flags + threadIdx.x, epoch, a.sig, true, t0, a.timeout_ns);
    if (w) {
      atomicExch(a.error, static_cast<uint32_t>(w));
      abort_s = 1;
    }
  }
  __syncthreads();
  if (abort_s) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.epoch = epoch;
    return;
  }
  const int ndst = ndst_s;

  const uint64_t tile = static_cast<uint64_t>(kThreads) * U;
  for (uint64_t base = a.v_begin + static_cast<uint64_t>(blockIdx.x) * tile; base < a.v_end;
       base += static_cast<uint64_t>(gridDim.x) * tile) {
    // every real GPU's slice first (local HBM + NVLink), then synthesis
    uint4 x[KMAX][U];
#pragma unroll
    for (int g = 0; g < KMAX; ++g) {
      if (g < a.k) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t v = base + static_cast<uint64_t>(u) * kThreads + threadIdx.x;
          if (v < a.v_end) x[g][u] = ld_stream(a.src[g] + v);
        }
      }
    }
    const uint64_t j0 = a.word_base + (base + threadIdx.x) * W;
    uint32_t ctr[NW];
    if constexpr (!cached(kMode)) tile_ctrs<W, U>(j0, ctr);
    uint32_t r[T::kWords ? NW : NW * 4];
    peer_sums<K, U, kMode>(ctr, skeys, a.nkeys, 1u, r, a.cache, j0, nullptr, a.keys, a.word_base + a.v_end * W);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t v = base + static_cast<uint64_t>(u) * kThreads + threadIdx.x;
      if (v >= a.v_end) continue;
      uint4 real = x[0][u];
#pragma unroll
      for (int g = 1; g < KMAX; ++g) {
        if (g < a.k) real = add_real<K>(real, x[g][u]);
      }
      const uint4 y = fold_vec<K>(real, r + u * W * (T::kWords ? 1 : 4));
      if (ndst == 0) {  // gated: the local copy only
        st_stream(a.dst[a.me] + v, y);
        continue;
      }
#pragma unroll
      for (int g = 0; g < KMAX; ++g) {
        if (g < ndst) st_stream(a.dst[g] + v, y);
      }
    }
  }
  if (a.ntail && blockIdx.x == gridDim.x - 1 && threadIdx.x < a.ntail) {
    fused_tail_elem<DT, kMode>(a, threadIdx.x, skeys + key_shift(kMode), ndst);
  }

  if (!a.barriers) return;
  // done barrier: the last CTA on this GPU publishes and waits
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(a.counter, 1u);
    if (prev == gridDim.x - 1) {
      *a.counter = 0;
      __threadfence_system();
      for (int g = 0; g < a.k; ++g) {
        if (g != a.me) st_release_sys(a.peer_flags[g] + 8 + a.me, flag_word(epoch, 0));
      }
      for (int g = 0; g < a.k; ++g) {
        if (g != a.me && wait_flag(a.flags + 8 + g, epoch, 0, false, globaltimer_ns(), a.timeout_ns)) {
          atomicExch(a.error, 2u);
        }
      }
      *a.epoch = epoch;
    }
  }
}

// The fused kernel's barriers alone (one warp): phase 0 = start (peers'
// send buffers complete, recv buffers free), phase 1 = done (every peer's
// copies into my recv have completed -- each peer launches this after its
// copy-engine pushes, in stream order -- then the epoch advances).
__global__ void peer_barrier_kernel(const __grid_constant__ FusedArgs a, int phase) {
  const uint64_t epoch = *a.epoch + 1;
  const int64_t t0 = globaltimer_ns();
  const int g = static_cast<int>(threadIdx.x);
  const bool peer = g < a.k && g != a.me;
  if (phase == 0) {
    if (a.stamp && g == 0) *a.stamp = t0;
    if (peer) st_release_sys(a.peer_flags[g] + a.me, flag_word(epoch, a.sig));
    if (peer) {
      const int w = wait_flag(a.flags + g, epoch, a.sig, true, t0, a.timeout_ns);
      if (w) atomicExch(a.error, static_cast<uint32_t>(w));
    }
  } else {
    __threadfence_system();
    if (peer) st_release_sys(a.peer_flags[g] + 8 + a.me, flag_word(epoch, 0));
    if (peer && wait_flag(a.flags + 8 + g, epoch, 0, false, t0, a.timeout_ns)) atomicExch(a.error, 2u);
    __syncwarp();
    if (g == 0) *a.epoch = epoch;
  }
}

// ---------------------------------------------------------------------------
// fills
// ---------------------------------------------------------------------------
template <int K>
__device__ __forceinline__ uint4 synth_vector(uint2 key, uint64_t word0) {
  using T = VT<K>;
  uint32_t wd[T::WPV];
#pragma unroll
  for (int w = 0; w < T::WPV; ++w) wd[w] = pword(key, word0 + w);
  uint4 r;
  if constexpr (K == kU8 || K == kI32) {
    r.x = wd[0];
    r.y = wd[1];
    r.z = wd[2];
    r.w = wd[3];
  } else if constexpr (K == kF32) {
    const uint32_t h = wd[0];
    r.x = u32_of(__int2float_rn(static_cast<int32_t>(h & 0xFFu) - 128) * kDyadicScale);
    r.y = u32_of(__int2float_rn(static_cast<int32_t>((h >> 8) & 0xFFu) - 128) * kDyadicScale);
    r.z = u32_of(__int2float_rn(static_cast<int32_t>((h >> 16) & 0xFFu) - 128) * kDyadicScale);
    r.w = u32_of(__int2float_rn(static_cast<int32_t>(h >> 24) - 128) * kDyadicScale);
  } else {
    uint32_t out[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {  // pair p = elements 2p, 2p+1
      const uint32_t h = wd[p >> 1];
      // (byte - 128) * 2^-7 exactly: the byte in the mantissa of 1.5 * 2^16
      // (one PRMT), minus 98305 -- no quarter-rate I2F
      const int e = (p & 1) * 2;
      const float2 ab = add_f32x2(byte_float(h, e), byte_float(h, e + 1), -98305.0f, -98305.0f);
      const float a = ab.x, b = ab.y;
      if constexpr (K == kBF16) {
        __nv_bfloat162 v;
        v.x = __float2bfloat16_rn(a);
        v.y = __float2bfloat16_rn(b);
        out[p] = *reinterpret_cast<uint32_t*>(&v);
      } else {
        __half2 v;
        v.x = __float2half_rn(a);
        v.y = __float2half_rn(b);
        out[p] = *reinterpret_cast<uint32_t*>(&v);
      }
    }
    r = make_uint4(out[0], out[1], out[2], out[3]);
  }
  return r;
}

template <int K>
__global__ void __launch_bounds__(kThreads) synth_fill_vec(uint4* dst, uint64_t nvec_per_block,
                                                           const uint32_t* __restrict__ index,
                                                           const uint32_t* __restrict__ keys,
                                                           uint32_t nblocks, uint32_t index0,
                                                           uint32_t key0, const uint4* own_src,
                                                           uint32_t own_index, int64_t* stamp,
                                                           uint64_t word_base) {
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *stamp = globaltimer_ns();
  const uint32_t b = blockIdx.y;
  const bool copy = b == nblocks;
  const uint32_t idx = copy ? own_index : (index ? index[b] : index0);
  const uint2 key = peer_consts(copy ? 0u : (keys ? keys[b] : key0));
  uint4* out = dst + static_cast<uint64_t>(idx) * nvec_per_block;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec_per_block;
       v += stride) {
    if (copy) {
      st_stream(out + v, ld_stream(own_src + v));
    } else {
      st_stream(out + v, synth_vector<K>(key, word_base + v * VT<K>::WPV));
    }
  }
}

// The same fill over a 1-D grid of address-ordered tiles (U vectors per
// thread): block i writes tile i mod T of rank block i / T, so consecutive
// blocks write consecutive HBM.
template <int K, int U>
__global__ void __launch_bounds__(kThreads) synth_fill_tiled(uint4* dst, uint64_t nvec_per_block,
                                                             uint64_t tiles_per_block,
                                                             const uint32_t* __restrict__ index,
                                                             const uint32_t* __restrict__ keys,
                                                             uint32_t nblocks, uint32_t index0, uint32_t key0,
                                                             const uint4* own_src, uint32_t own_index,
                                                             int64_t* stamp, uint64_t word_base) {
  if (stamp && blockIdx.x == 0 && threadIdx.x == 0) *stamp = globaltimer_ns();
  const uint64_t b = blockIdx.x / tiles_per_block;
  const uint64_t tile = blockIdx.x - b * tiles_per_block;
  const bool copy = b == nblocks;
  const uint32_t idx = copy ? own_index : (index ? index[b] : index0);
  uint4* out = dst + static_cast<uint64_t>(idx) * nvec_per_block;
  const uint64_t v0 = tile * kThreads * U + threadIdx.x;
  if (copy) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t v = v0 + static_cast<uint64_t>(u) * kThreads;
      if (v < nvec_per_block) st_stream(out + v, ld_stream(own_src + v));
    }
    return;
  }
  const uint2 key = peer_consts(keys ? keys[b] : key0);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t v = v0 + static_cast<uint64_t>(u) * kThreads;
    if (v < nvec_per_block) st_stream(out + v, synth_vector<K>(key, word_base + v * VT<K>::WPV));
  }
}

template <int DT>
__global__ void __launch_bounds__(kThreads) synth_fill_scalar(void* dst, uint64_t block_elems,
                                                              const uint32_t* index,
                                                              const uint32_t* keys, uint32_t nblocks,
                                                              uint32_t index0, uint32_t key0,
                                                              const void* own_src, uint32_t own_index,
                                                              int64_t* stamp, int elem_size,
                                                              uint64_t elem_base) {
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *stamp = globaltimer_ns();
  const uint32_t b = blockIdx.y;
  const bool copy = b == nblocks;
  const uint32_t idx = copy ? own_index : (index ? index[b] : index0);
  const uint32_t key = copy ? 0u : (keys ? keys[b] : key0);
  uint8_t* out = static_cast<uint8_t*>(dst) + static_cast<uint64_t>(idx) * block_elems * elem_size;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  if (copy) {
    const uint64_t nbytes = block_elems * elem_size;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nbytes;
         i += stride) {
      out[i] = static_cast<const uint8_t*>(own_src)[i];
    }
    return;
  }
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < block_elems;
       i += stride) {
    elem_fill<DT>(out, i, elem_base + i, key);
  }
}

// Fused allgather.  CTAs [0, push_ctas) copy the own block into every real
// GPU's recv (local store + NVLink P2P stores) after the start barrier; the
// remaining CTAs synthesise the emulated blocks into the local recv (HBM
// writes only: regenerating an emulated block beats moving it).  Real peers'
// blocks arrive by their own pushes; the done barrier makes them visible.
template <int K>
__global__ void __launch_bounds__(kThreads) fused_allgather_vec(const __grid_constant__ FusedGatherArgs a,
                                                                uint32_t push_ctas) {
  __shared__ int abort_s;
  const int64_t t0 = globaltimer_ns();
  const uint64_t epoch = *a.epoch + 1;
  if (a.stamp && blockIdx.x == 0 && threadIdx.x == 0) *a.stamp = t0;
  if (blockIdx.x == 0 && threadIdx.x < a.k && static_cast<int>(threadIdx.x) != a.me) {
    st_release_sys(a.peer_flags[threadIdx.x] + a.me, flag_word(epoch, a.sig));
  }
  if (blockIdx.x < push_ctas) {
    if (threadIdx.x == 0) abort_s = 0;
    __syncthreads();
    if (threadIdx.x < a.k && static_cast<int>(threadIdx.x) != a.me) {
      const int w = wait_flag(a.flags + threadIdx.x, epoch, a.sig, true, t0, a.timeout_ns);
      if (w) {
        atomicExch(a.error, static_cast<uint32_t>(w));
        abort_s = 1;
      }
    }
    __syncthreads();
    if (!abort_s) {
      const uint64_t off = static_cast<uint64_t>(a.own_block) * a.block_vecs;
      for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; v < a.block_vecs;
           v += static_cast<uint64_t>(push_ctas) * kThreads) {
        const uint4 x = ld_stream(a.own + v);
        for (int g = 0; g < a.k; ++g) st_stream(a.dst[g] + off + v, x);
      }
    }
  } else {
    const uint64_t total = static_cast<uint64_t>(a.nvirt) * a.block_vecs;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x - push_ctas) * kThreads;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x - push_ctas) * kThreads + threadIdx.x; i < total;
         i += stride) {
      const uint64_t b = i / a.block_vecs, v = i - b * a.block_vecs;
      const uint2 key = peer_consts(a.vkeys[b]);
      st_stream(a.dst[a.me] + static_cast<uint64_t>(a.vranks[b]) * a.block_vecs + v,
                synth_vector<K>(key, v * VT<K>::WPV));
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(a.counter, 1u);
    if (prev == gridDim.x - 1) {
      *a.counter = 0;
      __threadfence_system();
      for (int g = 0; g < a.k; ++g) {
        if (g != a.me) st_release_sys(a.peer_flags[g] + 8 + a.me, flag_word(epoch, 0));
      }
      for (int g = 0; g < a.k; ++g) {
        if (g != a.me && wait_flag(a.flags + 8 + g, epoch, 0, false, globaltimer_ns(), a.timeout_ns)) {
          atomicExch(a.error, 2u);
        }
      }
      *a.epoch = epoch;
    }
  }
}

// ---------------------------------------------------------------------------
// delay
// ---------------------------------------------------------------------------
__global__ void stamp_kernel(int64_t* slot) { slot[0] = globaltimer_ns(); }

// Compute emulation (clock.hpp:29-37 emulate_compute_us): hold the stream
// for `ns` of %globaltimer.  With a chain slot the layer ends at
// previous deadline + ns (device-absolute), so back-to-back launches do not
// accumulate their ~1-2 us launch gaps into the emulated compute timeline;
// `resync` (after a cross-stream wait) restarts the chain at the kernel's
// own start.
__global__ void spin_ns_kernel(int64_t ns, int64_t* chain, int resync) {
  const int64_t now = globaltimer_ns();
  const int64_t start = (chain && !resync) ? *chain : now;
  const int64_t end = start + ns;
  int64_t t = now;
  while (t < end) {
    if (end - t > 8000) __nanosleep(2000);
    t = globaltimer_ns();
  }
  if (chain) *chain = end;
}

// Join of two timelines: the compute chain continues from the later of its
// own deadline and the network's last release (the wait-all of a training
// step), so the event-to-kernel gap after a cross-stream wait is not added to
// the emulated compute.
__global__ void chain_join_kernel(int64_t* chain, const int64_t* other) {
  const int64_t o = *other;
  if (o > *chain) *chain = o;
}

// The last gate (= the largest floor, the call's modelled latency).
__device__ __forceinline__ int64_t run_max_floor(uint32_t k, const int64_t* sgate, const int64_t* gates_beyond) {
  if (k == 0) return 0;
  return k - 1 < static_cast<uint32_t>(kInlineOffsets) ? sgate[k - 1] : gates_beyond[k - 1];
}

__device__ __forceinline__ void delay_spin_body(const DelayLaunch& d, int64_t* slot, const double* inline_offs) {
  int64_t* floors = slot + kSlotHeader;
  int64_t* release = floors + d.kmax;
  double* offs = reinterpret_cast<double*>(release + d.kmax);
  __shared__ int64_t t0_s;
  if (threadIdx.x == 0) {
    // slot[0] keeps the call's real start (its first kernel's stamp); the
    // schedule's origin slot[4] moves back to the previous call's end only
    // when queue chaining is on (cemuCommSetQueueChaining) and this call was
    // queued right behind it
    const int64_t stamp = d.self_stamp ? globaltimer_ns() : slot[0];
    int64_t t0 = stamp;
    if (d.prev_end && d.queue_gap_ns > 0) {
      const int64_t pe = *d.prev_end;
      if (pe > 0 && t0 >= pe && t0 - pe <= d.queue_gap_ns) t0 = pe;
    }
    t0_s = t0;
    slot[0] = stamp;
    slot[4] = t0;
  }
  // Evaluate the model on the device: delay.cpp:23-47 offsets and
  // engine.cpp:41 llround floors, strided over the block.  A delay-model
  // plugin's offsets (DelayModelFn, delay.hpp:52-55) arrive preloaded.
  __shared__ int64_t sfloor[kInlineOffsets];
  __shared__ int64_t sgate[kInlineOffsets];
  __shared__ int64_t wmax[kThreads / 32];
  const double total = (!d.preloaded && d.model.kind == 1) ? model_total_us(d.model, d.coll, d.n, d.bytes) : 0.0;
  for (uint32_t j = threadIdx.x; j < d.k; j += blockDim.x) {
    const double o = inline_offs ? inline_offs[j] : d.preloaded ? offs[j] : release_offset_us(d.model, total, j, d.k);
    offs[j] = o;
    const int64_t f = llround(o);
    floors[j] = f;
    if (j < static_cast<uint32_t>(kInlineOffsets)) sfloor[j] = f;
  }
  __syncthreads();
  // Head-of-line release (engine.cpp:58-70): step j leaves once its floor
  // has passed and step j-1 has left -- at the first poll at or after its
  // gate, the running maximum of the floors up to j.  The gates are a
  // block-wide prefix maximum (each thread a contiguous segment), kept in
  // shared memory (first kInlineOffsets steps) or, beyond, in the release
  // array the times later overwrite.
  auto floor_at = [&](uint32_t j) { return j < static_cast<uint32_t>(kInlineOffsets) ? sfloor[j] : floors[j]; };
  auto gate_ref = [&](uint32_t j) -> int64_t& { return j < static_cast<uint32_t>(kInlineOffsets) ? sgate[j] : release[j]; };
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t seg = (d.k + blockDim.x - 1) / blockDim.x;
  const uint32_t sb = min(d.k, threadIdx.x * seg), se = min(d.k, sb + seg);
  int64_t m = 0;  // floors are >= 0
  for (uint32_t j = sb; j < se; ++j) m = max(m, floor_at(j));
  int64_t incl = m;  // inclusive scan of the segment maxima over the block
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl = max(incl, v);
  }
  if (lane == 31) wmax[warp] = incl;
  __syncthreads();
  int64_t run = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) run = 0;
  for (uint32_t w = 0; w < warp; ++w) run = max(run, wmax[w]);
  for (uint32_t j = sb; j < se; ++j) {
    run = max(run, floor_at(j));
    gate_ref(j) = run;
  }
  __syncthreads();
  const int64_t lat = run_max_floor(d.k, sgate, release);  // the last gate
  if (threadIdx.x == 0) slot[2] = lat;
  // A step released after its floor is late: the emulator's own work (the
  // synthesis kernels before this one) outlasted that step's floor, or the
  // spin overshot.  The largest lateness is recorded (slot[5]), and how far
  // the whole call overran its modelled latency (slot[6]), so such a call
  // is visible, never silently longer.
  // Thread 0 releases, one step per poll while the floors are spread out
  // (a few cycles per step: the last release follows the last floor by
  // nanoseconds).  When it is catching up -- step j's floor had already
  // passed -- and the gate 8 steps on has passed too, the whole run of
  // passed steps (a fixed or injected delay gives every step the same
  // floor) is found by binary search over the non-decreasing gates and
  // released at once; its per-step times are written after the call's end
  // is recorded.  A serial K-step loop would lengthen the call (126 steps on
  // one floor at world 64 took 8.8 us).
  if (threadIdx.x != 0) return;
  constexpr uint32_t kRuns = 64, kSerialRun = 8;
  __shared__ uint32_t run_b[kRuns], run_e[kRuns];
  __shared__ int64_t run_t[kRuns];
  auto gate = [&](uint32_t j) { return j < static_cast<uint32_t>(kInlineOffsets) ? sgate[j] : release[j]; };
  uint32_t nruns = 0;
  const int64_t t0 = t0_s;
  int64_t late = 0;
  int64_t t = globaltimer_ns();
  // the longest interval between two consecutive clock reads: a few us
  // (the sleep) normally; a pause of the whole device -- nothing of this
  // kernel running -- shows here and explains a late release (slot[3])
  int64_t prev = t, stall = 0;
  for (uint32_t j = 0; j < d.k;) {
    const int64_t target = t0 + floor_at(j) * 1000;
    if (t < target) {
      do {
        if (target - t > 8000) __nanosleep(2000);
        t = globaltimer_ns();
        stall = max(stall, t - prev);
        prev = t;
      } while (t < target);
    } else if (j + kSerialRun < d.k && t0 + gate(j + kSerialRun) * 1000 <= t) {
      uint32_t lo = j + kSerialRun + 1, hi = d.k;  // the first step whose gate is still ahead
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (t0 + gate(mid) * 1000 <= t) lo = mid + 1; else hi = mid;
      }
      if (nruns < kRuns) {
        run_b[nruns] = j;
        run_e[nruns] = lo;
        run_t[nruns] = t;
        ++nruns;
      } else {
        for (uint32_t i = j; i < lo; ++i) {
          late = max(late, t - (t0 + floor_at(i) * 1000));
          release[i] = t;
        }
      }
      j = lo;
      continue;
    }
    release[j] = t;
    late = max(late, t - target);
    ++j;
  }
  const int64_t end = globaltimer_ns();
  slot[6] = max(int64_t{0}, end - (t0 + lat * 1000));  // the call itself ran long by this much
  slot[1] = end;
  slot[3] = max(stall, end - prev);
  for (uint32_t r = 0; r < nruns; ++r) {  // the runs' per-step times and lateness
    for (uint32_t i = run_b[r]; i < run_e[r]; ++i) {
      late = max(late, run_t[r] - (t0 + floor_at(i) * 1000));
      release[i] = run_t[r];
    }
  }
  slot[5] = late;
}

__global__ void __launch_bounds__(kThreads) delay_spin_kernel(DelayLaunch d, int64_t* slot) {
  delay_spin_body(d, slot, nullptr);
}

// The real collective's SM footprint: `gridDim.x` CTAs stand in
// for the real collective's kernel (e.g. NCCL's channels) and hold an SM
// slot each -- kHoldThreads threads and the launch's shared-memory
// reservation -- from the call's start until its modelled end, so compute
// beside the collective on other streams loses the SMs a real collective
// would take.  Launched on a side stream forked at the call's start (ahead
// of the synthesis, as a real collective's kernel is dispatched), the first
// holder to run publishes the start in *start (zeroed before the launch);
// every holder leaves at start + lat_ns.
constexpr int kHoldThreads = 544;  // NCCL's CTA width on these boxes
__global__ void __launch_bounds__(kHoldThreads) footprint_kernel(unsigned long long* start, int64_t lat_ns,
                                                                 int active) {
  extern __shared__ char hold_smem[];
  __shared__ int64_t end_s;
  if (threadIdx.x == 0) {
    const unsigned long long now = static_cast<unsigned long long>(globaltimer_ns());
    const unsigned long long first = atomicCAS(start, 0ull, now);
    end_s = static_cast<int64_t>(first ? first : now) + lat_ns;
    hold_smem[0] = 0;  // the reservation is the point; touch it so it is kept
  }
  __syncthreads();
  const int64_t end = end_s;
  if (active) {
    while (globaltimer_ns() < end) {
    }
  } else {
    while (globaltimer_ns() < end) __nanosleep(2000);
  }
}

// A plugin's offsets travel in the launch's own parameter block (<= 16 KB):
// no host staging to recycle, and a captured graph keeps the captured call's
// offsets.
__global__ void __launch_bounds__(kThreads) delay_spin_inline_kernel(DelayLaunch d, int64_t* slot,
                                                                     const __grid_constant__ InlineOffsets o) {
  delay_spin_body(d, slot, o.us);
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = sms > 0 ? sms : 148;
  }
  return cached[dev];
}

// Opts a kernel into > 48 KB of dynamic shared memory when a large emulated
// world needs it (the default limit covers 6143 peers).
template <typename Kern>
cudaError_t fit_smem(Kern k, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}

template <typename Kern>
int blocks_per_sm(Kern k, size_t smem) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, kThreads, smem) != cudaSuccess || b < 1) {
    cudaGetLastError();
    b = 1;
  }
  return b;
}

// Launch shape of the hot kernel: U vectors per thread per tile and resident
// blocks per SM.  Few peers -> memory bound: small U, many resident warps
// (ncu at 7 peers: 6.47 TB/s with U=2 x 4 blocks/SM).  Many peers -> ALU
// bound: U=8 amortises the shared-memory key loads over more words.
// CEMU_SYNTH_U / CEMU_SYNTH_BPS override both (tuning only).
struct Shape {
  int u;
  int bps;
};

Shape pick_shape(int words_per_vec, uint32_t nkeys, uint64_t nvec) {
  static const int env_u = [] {
    const char* e = std::getenv("CEMU_SYNTH_U");
    return e ? std::atoi(e) : 0;
  }();
  static const int env_bps = [] {
    const char* e = std::getenv("CEMU_SYNTH_BPS");
    return e ? std::atoi(e) : 0;
  }();
  // <= 8 payload words and <= 4 vectors per thread per tile (8 resident
  // 16-byte loads push ptxas into a register-starved serial schedule of
  // the peer loop: measured 8% slower at 63 peers)
  const int u_max = std::min(4, 8 / words_per_vec);
  Shape sh{nkeys * static_cast<uint32_t>(words_per_vec) <= 8 ? 2 : std::max(2, u_max), 0};
  // small buffers: spread the synthesis over the machine before amortising
  // it over more words per thread (a 4 KiB call at 63 peers is otherwise
  // one block doing all 63 x 8 hashes per thread serially)
  const uint64_t fill = static_cast<uint64_t>(sm_count()) * 4 * kThreads;
  while (sh.u > 1 && nvec < fill * static_cast<uint64_t>(sh.u)) sh.u /= 2;
  if ((env_u == 1 || env_u == 2 || env_u == 4 || env_u == 8) && env_u <= std::max(2, 8 / words_per_vec)) sh.u = env_u;
  if (env_bps > 0) sh.bps = env_bps;
  return sh;
}

template <int K, int DT, int U>
cudaError_t run_vec_u(const void* src, void* dst, uint64_t count, uint64_t elem_base,
                      const uint32_t* keys, uint32_t nkeys, int64_t* stamp, cudaStream_t s, int bps_req,
                      void* fill = nullptr, uint32_t grid_cap = 0) {
  using T = VT<K>;
  const uint64_t nvec = count / T::EPV;
  const uint32_t ntail = static_cast<uint32_t>(count - nvec * T::EPV);
  const size_t es = T::kWords ? 4 : (K == kF32 ? 4 : (K == kU8 ? 1 : 2));
  const uint64_t word_base = T::kWords ? elem_base : elem_base / 4;
  const size_t smem = (static_cast<size_t>(nkeys) + 1) * 8;
  const int mode = peer_mode(T::kWords, nkeys);
  auto kern = mode == kGroups ? synth_reduce_vec<K, DT, U, kGroups>
              : mode == kSeed1 ? synth_reduce_vec<K, DT, U, kSeed1> : synth_reduce_vec<K, DT, U, kSeed2>;
  if (fill) {  // the same pass also writes the synthesis cache's entries
    if (mode == kGroups) return cudaErrorInvalidValue;
    kern = mode == kSeed1 ? synth_reduce_vec<K, DT, U, kSeed1, true> : synth_reduce_vec<K, DT, U, kSeed2, true>;
  }
  if (const cudaError_t e = fit_smem(kern, smem)) return e;
  const uint64_t tiles = (nvec + static_cast<uint64_t>(kThreads) * U - 1) / (static_cast<uint64_t>(kThreads) * U);
  // One tile per block over the whole buffer (not a persistent grid-stride
  // loop): the hardware block scheduler then sweeps HBM in address order,
  // measured 6.89 vs 6.30 TB/s for the fp32 world-8 pass (and faster at every
  // world size: scratch/tune_grid.py).  CEMU_SYNTH_GRID=persistent (or an
  // explicit CEMU_SYNTH_BPS) restores the persistent shape.
  static const bool persistent = [] {
    const char* e = std::getenv("CEMU_SYNTH_GRID");
    return (e && std::string(e) == "persistent") || std::getenv("CEMU_SYNTH_BPS");
  }();
  uint64_t cap = grid_cap ? grid_cap : 0x7FFFFFFFull;
  if (persistent) {
    const int occ = blocks_per_sm(kern, smem);
    cap = static_cast<uint64_t>(sm_count()) * (bps_req > 0 ? std::min(bps_req, occ) : std::min(occ, 4));
  }
  const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(tiles, cap));
  kern<<<static_cast<unsigned>(grid), kThreads, smem, s>>>(
      static_cast<const uint4*>(src), static_cast<uint4*>(dst), nvec, word_base, keys, nkeys,
      stamp, static_cast<const uint8_t*>(src) + nvec * T::EPV * es,
      static_cast<uint8_t*>(dst) + nvec * T::EPV * es, ntail, elem_base + nvec * T::EPV, 1u, fill);
  return cudaGetLastError();
}

// The fold of a cached call: the hot kernel in a cached mode, one tile of
// U = 2 vectors per thread per block (the memory-bound shape).
template <int K, int DT>
cudaError_t run_vec_cached(const void* src, void* dst, uint64_t count, uint64_t elem_base, const uint32_t* keys,
                           uint32_t nkeys, int64_t* stamp, cudaStream_t s, CacheRef cache, uint32_t grid_cap = 0) {
  using T = VT<K>;
  constexpr int U = 2;
  const uint64_t nvec = count / T::EPV;
  const uint32_t ntail = static_cast<uint32_t>(count - nvec * T::EPV);
  const size_t es = T::kWords ? 4 : (K == kF32 ? 4 : (K == kU8 ? 1 : 2));
  const uint64_t word_base = T::kWords ? elem_base : elem_base / 4;
  const uint64_t tiles = (nvec + static_cast<uint64_t>(kThreads) * U - 1) / (static_cast<uint64_t>(kThreads) * U);
  const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(tiles, grid_cap ? grid_cap : 0x7FFFFFFFull));
  auto kern = synth_reduce_vec<K, DT, U, kCache32>;
  if constexpr (!T::kWords) {
    if (cache.kind == kCacheLanes16) kern = synth_reduce_vec<K, DT, U, kCache16>;
    if (cache.kind == kCacheCentered16) {
      kern = cache.clean ? synth_reduce_vec<K, DT, U, kCacheC16F> : synth_reduce_vec<K, DT, U, kCacheC16>;
    }
  }
  kern<<<static_cast<unsigned>(grid), kThreads, 0, s>>>(
      static_cast<const uint4*>(src), static_cast<uint4*>(dst), nvec, word_base, keys, nkeys, stamp,
      static_cast<const uint8_t*>(src) + nvec * T::EPV * es, static_cast<uint8_t*>(dst) + nvec * T::EPV * es, ntail,
      elem_base + nvec * T::EPV, 1u, cache.ptr);
  return cudaGetLastError();
}

// Peer-split width for a buffer of nvec vectors: 0 = the per-vector kernels.
// Otherwise the largest power of two P <= 32 with >= 4 peers per thread and
// nvec * P within half a wave of resident threads.  Byte kinds need the
// whole peer set in one lane group (<= 256 peers).
int split_ways(bool words, uint32_t nkeys, uint64_t nvec) {
  static const int env = [] {
    const char* e = std::getenv("CEMU_SYNTH_SPLIT");
    return e ? std::atoi(e) : -1;  // 0 disables, P forces
  }();
  if (env == 0 || nvec == 0 || (!words && nkeys > 256)) return 0;
  if (env > 1) return env;
  // measured (world 64, graph replay): 4-64 KiB 2.4-3.0 -> 1.6-1.8 us, a tie
  // at 256 KiB, slower from 1 MiB -- so only up to 64 vectors per SM
  const uint64_t wave = static_cast<uint64_t>(sm_count()) * 2048;
  if (nkeys < 8 || nvec > static_cast<uint64_t>(sm_count()) * 64) return 0;
  int p = 1;
  while (p < 32 && static_cast<uint32_t>(p) * 8 <= nkeys && nvec * p * 2 <= wave) p *= 2;
  return p >= 2 ? p : 0;
}

template <int K, int DT, int P>
cudaError_t run_split(const void* src, void* dst, uint64_t count, uint64_t elem_base, const uint32_t* keys,
                      uint32_t nkeys, int64_t* stamp, cudaStream_t s) {
  using T = VT<K>;
  const uint64_t nvec = count / T::EPV;
  const uint32_t ntail = static_cast<uint32_t>(count - nvec * T::EPV);
  const size_t es = T::kWords ? 4 : (K == kF32 ? 4 : (K == kU8 ? 1 : 2));
  const uint64_t word_base = T::kWords ? elem_base : elem_base / 4;
  const uint64_t per_block = kThreads / P;
  const uint64_t grid = std::max<uint64_t>(1, (nvec + per_block - 1) / per_block);
  if (const cudaError_t e = fit_smem(synth_reduce_split<K, DT, P>, static_cast<size_t>(nkeys) * 8)) return e;
  synth_reduce_split<K, DT, P><<<static_cast<unsigned>(grid), kThreads, static_cast<size_t>(nkeys) * 8, s>>>(
      static_cast<const uint4*>(src), static_cast<uint4*>(dst), nvec, word_base, keys, nkeys, stamp,
      static_cast<const uint8_t*>(src) + nvec * T::EPV * es, static_cast<uint8_t*>(dst) + nvec * T::EPV * es,
      ntail, elem_base + nvec * T::EPV, 1u);
  return cudaGetLastError();
}

template <int K, int DT>
cudaError_t run_vec(const void* src, void* dst, uint64_t count, uint64_t elem_base,
                    const uint32_t* keys, uint32_t nkeys, int64_t* stamp, cudaStream_t s, void* fill = nullptr,
                    uint32_t grid_cap = 0) {
  constexpr int W = VT<K>::WPV;
  if (fill && split_ways(VT<K>::kWords, nkeys, count / VT<K>::EPV)) return cudaErrorInvalidValue;
  if (const int P = split_ways(VT<K>::kWords, nkeys, count / VT<K>::EPV)) {
    switch (P) {
      case 2: return run_split<K, DT, 2>(src, dst, count, elem_base, keys, nkeys, stamp, s);
      case 4: return run_split<K, DT, 4>(src, dst, count, elem_base, keys, nkeys, stamp, s);
      case 8: return run_split<K, DT, 8>(src, dst, count, elem_base, keys, nkeys, stamp, s);
      case 16: return run_split<K, DT, 16>(src, dst, count, elem_base, keys, nkeys, stamp, s);
      default: return run_split<K, DT, 32>(src, dst, count, elem_base, keys, nkeys, stamp, s);
    }
  }
  const Shape sh = pick_shape(W, nkeys, count / VT<K>::EPV);
  if constexpr (8 / W >= 8) {
    if (sh.u == 8 && !fill) return run_vec_u<K, DT, 8>(src, dst, count, elem_base, keys, nkeys, stamp, s, sh.bps, nullptr, grid_cap);
  }
  if constexpr (8 / W >= 4) {
    if (sh.u >= 4) return run_vec_u<K, DT, 4>(src, dst, count, elem_base, keys, nkeys, stamp, s, sh.bps, fill, grid_cap);
  }
  if (sh.u == 1) return run_vec_u<K, DT, 1>(src, dst, count, elem_base, keys, nkeys, stamp, s, sh.bps, fill, grid_cap);
  return run_vec_u<K, DT, 2>(src, dst, count, elem_base, keys, nkeys, stamp, s, sh.bps, fill, grid_cap);
}

template <int DT>
cudaError_t run_scalar(const void* src, void* dst, uint64_t count, uint64_t elem_base,
                       const uint32_t* keys, uint32_t nkeys, int64_t* stamp, cudaStream_t s) {
  const uint64_t blocks = std::max<uint64_t>(
      1, std::min<uint64_t>((count + kThreads - 1) / kThreads, static_cast<uint64_t>(sm_count()) * 8));
  if (const cudaError_t e = fit_smem(synth_reduce_scalar<DT>, static_cast<size_t>(nkeys) * 8)) return e;
  synth_reduce_scalar<DT><<<static_cast<unsigned>(blocks), kThreads, static_cast<size_t>(nkeys) * 8, s>>>(
      src, dst, count, elem_base, keys, nkeys, stamp);
  return cudaGetLastError();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

cudaError_t launch_synth_reduce(int dtype, const void* src, void* dst, uint64_t count,
                                uint64_t elem_base, const uint32_t* d_keys, uint32_t nkeys,
                                int64_t* stamp, cudaStream_t s, int* launches, CacheRef cache, uint32_t grid_cap) {
  if (nkeys > kMaxKeys) return cudaErrorInvalidValue;
  if (count == 0) return cudaSuccess;
  if (cache.ptr) {
    // callers route only the vector kinds, aligned, word-aligned element offsets
    if (!aligned16(src) || !aligned16(dst) || elem_base % 4 != 0 || nkeys == 0) return cudaErrorInvalidValue;
    const bool words = dtype == cemuInt32 || dtype == cemuUint32;
    if (words && cache.kind != kCacheWide32) return cudaErrorInvalidValue;
    ++*launches;
    switch (dtype) {
      case cemuFloat32: return run_vec_cached<kF32, cemuFloat32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache, grid_cap);
      case cemuBfloat16: return run_vec_cached<kBF16, cemuBfloat16>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache, grid_cap);
      case cemuFloat16: return run_vec_cached<kF16, cemuFloat16>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache, grid_cap);
      case cemuUint8: return run_vec_cached<kU8, cemuUint8>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache, grid_cap);
      case cemuInt8: return run_vec_cached<kU8, cemuInt8>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache, grid_cap);
      case cemuInt32: return run_vec_cached<kI32, cemuInt32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache, grid_cap);
      case cemuUint32: return run_vec_cached<kI32, cemuUint32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache, grid_cap);
      default: --*launches; return cudaErrorInvalidValue;
    }
  }
  ++*launches;
  // vector path: 16-byte aligned pointers, payload words aligned to vectors,
  // at least one emulated peer (the vector kernels seed their sums from it)
  const bool al = aligned16(src) && aligned16(dst) && nkeys > 0;
  const bool word_al = (elem_base % 4) == 0;
  switch (dtype) {
    case cemuFloat32:
      if (al && word_al) return run_vec<kF32, cemuFloat32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, nullptr, grid_cap);
      return run_scalar<cemuFloat32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s);
    case cemuBfloat16:
      if (al && word_al) return run_vec<kBF16, cemuBfloat16>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, nullptr, grid_cap);
      return run_scalar<cemuBfloat16>(src, dst, count, elem_base, d_keys, nkeys, stamp, s);
    case cemuFloat16:
      if (al && word_al) return run_vec<kF16, cemuFloat16>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, nullptr, grid_cap);
      return run_scalar<cemuFloat16>(src, dst, count, elem_base, d_keys, nkeys, stamp, s);
    case cemuUint8:
      if (al && word_al) return run_vec<kU8, cemuUint8>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, nullptr, grid_cap);
      return run_scalar<cemuUint8>(src, dst, count, elem_base, d_keys, nkeys, stamp, s);
    case cemuInt8:
      if (al && word_al) return run_vec<kU8, cemuInt8>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, nullptr, grid_cap);
      return run_scalar<cemuInt8>(src, dst, count, elem_base, d_keys, nkeys, stamp, s);
    case cemuInt32:
      if (al) return run_vec<kI32, cemuInt32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, nullptr, grid_cap);
      return run_scalar<cemuInt32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s);
    case cemuUint32:
      if (al) return run_vec<kI32, cemuUint32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, nullptr, grid_cap);
      return run_scalar<cemuUint32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s);
    case cemuInt64: return run_scalar<cemuInt64>(src, dst, count, elem_base, d_keys, nkeys, stamp, s);
    case cemuUint64: return run_scalar<cemuUint64>(src, dst, count, elem_base, d_keys, nkeys, stamp, s);
    case cemuFloat64: return run_scalar<cemuFloat64>(src, dst, count, elem_base, d_keys, nkeys, stamp, s);
    default: --*launches; return cudaErrorInvalidValue;
  }
}

cudaError_t launch_synth_reduce_filling(int dtype, const void* src, void* dst, uint64_t count, uint64_t elem_base,
                                        const uint32_t* d_keys, uint32_t nkeys, int64_t* stamp, cudaStream_t s,
                                        int* launches, CacheRef cache, uint32_t grid_cap) {
  const bool words = dtype == cemuInt32 || dtype == cemuUint32;
  if (!cache.ptr || count == 0 || nkeys == 0 || !aligned16(src) || !aligned16(dst) || elem_base % 4 != 0 ||
      (words ? cache.kind != kCacheWide32 : (cache.kind != kCacheLanes16 || nkeys > 256))) {
    return cudaErrorInvalidValue;
  }
  {
    // buffers small enough for the peer-split kernels (which have no
    // filling variant): the entries first, then the cached fold
    const uint64_t ev = words || dtype == cemuFloat32 ? 4 : (dtype == cemuUint8 || dtype == cemuInt8 ? 16 : 8);
    if (split_ways(words, nkeys, count / ev)) {
      if (stamp) {  // the call starts with the fill
        if (const cudaError_t e = launch_stamp(stamp, s, launches)) return e;
        stamp = nullptr;
      }
      if (const cudaError_t e = launch_synth_cache_fill(words, elem_base, count, d_keys, nkeys, cache, s, launches)) {
        return e;
      }
      return launch_synth_reduce(dtype, src, dst, count, elem_base, d_keys, nkeys, stamp, s, launches, cache, grid_cap);
    }
  }
  ++*launches;
  cudaError_t e = cudaErrorInvalidValue;
  uint32_t epv = 4;
  switch (dtype) {
    case cemuFloat32: e = run_vec<kF32, cemuFloat32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache.ptr, grid_cap); epv = 4; break;
    case cemuBfloat16: e = run_vec<kBF16, cemuBfloat16>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache.ptr, grid_cap); epv = 8; break;
    case cemuFloat16: e = run_vec<kF16, cemuFloat16>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache.ptr, grid_cap); epv = 8; break;
    case cemuUint8: e = run_vec<kU8, cemuUint8>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache.ptr, grid_cap); epv = 16; break;
    case cemuInt8: e = run_vec<kU8, cemuInt8>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache.ptr, grid_cap); epv = 16; break;
    case cemuInt32: e = run_vec<kI32, cemuInt32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache.ptr, grid_cap); epv = 4; break;
    case cemuUint32: e = run_vec<kI32, cemuUint32>(src, dst, count, elem_base, d_keys, nkeys, stamp, s, cache.ptr, grid_cap); epv = 4; break;
    default: break;
  }
  if (e != cudaSuccess) {
    --*launches;
    return e;
  }
  // the ragged tail's entries (elements after the last vector): a small fill
  const uint64_t done = count / epv * epv;
  if (done < count) return launch_synth_cache_fill(words, elem_base + done, count - done, d_keys, nkeys, cache, s, launches);
  return cudaSuccess;
}

cudaError_t launch_synth_cache_fill(bool words, uint64_t elem_base, uint64_t count, const uint32_t* d_keys,
                                    uint32_t nkeys, CacheRef cache, cudaStream_t s, int* launches) {
  if (count == 0) return cudaSuccess;
  if (!cache.ptr || nkeys == 0 || nkeys > kMaxKeys || (words && cache.kind != kCacheWide32)) {
    return cudaErrorInvalidValue;
  }
  constexpr int U = 2;
  const uint64_t wb = words ? elem_base : elem_base / 4;
  const uint64_t we = words ? elem_base + count : (elem_base + count + 3) / 4;
  const uint64_t per_block = static_cast<uint64_t>(kThreads) * U * 4;
  const uint64_t grid = (we - wb + per_block - 1) / per_block;
  if (grid > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  const size_t smem = static_cast<size_t>(nkeys) * 8;
  auto kern = words ? synth_cache_fill<U, 2>
                    : (cache.kind == kCacheLanes16      ? synth_cache_fill<U, 0>
                       : cache.kind == kCacheCentered16 ? synth_cache_fill<U, 3>
                                                        : synth_cache_fill<U, 1>);
  if (const cudaError_t e = fit_smem(kern, smem)) return e;
  ++*launches;
  kern<<<static_cast<unsigned>(grid), kThreads, smem, s>>>(wb, we, d_keys, nkeys, cache.ptr, 1u, cache.esc);
  return cudaGetLastError();
}

namespace {
template <int K>
cudaError_t fill_vec(void* dst, uint64_t block_elems, const uint32_t* idx, const uint32_t* keys,
                     uint32_t nblocks, uint32_t index0, uint32_t key0, const void* own,
                     uint32_t own_index, int64_t* stamp, cudaStream_t s, uint64_t elem_base) {
  const uint64_t nvec = block_elems / VT<K>::EPV;
  const uint32_t ny = nblocks + (own ? 1 : 0);
  // Address-ordered tiles, 4 vectors per thread: the fill then runs at the
  // write-stream ceiling -- 1 GiB allgather at world 8 in 0.128 ms (7.3 TB/s
  // written) vs 0.153 ms for the 2-D persistent grid below, which remains
  // for grids beyond 2^31 blocks (profiles/r01_fill_tiled.txt)
  {
    constexpr int U = 4;
    const uint64_t tiles = (nvec + kThreads * U - 1) / (kThreads * U);
    if (tiles * ny < 0x7FFFFFFFull) {
      synth_fill_tiled<K, U><<<static_cast<unsigned>(tiles * ny), kThreads, 0, s>>>(
          static_cast<uint4*>(dst), nvec, tiles, idx, keys, nblocks, index0, key0, static_cast<const uint4*>(own),
          own_index, stamp, VT<K>::kWords ? elem_base : elem_base / 4);
      return cudaGetLastError();
    }
  }
  const uint64_t want = (nvec + kThreads - 1) / kThreads;
  const uint64_t cap = std::max<uint64_t>(1, static_cast<uint64_t>(sm_count()) * 8 / std::max<uint32_t>(ny, 1));
  const unsigned gx = static_cast<unsigned>(std::max<uint64_t>(1, std::min(want, cap)));
  synth_fill_vec<K><<<dim3(gx, ny), kThreads, 0, s>>>(static_cast<uint4*>(dst), nvec, idx, keys, nblocks,
                                                      index0, key0, static_cast<const uint4*>(own),
                                                      own_index, stamp,
                                                      VT<K>::kWords ? elem_base : elem_base / 4);
  return cudaGetLastError();
}

template <int DT>
cudaError_t fill_scalar(void* dst, uint64_t block_elems, const uint32_t* idx, const uint32_t* keys,
                        uint32_t nblocks, uint32_t index0, uint32_t key0, const void* own,
                        uint32_t own_index, int64_t* stamp, cudaStream_t s, int es, uint64_t elem_base) {
  const uint32_t ny = nblocks + (own ? 1 : 0);
  const uint64_t want = (block_elems * es + kThreads - 1) / kThreads;
  const uint64_t cap = std::max<uint64_t>(1, static_cast<uint64_t>(sm_count()) * 8 / std::max<uint32_t>(ny, 1));
  const unsigned gx = static_cast<unsigned>(std::max<uint64_t>(1, std::min(want, cap)));
  synth_fill_scalar<DT><<<dim3(gx, ny), kThreads, 0, s>>>(dst, block_elems, idx, keys, nblocks, index0,
                                                          key0, own, own_index, stamp, es, elem_base);
  return cudaGetLastError();
}

int dsize(int dt) {
  switch (dt) {
    case cemuInt8: case cemuUint8: return 1;
    case cemuFloat16: case cemuBfloat16: return 2;
    case cemuInt32: case cemuUint32: case cemuFloat32: return 4;
    default: return 8;
  }
}
}  // namespace

cudaError_t launch_synth_fill(int dtype, void* dst, uint64_t block_elems, const uint32_t* d_index,
                              const uint32_t* d_keys, uint32_t nblocks, uint32_t index0,
                              uint32_t key0, const void* own_src, uint32_t own_index,
                              int64_t* stamp, cudaStream_t s, int* launches, uint64_t elem_base) {
  if (block_elems == 0 || (nblocks == 0 && !own_src)) return cudaSuccess;
  if (nblocks + 1 > 65535) return cudaErrorInvalidValue;
  ++*launches;
  const int es = dsize(dtype);
  const bool word_kind = dtype == cemuInt32 || dtype == cemuUint32;
  const bool al = aligned16(dst) && (!own_src || aligned16(own_src)) && (block_elems * es) % 16 == 0 &&
                  (word_kind || elem_base % 4 == 0);
  switch (dtype) {
    case cemuFloat32:
      if (al) return fill_vec<kF32>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, elem_base);
      return fill_scalar<cemuFloat32>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, es, elem_base);
    case cemuBfloat16:
      if (al) return fill_vec<kBF16>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, elem_base);
      return fill_scalar<cemuBfloat16>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, es, elem_base);
    case cemuFloat16:
      if (al) return fill_vec<kF16>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, elem_base);
      return fill_scalar<cemuFloat16>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, es, elem_base);
    case cemuInt8: case cemuUint8:
      if (al) return fill_vec<kU8>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, elem_base);
      return fill_scalar<cemuUint8>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, es, elem_base);
    case cemuInt32: case cemuUint32:
      if (al) return fill_vec<kI32>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, elem_base);
      return fill_scalar<cemuUint32>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, es, elem_base);
    case cemuInt64: case cemuUint64:
      return fill_scalar<cemuUint64>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, es, elem_base);
    case cemuFloat64:
      return fill_scalar<cemuFloat64>(dst, block_elems, d_index, d_keys, nblocks, index0, key0, own_src, own_index, stamp, s, es, elem_base);
    default: --*launches; return cudaErrorInvalidValue;
  }
}

namespace {
// Launch shape of the fused kernel: U vectors per thread per tile, blocks
// per SM (CEMU_FUSED_U / CEMU_FUSED_BPS override, tuning only).
int fused_env(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

template <int K, int DT, int KMAX, int U>
cudaError_t fused_ku(const FusedArgs& a, cudaStream_t s) {
  static const int bps = std::max(1, fused_env("CEMU_FUSED_BPS", 4));
  const int mode = peer_mode(VT<K>::kWords, a.nkeys);
  auto kern = mode == kGroups ? fused_allreduce_vec<K, DT, KMAX, U, kGroups>
              : mode == kSeed1 ? fused_allreduce_vec<K, DT, KMAX, U, kSeed1>
                               : fused_allreduce_vec<K, DT, KMAX, U, kSeed2>;
  size_t smem = (static_cast<size_t>(a.nkeys) + 1) * 8;
  if (a.cache && a.cache_kind == kCacheWide32) {
    kern = fused_allreduce_vec<K, DT, KMAX, U, kCache32>;
    smem = 0;
  }
  if constexpr (!VT<K>::kWords) {
    if (a.cache && a.cache_kind == kCacheLanes16) {
      kern = fused_allreduce_vec<K, DT, KMAX, U, kCache16>;
      smem = 0;
    }
    if (a.cache && a.cache_kind == kCacheCentered16) {
      kern = a.cache_clean ? fused_allreduce_vec<K, DT, KMAX, U, kCacheC16F> : fused_allreduce_vec<K, DT, KMAX, U, kCacheC16>;
      smem = 0;
    }
  }
  const uint64_t nvec = a.v_end - a.v_begin;
  const uint64_t tiles = (nvec + static_cast<uint64_t>(U) * kThreads - 1) / (static_cast<uint64_t>(U) * kThreads);
  // persistent: NVLink-bound, and every CTA passes the start barrier (one
  // tile per block measured 1.64 -> 2.10 ms for the 1 GiB k=2 allreduce)
  const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(tiles, static_cast<uint64_t>(sm_count()) * bps));
  if (const cudaError_t e = fit_smem(kern, smem)) return e;
  kern<<<static_cast<unsigned>(grid), kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

template <int K, int DT, int KMAX>
cudaError_t fused_k(const FusedArgs& a, cudaStream_t s) {
  static const int u = fused_env("CEMU_FUSED_U", 2);
  if constexpr (KMAX <= 4 && VT<K>::WPV == 1) {
    if (u == 4) return fused_ku<K, DT, KMAX, 4>(a, s);
  }
  return fused_ku<K, DT, KMAX, 2>(a, s);
}

template <int K, int DT>
cudaError_t fused_kind(const FusedArgs& a, cudaStream_t s) {
  // CEMU_FUSED_KMAX=8 runs the 8-GPU instantiation for any k (lets boxes
  // with fewer GPUs exercise the code an 8-GPU job runs)
  static const int force = fused_env("CEMU_FUSED_KMAX", 0);
  if (force != 8) {
    if (a.k <= 2) return fused_k<K, DT, 2>(a, s);
    if (a.k <= 4) return fused_k<K, DT, 4>(a, s);
  }
  return fused_k<K, DT, 8>(a, s);
}
}  // namespace

cudaError_t launch_fused_allreduce(int dtype, const FusedArgs& a, cudaStream_t s, int* launches) {
  if (a.k < 2 || a.k > kMaxReal || a.nkeys == 0 || a.nkeys > kMaxKeys) return cudaErrorInvalidValue;
  ++*launches;
  switch (dtype) {
    case cemuFloat32: return fused_kind<kF32, cemuFloat32>(a, s);
    case cemuBfloat16: return fused_kind<kBF16, cemuBfloat16>(a, s);
    case cemuFloat16: return fused_kind<kF16, cemuFloat16>(a, s);
    case cemuUint8: return fused_kind<kU8, cemuUint8>(a, s);
    case cemuInt8: return fused_kind<kU8, cemuInt8>(a, s);
    case cemuInt32: return fused_kind<kI32, cemuInt32>(a, s);
    case cemuUint32: return fused_kind<kI32, cemuUint32>(a, s);
    default: --*launches; return cudaErrorNotSupported;
  }
}

cudaError_t launch_peer_barrier(const FusedArgs& a, int phase, cudaStream_t s, int* launches) {
  if (a.k < 2 || a.k > 32) return cudaErrorInvalidValue;
  ++*launches;
  peer_barrier_kernel<<<1, 32, 0, s>>>(a, phase);
  return cudaGetLastError();
}

cudaError_t launch_fused_allgather(int dtype, const FusedGatherArgs& a, cudaStream_t s, int* launches) {
  if (a.k < 2 || a.k > kMaxReal) return cudaErrorInvalidValue;
  // NVLink push CTAs vs local synthesis CTAs, split by the bytes each writes
  // (k destinations of the own block vs the emulated blocks): measured 24-27%
  // faster than an even split at 1 GiB (k = 2: 0.295 -> 0.225 ms, k = 4:
  // 0.369 -> 0.270 ms), with 8 CTAs per SM (write streams need many in flight)
  const uint64_t push_vecs = a.block_vecs;
  const uint64_t synth_vecs = static_cast<uint64_t>(a.nvirt) * a.block_vecs;
  static const int per_sm = std::max(1, fused_env("CEMU_FUSED_AG_CTAS", 8));
  const uint64_t total_ctas = static_cast<uint64_t>(sm_count()) * per_sm;
  const uint64_t share = total_ctas * static_cast<uint64_t>(a.k) / (static_cast<uint64_t>(a.k) + a.nvirt);
  uint64_t push = std::max<uint64_t>(1, std::min<uint64_t>((push_vecs + kThreads - 1) / kThreads,
                                                           std::max<uint64_t>(share, 1)));
  uint64_t synth = synth_vecs ? std::max<uint64_t>(1, std::min<uint64_t>((synth_vecs + kThreads - 1) / kThreads,
                                                                          total_ctas - push))
                              : 0;
  ++*launches;
  const unsigned grid = static_cast<unsigned>(push + synth);
  switch (dtype) {
    case cemuFloat32: fused_allgather_vec<kF32><<<grid, kThreads, 0, s>>>(a, static_cast<uint32_t>(push)); break;
    case cemuBfloat16: fused_allgather_vec<kBF16><<<grid, kThreads, 0, s>>>(a, static_cast<uint32_t>(push)); break;
    case cemuFloat16: fused_allgather_vec<kF16><<<grid, kThreads, 0, s>>>(a, static_cast<uint32_t>(push)); break;
    case cemuInt8: case cemuUint8: fused_allgather_vec<kU8><<<grid, kThreads, 0, s>>>(a, static_cast<uint32_t>(push)); break;
    case cemuInt32: case cemuUint32:
      fused_allgather_vec<kI32><<<grid, kThreads, 0, s>>>(a, static_cast<uint32_t>(push));
      break;
    default: --*launches; return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}

// Wire-mode fold of a received DATA payload (collective.cpp:343-350):
// int32 lanes (wrapping) when the plan's elem_size is 4, bytes otherwise.
__global__ void wire_fold_kernel(uint8_t* dst, const uint8_t* src, uint64_t bytes, int words) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (words) {
    auto* d = reinterpret_cast<uint32_t*>(dst);
    const auto* q = reinterpret_cast<const uint32_t*>(src);
    for (uint64_t i = t0; i < bytes / 4; i += stride) d[i] += q[i];
  } else {
    for (uint64_t i = t0; i < bytes; i += stride) dst[i] = static_cast<uint8_t>(dst[i] + src[i]);
  }
}

cudaError_t launch_wire_fold(void* dst, const void* src, uint64_t bytes, bool words, cudaStream_t s,
                             int* launches) {
  if (bytes == 0) return cudaSuccess;
  ++*launches;
  const uint64_t units = words ? bytes / 4 : bytes;
  const unsigned grid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>((units + kThreads - 1) / kThreads, sm_count() * 8ull)));
  wire_fold_kernel<<<grid, kThreads, 0, s>>>(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), bytes,
                                             words ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_stamp(int64_t* slot, cudaStream_t s, int* launches) {
  ++*launches;
  stamp_kernel<<<1, 1, 0, s>>>(slot);
  return cudaGetLastError();
}

cudaError_t launch_spin_ns(int64_t ns, cudaStream_t s, int* launches, int64_t* chain, bool resync) {
  if (ns <= 0 && !chain) return cudaSuccess;
  ++*launches;
  spin_ns_kernel<<<1, 1, 0, s>>>(ns, chain, resync ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_chain_join(int64_t* chain, const int64_t* other, cudaStream_t s, int* launches) {
  ++*launches;
  chain_join_kernel<<<1, 1, 0, s>>>(chain, other);
  return cudaGetLastError();
}

int64_t queue_gap_ns() {
  static const int64_t gap = [] {
    const char* e = std::getenv("CEMU_QUEUE_GAP_US");
    return e ? std::max<int64_t>(0, std::atoll(e)) * 1000 : int64_t{0};
  }();
  return gap;
}

cudaError_t launch_footprint(unsigned long long* start, int64_t lat_ns, int ctas, int smem, int active,
                             cudaStream_t s, int* launches) {
  if (ctas <= 0) return cudaSuccess;
  if (smem > 48 * 1024) {
    if (const cudaError_t e = cudaFuncSetAttribute(footprint_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   smem)) {
      return e;
    }
  }
  if (const cudaError_t e = cudaMemsetAsync(start, 0, sizeof *start, s)) return e;
  ++*launches;
  footprint_kernel<<<ctas, kHoldThreads, static_cast<size_t>(std::max(0, smem)), s>>>(start, lat_ns, active);
  return cudaGetLastError();
}

// Loads the delay path's kernels now (CUDA lazy loading would otherwise
// load each at its first launch -- inside the first delayed call's wait).
cudaError_t preload_delay_kernels() {
  cudaFuncAttributes a;
  for (const void* f : {reinterpret_cast<const void*>(delay_spin_kernel),
                        reinterpret_cast<const void*>(delay_spin_inline_kernel),
                        reinterpret_cast<const void*>(footprint_kernel),
                        reinterpret_cast<const void*>(stamp_kernel)}) {
    if (const cudaError_t e = cudaFuncGetAttributes(&a, f)) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_delay_spin(const DelayLaunch& d, int64_t* slot, cudaStream_t s, int* launches,
                              const InlineOffsets* offs) {
  ++*launches;
  if (offs && d.k > static_cast<uint32_t>(kInlineOffsets)) return cudaErrorInvalidValue;
  if (offs) {
    if (d.k > static_cast<uint32_t>(kInlineOffsets)) return cudaErrorInvalidValue;
    delay_spin_inline_kernel<<<1, kThreads, 0, s>>>(d, slot, *offs);
  } else {
    delay_spin_kernel<<<1, kThreads, 0, s>>>(d, slot);
  }
  return cudaGetLastError();
}

}  // namespace cemu_b200
