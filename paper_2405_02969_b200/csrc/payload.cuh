// payload.cuh -- the counter-based payload generator shared by host and
// device code.  Its bits are the specification of what an emulated peer
// "sends" (the reference sends zeros: proj/src/transport.cpp:45-47; the
// zero mode reproduces that, the hash mode below replaces it).
//
//   key(seed, rank)   32-bit per-rank key: the splitmix64 finalizer `mix` of
//                     proj/tools/cemu_coll.cpp:22-31 (trial 0), folded to 32.
//   word(key, j)      32-bit word j of the rank's stream:
//                       x  = (key + ctr(j)) * M1        ctr = Weyl counter of j
//                       x ^= x >> 15
//                       x *= key | 1                    key-dependent odd multiplier
//                       x += x >> 16
//                     (key + ctr) * M1 == key*M1 + ctr*M1, so kernels hoist
//                     key*M1 per peer and ctr*M1 per word: per peer-word the
//                     hash is 1 add, 1 xorshift, 1 IMAD, 1 IMAD.HI -- split
//                     across the FMA and ALU pipes.
//   byte(key, e)      byte (e & 3) of word(key, e >> 2).
//
// Element e of a rank's contribution, by datatype:
//   int8/uint8      byte(key, e)
//   int32/uint32    word(key, e)
//   int64/uint64    word(key, 2e) | word(key, 2e+1) << 32
//   fp16/bf16/fp32/fp64   (byte(key, e) - 128) * 2^-7   (dyadic, exact)
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define CEMU_HD __host__ __device__ __forceinline__
#else
#define CEMU_HD inline
#endif

namespace cemu_b200 {

constexpr uint32_t kWeyl = 0x9E3779B9u;
constexpr uint32_t kWeylHi = 0x85EBCA77u;
constexpr uint32_t kMul1 = 0x7FEB352Du;
constexpr float kDyadicScale = 0.0078125f;  // 2^-7

CEMU_HD uint32_t payload_key(uint64_t seed, uint32_t rank) {
  uint64_t h = seed ^ (static_cast<uint64_t>(rank) * 0xbf58476d1ce4e5b9ull);
  h ^= h >> 30;
  h *= 0xbf58476d1ce4e5b9ull;
  h ^= h >> 27;
  h *= 0x94d049bb133111ebull;
  h ^= h >> 31;
  return static_cast<uint32_t>(h ^ (h >> 32));
}

// The per-word counter, premultiplied by M1; kernels hoist it across peers.
CEMU_HD uint32_t payload_c1(uint64_t j) {
  return (static_cast<uint32_t>(j) * kWeyl ^ static_cast<uint32_t>(j >> 32) * kWeylHi) * kMul1;
}

// Per-peer constants: k1 = key * M1, km = key | 1.
CEMU_HD uint32_t payload_k1(uint32_t key) { return key * kMul1; }
CEMU_HD uint32_t payload_km(uint32_t key) { return key | 1u; }

CEMU_HD uint32_t payload_mix(uint32_t k1, uint32_t km, uint32_t c1) {
  uint32_t x = k1 + c1;
  x ^= x >> 15;
  x *= km;
#if defined(__CUDA_ARCH__)
  x = __umulhi(x, 0x10000u) + x;  // x + (x >> 16) as one IMAD.HI (FMA pipe)
#else
  x += x >> 16;
#endif
  return x;
}

CEMU_HD uint32_t payload_word(uint32_t key, uint64_t j) {
  return payload_mix(payload_k1(key), payload_km(key), payload_c1(j));
}

}  // namespace cemu_b200
