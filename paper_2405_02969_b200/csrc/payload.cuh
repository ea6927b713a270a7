// payload.cuh -- the counter-based payload generator shared by host and
// device code.  Its bits are the specification of what an emulated peer
// "sends" (the reference sends zeros: proj/src/transport.cpp:45-47; the
// zero mode reproduces that, the hash mode below replaces it).
//
//   key(seed, rank)   32-bit per-rank key: the splitmix64 finalizer `mix` of
//                     proj/tools/cemu_coll.cpp:22-31 (trial 0), folded to 32.
//   word(key, j)      32-bit word j of the rank's stream: Weyl counter XOR
//                     key, then two multiply/xorshift rounds.
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
constexpr uint32_t kMul2 = 0x846CA68Bu;
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

// The per-word counter; split out so kernels hoist it across peers.
CEMU_HD uint32_t payload_ctr(uint64_t j) {
  return static_cast<uint32_t>(j) * kWeyl ^
         static_cast<uint32_t>(j >> 32) * kWeylHi;
}

CEMU_HD uint32_t payload_mix(uint32_t key, uint32_t ctr) {
  uint32_t x = key ^ ctr;
  x *= kMul1;
  x ^= x >> 15;
  x *= kMul2;
  x ^= x >> 16;
  return x;
}

CEMU_HD uint32_t payload_word(uint32_t key, uint64_t j) {
  return payload_mix(key, payload_ctr(j));
}

}  // namespace cemu_b200
