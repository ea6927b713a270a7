// delay_math.cuh -- the alpha-beta delay model, one source for host and
// device.  On the device every double operation goes through the _rn
// intrinsics so nvcc cannot contract a*b+c into an FMA; on the host the
// translation units are built with -ffp-contract=off.  Both therefore round
// in exactly the source order of proj/src/delay.cpp:5-47 -- the per-step
// floors evaluated on the B200 are bit-identical to the reference's.
#pragma once
#include <cstdint>

#include "cemu_b200.h"

#if defined(__CUDACC__)
#define CEMU_DM_HD __host__ __device__ __forceinline__
#else
#define CEMU_DM_HD inline
#endif

#if defined(__CUDA_ARCH__)
#define DMUL(a, b) __dmul_rn((a), (b))
#define DADD(a, b) __dadd_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))
#else
#define DMUL(a, b) ((a) * (b))
#define DADD(a, b) ((a) + (b))
#define DDIV(a, b) ((a) / (b))
#endif

namespace cemu_b200 {

enum Coll : int32_t { kAllReduce = 0, kAllGather = 1, kReduceScatter = 2, kBroadcast = 3 };

// delay.cpp:5-13: steps*a + 2*frac*m*b + frac*m*g
CEMU_DM_HD double ring_allreduce_us(uint32_t n, uint64_t bytes, double a, double b, double g) {
  const double steps = DMUL(2.0, static_cast<double>(n - 1));
  const double frac = DDIV(static_cast<double>(n - 1), static_cast<double>(n));
  const double m = static_cast<double>(bytes);
  return DADD(DADD(DMUL(steps, a), DMUL(DMUL(DMUL(2.0, frac), m), b)), DMUL(DMUL(frac, m), g));
}

// delay.cpp:15-21: steps*a + steps*m*b
CEMU_DM_HD double ring_allgather_us(uint32_t n, uint64_t bytes, double a, double b) {
  const double steps = static_cast<double>(n - 1);
  const double m = static_cast<double>(bytes);
  return DADD(DMUL(steps, a), DMUL(DMUL(steps, m), b));
}

// NEW: the reduce-scatter half of the ring allreduce
CEMU_DM_HD double ring_reducescatter_us(uint32_t n, uint64_t bytes, double a, double b, double g) {
  const double steps = static_cast<double>(n - 1);
  const double frac = DDIV(static_cast<double>(n - 1), static_cast<double>(n));
  const double m = static_cast<double>(bytes);
  return DADD(DADD(DMUL(steps, a), DMUL(DMUL(frac, m), b)), DMUL(DMUL(frac, m), g));
}

// NEW: pipelined ring broadcast
CEMU_DM_HD double ring_broadcast_us(uint32_t n, uint64_t bytes, double a, double b) {
  const double steps = static_cast<double>(n - 1);
  const double m = static_cast<double>(bytes);
  return DADD(DMUL(steps, a), DMUL(m, b));
}

CEMU_DM_HD uint32_t ceil_log2_u32(uint32_t n) {
  uint32_t d = 0;
  while ((1u << d) < n) ++d;
  return d;
}

// NEW: pipelined double binary tree
CEMU_DM_HD double tree_allreduce_us(uint32_t n, uint64_t bytes, double a, double b, double g) {
  const double steps = DMUL(2.0, static_cast<double>(ceil_log2_u32(n)));
  const double m = static_cast<double>(bytes);
  return DADD(DADD(DMUL(steps, a), DMUL(DMUL(2.0, m), b)), DMUL(m, g));
}

// NEW: tree-scheduled (PAT-style) allgather / reduce-scatter: ceil(log2 n)
// latency terms, the ring's bandwidth term (every byte still crosses once).
CEMU_DM_HD double tree_allgather_us(uint32_t n, uint64_t bytes, double a, double b) {
  const double steps = static_cast<double>(ceil_log2_u32(n));
  const double m = static_cast<double>(bytes);
  return DADD(DMUL(steps, a), DMUL(DMUL(static_cast<double>(n - 1), m), b));
}

CEMU_DM_HD double tree_reducescatter_us(uint32_t n, uint64_t bytes, double a, double b, double g) {
  const double steps = static_cast<double>(ceil_log2_u32(n));
  const double frac = DDIV(static_cast<double>(n - 1), static_cast<double>(n));
  const double m = static_cast<double>(bytes);
  return DADD(DADD(DMUL(steps, a), DMUL(DMUL(frac, m), b)), DMUL(DMUL(frac, m), g));
}

CEMU_DM_HD double tree_broadcast_us(uint32_t n, uint64_t bytes, double a, double b) {
  const double steps = static_cast<double>(ceil_log2_u32(n));
  const double m = static_cast<double>(bytes);
  return DADD(DMUL(steps, a), DMUL(m, b));
}

// NEW: hierarchical ring, N = n / G nodes of G ranks: intra reduce-scatter,
// inter ring over the 1/G shard, intra allgather.
CEMU_DM_HD double hier_us(const cemuDelayModel& M, int coll, uint32_t n, uint64_t bytes) {
  const uint32_t G = M.gpus_per_node ? M.gpus_per_node : 1;
  const uint32_t N = n / G;
  const double ai = M.intra_alpha_us, bi = M.intra_beta_us_per_byte;
  const double ae = M.alpha_us, be = M.beta_us_per_byte, g = M.gamma_us_per_byte;
  const double m = static_cast<double>(bytes);
  const double gm1 = static_cast<double>(G - 1);
  const double fi = DDIV(static_cast<double>(G - 1), static_cast<double>(G));
  const double nm1 = static_cast<double>(N - 1);
  const double fe = DDIV(static_cast<double>(N - 1), static_cast<double>(N));
  const double shard = DDIV(m, static_cast<double>(G));
  switch (coll) {
    case kAllReduce: {
      const double intra_rs = DADD(DADD(DMUL(gm1, ai), DMUL(DMUL(fi, m), bi)), DMUL(DMUL(fi, m), g));
      const double inter_ar = DADD(DADD(DMUL(DMUL(2.0, nm1), ae), DMUL(DMUL(DMUL(2.0, fe), shard), be)),
                                   DMUL(DMUL(fe, shard), g));
      const double intra_ag = DADD(DMUL(gm1, ai), DMUL(DMUL(fi, m), bi));
      return DADD(DADD(intra_rs, inter_ar), intra_ag);
    }
    case kAllGather: {  // m = per-rank block: G parallel inter-node rings, then a node-local gather
      const double inter_ag = DADD(DMUL(nm1, ae), DMUL(DMUL(nm1, m), be));
      const double intra_ag = DADD(DMUL(gm1, ai), DMUL(DMUL(gm1, DMUL(static_cast<double>(N), m)), bi));
      return DADD(inter_ag, intra_ag);
    }
    case kReduceScatter: {
      const double intra_rs = DADD(DADD(DMUL(gm1, ai), DMUL(DMUL(fi, m), bi)), DMUL(DMUL(fi, m), g));
      const double inter_rs = DADD(DADD(DMUL(nm1, ae), DMUL(DMUL(fe, shard), be)), DMUL(DMUL(fe, shard), g));
      return DADD(intra_rs, inter_rs);
    }
    default: {
      const double inter = DADD(DMUL(nm1, ae), DMUL(m, be));
      const double intra = DADD(DMUL(gm1, ai), DMUL(m, bi));
      return DADD(inter, intra);
    }
  }
}

CEMU_DM_HD double model_total_us(const cemuDelayModel& M, int coll, uint32_t n, uint64_t bytes) {
  if (M.algo == 2) return hier_us(M, coll, n, bytes);
  if (M.algo == 1) {
    switch (coll) {
      case kAllReduce: return tree_allreduce_us(n, bytes, M.alpha_us, M.beta_us_per_byte, M.gamma_us_per_byte);
      case kAllGather: return tree_allgather_us(n, bytes, M.alpha_us, M.beta_us_per_byte);
      case kReduceScatter:
        return tree_reducescatter_us(n, bytes, M.alpha_us, M.beta_us_per_byte, M.gamma_us_per_byte);
      default: return tree_broadcast_us(n, bytes, M.alpha_us, M.beta_us_per_byte);
    }
  }
  switch (coll) {
    case kAllReduce: return ring_allreduce_us(n, bytes, M.alpha_us, M.beta_us_per_byte, M.gamma_us_per_byte);
    case kAllGather: return ring_allgather_us(n, bytes, M.alpha_us, M.beta_us_per_byte);
    case kReduceScatter: return ring_reducescatter_us(n, bytes, M.alpha_us, M.beta_us_per_byte, M.gamma_us_per_byte);
    default: return ring_broadcast_us(n, bytes, M.alpha_us, M.beta_us_per_byte);
  }
}

// delay.cpp:23-47; `total` is model_total_us (only used for alpha_beta)
CEMU_DM_HD double release_offset_us(const cemuDelayModel& M, double total, uint32_t j, uint32_t k) {
  double o = 0.0;
  if (M.kind == 1) {
    o = DDIV(DMUL(total, static_cast<double>(j + 1)), static_cast<double>(k));
  } else if (M.kind == 2) {
    o = M.fixed_us;
  }
  if (j == 0) o = DADD(o, M.inject_us);
  return o;
}

}  // namespace cemu_b200
