// NVLink P2P through the SM's bulk-copy (TMA) engine: cp.async.bulk global ->
// shared of a peer GPU's memory (pull) and shared -> global into a peer's
// memory (push), both GPUs at once, against SM-issued loads / stores (round 1:
// profiles/p2pbench.cu) and the copy engines (cudaMemcpyPeerAsync, 768 GB/s).
// Question: do bulk copies' larger NVLink requests reach the copy-engine rate
// from inside a kernel (the fused allreduce's legs)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

// role per block: 0 = copy tiles src -> dst.  A mixed run launches two
// grids' worth of blocks: the first `split` blocks pull, the rest push.
template <int TILE, int NS>
__global__ void __launch_bounds__(32) tma_copy2(const uint8_t* __restrict__ s0, uint8_t* d0, const uint8_t* __restrict__ s1,
                                                uint8_t* d1, uint64_t ntiles, uint32_t split) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[NS];
  if (threadIdx.x != 0) return;
  const bool second = blockIdx.x >= split;
  const uint8_t* src = second ? s1 : s0;
  uint8_t* dst = second ? d1 : d0;
  const uint64_t first = second ? blockIdx.x - split : blockIdx.x;
  const uint64_t stride = second ? gridDim.x - split : split;
  for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&mbar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[NS] = {0};
  auto issue = [&](uint64_t t, int s) {
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar[s]);
    const uint32_t sm = (uint32_t)__cvta_generic_to_shared(smem + s * TILE);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(TILE) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(sm), "l"(src + t * TILE), "r"(TILE), "r"(mb) : "memory");
  };
  int s = 0;
  uint64_t t = first;
  for (int k = 0; k < NS && t + (uint64_t)k * stride < ntiles; ++k) issue(t + (uint64_t)k * stride, k);
  for (; t < ntiles; t += stride) {
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar[s]);
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(mb), "r"(phase[s]) : "memory");
    }
    phase[s] ^= 1;
    const uint32_t sm = (uint32_t)__cvta_generic_to_shared(smem + s * TILE);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst + t * TILE), "r"(sm), "r"(TILE) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    const uint64_t nt = t + (uint64_t)NS * stride;
    if (nt < ntiles) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue(nt, s);
    }
    s = (s + 1) % NS;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = 512ull << 20;  // per direction per GPU
  uint8_t *a[2], *b[2], *c[2];
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g)); CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&a[g], bytes)); CK(cudaMalloc(&b[g], bytes)); CK(cudaMalloc(&c[g], bytes));
    CK(cudaMemset(a[g], 1, bytes));
  }
  cudaStream_t st[2]; cudaEvent_t e0[2], e1[2];
  for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaStreamCreate(&st[g]); cudaEventCreate(&e0[g]); cudaEventCreate(&e1[g]); }
  auto run = [&](const char* name, auto launch, double dir_bytes) {
    for (int it = 0; it < 3; ++it) for (int g = 0; g < 2; ++g) { cudaSetDevice(g); launch(g); }
    for (int g = 0; g < 2; ++g) { cudaSetDevice(g); if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s failed\n", name); return; } }
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaEventRecord(e0[g], st[g]); launch(g); cudaEventRecord(e1[g], st[g]); }
      float worst = 0;
      for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaEventSynchronize(e1[g]); float ms; cudaEventElapsedTime(&ms, e0[g], e1[g]); if (ms > worst) worst = ms; }
      if (worst < best) best = worst;
    }
    printf("%-44s %.3f ms  %.1f GB/s per direction per GPU\n", name, best, dir_bytes / best / 1e6);
  };
  run("cudaMemcpyPeerAsync push", [&](int g) { cudaMemcpyPeerAsync(b[1 - g], 1 - g, a[g], g, bytes, st[g]); }, (double)bytes);
#define RUNT(T, NS, CPS) { \
    auto k = tma_copy2<T, NS>; \
    for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, T * NS); } \
    const uint64_t nt = bytes / T; const unsigned grid = sms * CPS; char nm[96]; \
    snprintf(nm, 96, "bulk pull tile%dK ns%d cta/sm%d", T / 1024, NS, CPS); \
    run(nm, [&](int g) { k<<<grid, 32, T * NS, st[g]>>>(a[1 - g], b[g], a[1 - g], b[g], nt, grid); }, (double)bytes); \
    snprintf(nm, 96, "bulk push tile%dK ns%d cta/sm%d", T / 1024, NS, CPS); \
    run(nm, [&](int g) { k<<<grid, 32, T * NS, st[g]>>>(a[g], b[1 - g], a[g], b[1 - g], nt, grid); }, (double)bytes); \
    snprintf(nm, 96, "bulk mixed tile%dK ns%d cta/sm%d", T / 1024, NS, CPS); \
    run(nm, [&](int g) { k<<<grid, 32, T * NS, st[g]>>>(a[1 - g], b[g], a[g], c[1 - g], nt / 2, grid / 2); }, (double)bytes); }
  RUNT(16384, 4, 2) RUNT(16384, 4, 4) RUNT(32768, 3, 2) RUNT(32768, 4, 1) RUNT(65536, 3, 1) RUNT(8192, 8, 4) RUNT(4096, 8, 8)
  return 0;
}
