// 1 GiB read + 1 GiB write with TMA bulk copies (cp.async.bulk) vs plain loads
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int TILE, int NS>
__global__ void __launch_bounds__(32) tma_copy(const uint8_t* __restrict__ src, uint8_t* dst, uint64_t ntiles) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[NS];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NS; ++s) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&mbar[s])));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t first = blockIdx.x, stride = gridDim.x;
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
  for (uint64_t i = 0; t < ntiles; ++i, t += stride) {
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
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // this stage's store has read smem
      issue(nt, s);
    }
    s = (s + 1) % NS;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
int main() {
  const size_t bytes = 1ull << 30; uint8_t *a, *b; cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMemset(a, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto f) {
    for (int i = 0; i < 3; ++i) f(); cudaError_t e = cudaDeviceSynchronize();
    float best = 1e9; for (int r = 0; r < 10; ++r) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    bool ok = true; // spot check
    uint8_t h[16]; cudaMemcpy(h, b + bytes - 16, 16, cudaMemcpyDeviceToHost); for (int i = 0; i < 16; ++i) ok &= h[i] == 1;
    printf("%-30s %.4f ms  %.1f GB/s %s %s\n", name, best, 2.0 * bytes / best / 1e6, ok ? "" : "BAD", e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaMemset(b, 0, bytes);
  };
  run("cudaMemcpy D2D", [&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); });
#define RUN(T, NS, CPS) { auto k = tma_copy<T, NS>; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, T * NS); \
    char nm[64]; snprintf(nm, 64, "tma tile%dK ns%d cta/sm%d", T / 1024, NS, CPS); \
    run(nm, [&] { k<<<sms * CPS, 32, T * NS>>>(a, b, bytes / T); }); }
  RUN(16384, 4, 2) RUN(16384, 4, 4) RUN(32768, 3, 2) RUN(32768, 4, 1) RUN(65536, 3, 1) RUN(8192, 8, 4) RUN(16384, 6, 2)
  return 0;
}
