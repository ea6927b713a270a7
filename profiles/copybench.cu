// streaming read+write microbenchmark: what HBM rate can a 1 GiB -> 1 GiB pass reach on B200?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ld4(const uint4* p) {
  uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p)); return v;
}
__device__ __forceinline__ void st4(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
struct u8x { uint32_t a[8]; };
__device__ __forceinline__ u8x ld8(const u8x* p) {
  u8x v; asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(v.a[0]), "=r"(v.a[1]), "=r"(v.a[2]), "=r"(v.a[3]), "=r"(v.a[4]), "=r"(v.a[5]), "=r"(v.a[6]), "=r"(v.a[7]) : "l"(p)); return v;
}
__device__ __forceinline__ void st8(u8x* p, u8x v) {
  asm volatile("st.global.cs.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(v.a[0]), "r"(v.a[1]), "r"(v.a[2]), "r"(v.a[3]), "r"(v.a[4]), "r"(v.a[5]), "r"(v.a[6]), "r"(v.a[7]) : "memory");
}
template <int U>
__global__ void __launch_bounds__(256) k4(const uint4* __restrict__ s, uint4* d, uint64_t n) {
  const uint64_t tile = 256ull * U;
  for (uint64_t b = blockIdx.x * tile; b < n; b += gridDim.x * tile) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { uint64_t v = b + u * 256 + threadIdx.x; if (v < n) x[u] = ld4(s + v); }
#pragma unroll
    for (int u = 0; u < U; ++u) { uint64_t v = b + u * 256 + threadIdx.x; if (v < n) { x[u].x += 1; st4(d + v, x[u]); } }
  }
}
template <int U>
__global__ void __launch_bounds__(256) k8(const u8x* __restrict__ s, u8x* d, uint64_t n) {
  const uint64_t tile = 256ull * U;
  for (uint64_t b = blockIdx.x * tile; b < n; b += gridDim.x * tile) {
    u8x x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { uint64_t v = b + u * 256 + threadIdx.x; if (v < n) x[u] = ld8(s + v); }
#pragma unroll
    for (int u = 0; u < U; ++u) { uint64_t v = b + u * 256 + threadIdx.x; if (v < n) { x[u].a[0] += 1; st8(d + v, x[u]); } }
  }
}
int main() {
  const size_t bytes = 1ull << 30;
  void *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes)); CK(cudaMemset(a, 1, bytes));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 10; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    cudaError_t e = cudaGetLastError();
    printf("%-28s %.4f ms  %.1f GB/s %s\n", name, best, 2.0 * bytes / best / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  run("cudaMemcpy D2D", [&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); });
  const uint64_t n4 = bytes / 16, n8 = bytes / 32;
  for (int bps : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "v4 U2 bps%d", bps); run(nm, [&] { k4<2><<<sms * bps, 256>>>((const uint4*)a, (uint4*)b, n4); });
    snprintf(nm, 64, "v4 U4 bps%d", bps); run(nm, [&] { k4<4><<<sms * bps, 256>>>((const uint4*)a, (uint4*)b, n4); });
    snprintf(nm, 64, "v8 U1 bps%d", bps); run(nm, [&] { k8<1><<<sms * bps, 256>>>((const u8x*)a, (u8x*)b, n8); });
    snprintf(nm, 64, "v8 U2 bps%d", bps); run(nm, [&] { k8<2><<<sms * bps, 256>>>((const u8x*)a, (u8x*)b, n8); });
  }
  // non-persistent: one tile per block
  run("v4 U2 full grid", [&] { k4<2><<<(unsigned)(n4 / 512), 256>>>((const uint4*)a, (uint4*)b, n4); });
  run("v8 U1 full grid", [&] { k8<1><<<(unsigned)(n8 / 256), 256>>>((const u8x*)a, (u8x*)b, n8); });
  return 0;
}
