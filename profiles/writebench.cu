#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void st4(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st4wb(uint4* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
template <bool CS>
__global__ void gs(uint4* d, uint64_t n) {  // grid-stride
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v = make_uint4(i, i, i, i); if (CS) st4(d + i, v); else st4wb(d + i, v);
  }
}
template <bool CS, int U>
__global__ void full(uint4* d, uint64_t n) {  // one tile per block
  const uint64_t b = blockIdx.x * 256ull * U;
#pragma unroll
  for (int u = 0; u < U; ++u) { uint64_t i = b + u * 256 + threadIdx.x; if (i < n) { uint4 v = make_uint4(i, i, i, i); if (CS) st4(d + i, v); else st4wb(d + i, v); } }
}
int main() {
  const size_t bytes = 1ull << 30; void* a; cudaMalloc(&a, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const uint64_t n = bytes / 16;
  auto run = [&](const char* name, auto f) {
    for (int i = 0; i < 3; ++i) f(); cudaDeviceSynchronize();
    float best = 1e9; for (int r = 0; r < 10; ++r) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    printf("%-28s %.4f ms  %.1f GB/s\n", name, best, bytes / best / 1e6);
  };
  run("cudaMemsetAsync", [&] { cudaMemsetAsync(a, 0, bytes); });
  for (int bps : {4, 8, 16}) { char nm[64];
    snprintf(nm, 64, "gs cs bps%d", bps); run(nm, [&] { gs<true><<<sms * bps, 256>>>((uint4*)a, n); });
    snprintf(nm, 64, "gs wb bps%d", bps); run(nm, [&] { gs<false><<<sms * bps, 256>>>((uint4*)a, n); }); }
  run("full cs U1", [&] { full<true, 1><<<(unsigned)(n / 256), 256>>>((uint4*)a, n); });
  run("full cs U4", [&] { full<true, 4><<<(unsigned)(n / 1024), 256>>>((uint4*)a, n); });
  run("full wb U1", [&] { full<false, 1><<<(unsigned)(n / 256), 256>>>((uint4*)a, n); });
  run("full wb U4", [&] { full<false, 4><<<(unsigned)(n / 1024), 256>>>((uint4*)a, n); });
  return 0;
}
