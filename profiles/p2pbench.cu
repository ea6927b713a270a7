// NVLink P2P: pull (remote loads) vs push (remote stores) vs mixed, both GPUs at once
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void copyk(const uint4* __restrict__ s, uint4* d, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) d[i] = s[i];
}
struct u8x { uint32_t a[8]; };
__device__ __forceinline__ u8x ld8(const u8x* p) {
  u8x v; asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(v.a[0]), "=r"(v.a[1]), "=r"(v.a[2]), "=r"(v.a[3]), "=r"(v.a[4]), "=r"(v.a[5]), "=r"(v.a[6]), "=r"(v.a[7]) : "l"(p)); return v;
}
__device__ __forceinline__ void st8(u8x* p, u8x v) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(v.a[0]), "r"(v.a[1]), "r"(v.a[2]), "r"(v.a[3]), "r"(v.a[4]), "r"(v.a[5]), "r"(v.a[6]), "r"(v.a[7]) : "memory");
}
__global__ void copy8(const u8x* s, u8x* d, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) st8(d + i, ld8(s + i));
}
__global__ void mix8(const u8x* peer_src, u8x* local_dst, const u8x* local_src, u8x* peer_dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    st8(local_dst + i, ld8(peer_src + i));
    st8(peer_dst + i, ld8(local_src + i));
  }
}
// mixed: pull half from peer into local, push other half from local to peer
__global__ void mixk(const uint4* peer_src, uint4* local_dst, const uint4* local_src, uint4* peer_dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    local_dst[i] = peer_src[i];
    peer_dst[i] = local_src[i];
  }
}
int main() {
  const size_t bytes = 512ull << 20;  // per direction per GPU
  void *a[2], *b[2], *c[2];
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g)); CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&a[g], bytes)); CK(cudaMalloc(&b[g], bytes)); CK(cudaMalloc(&c[g], bytes));
    CK(cudaMemset(a[g], 1, bytes));
  }
  const uint64_t n = bytes / 16;
  cudaStream_t st[2]; cudaEvent_t e0[2], e1[2];
  for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaStreamCreate(&st[g]); cudaEventCreate(&e0[g]); cudaEventCreate(&e1[g]); }
  auto run = [&](const char* name, auto launch, double dir_bytes) {
    for (int it = 0; it < 3; ++it) for (int g = 0; g < 2; ++g) { cudaSetDevice(g); launch(g); }
    for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaDeviceSynchronize(); }
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaEventRecord(e0[g], st[g]); launch(g); cudaEventRecord(e1[g], st[g]); }
      float worst = 0;
      for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaEventSynchronize(e1[g]); float ms; cudaEventElapsedTime(&ms, e0[g], e1[g]); if (ms > worst) worst = ms; }
      if (worst < best) best = worst;
    }
    printf("%-40s %.3f ms  %.1f GB/s per direction per GPU\n", name, best, dir_bytes / best / 1e6);
  };
  for (int bps : {2, 4, 8}) {
    char nm[80];
    snprintf(nm, 80, "pull (remote load) bps%d", bps);
    run(nm, [&](int g) { copyk<<<sms * bps, 256, 0, st[g]>>>((const uint4*)a[1 - g], (uint4*)b[g], n); }, (double)bytes);
    snprintf(nm, 80, "push (remote store) bps%d", bps);
    run(nm, [&](int g) { copyk<<<sms * bps, 256, 0, st[g]>>>((const uint4*)a[g], (uint4*)b[1 - g], n); }, (double)bytes);
    snprintf(nm, 80, "mixed pull+push (half each) bps%d", bps);
    run(nm, [&](int g) { mixk<<<sms * bps, 256, 0, st[g]>>>((const uint4*)a[1 - g], (uint4*)b[g], (const uint4*)c[g], (uint4*)c[1 - g], n / 2); }, (double)bytes);
  }
  const uint64_t n8 = bytes / 32;
  for (int bps : {4, 8}) {
    char nm[80];
    snprintf(nm, 80, "v8 pull bps%d", bps);
    run(nm, [&](int g) { copy8<<<sms * bps, 256, 0, st[g]>>>((const u8x*)a[1 - g], (u8x*)b[g], n8); }, (double)bytes);
    snprintf(nm, 80, "v8 push bps%d", bps);
    run(nm, [&](int g) { copy8<<<sms * bps, 256, 0, st[g]>>>((const u8x*)a[g], (u8x*)b[1 - g], n8); }, (double)bytes);
    snprintf(nm, 80, "v8 mixed bps%d", bps);
    run(nm, [&](int g) { mix8<<<sms * bps, 256, 0, st[g]>>>((const u8x*)a[1 - g], (u8x*)b[g], (const u8x*)c[g], (u8x*)c[1 - g], n8 / 2); }, (double)bytes);
  }
  run("cudaMemcpyPeerAsync push", [&](int g) { cudaMemcpyPeerAsync(b[1 - g], 1 - g, a[g], g, bytes, st[g]); }, (double)bytes);
  return 0;
}
