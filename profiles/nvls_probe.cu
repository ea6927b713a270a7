// NVLS probe: single process, n GPUs, one multicast object bound to each GPU's
// buffer; allreduce of S bytes per GPU = multimem.ld_reduce of the own 1/n
// shard + multimem.st of the sum to every GPU.  Compared with the fused P2P
// kernel's 2(n-1)/n*S per direction.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)
#define CK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)

__global__ void nvls_allreduce(float* mc_in, float* mc_out, uint64_t v0, uint64_t v1) {
  for (uint64_t v = v0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < v1; v += (uint64_t)gridDim.x * blockDim.x) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc_in + 4 * v) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(mc_out + 4 * v), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
  }
}

int main() {
  int n = 0; CK(cudaGetDeviceCount(&n)); if (n > 8) n = 8;
  CU(cuInit(0));
  const size_t want = 1ull << 30;
  std::vector<CUdevice> dev(n);
  for (int d = 0; d < n; ++d) { CU(cuDeviceGet(&dev[d], d)); CK(cudaSetDevice(d)); CK(cudaFree(0)); }
  int mcs = 0; CU(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev[0]));
  printf("devices %d multicast %d\n", n, mcs);
  CUmulticastObjectProp mp = {};
  mp.numDevices = n; mp.size = want; mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
  size_t mgran = 0; CU(cuMulticastGetGranularity(&mgran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0; size_t agran = 0; CU(cuMemGetAllocationGranularity(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  size_t gran = mgran > agran ? mgran : agran;
  const size_t S = (want + gran - 1) / gran * gran;
  mp.size = S;
  CUmemGenericAllocationHandle mc[2];
  CUdeviceptr mcva[2];
  std::vector<std::vector<CUdeviceptr>> va(2, std::vector<CUdeviceptr>(n));
  std::vector<CUmemAccessDesc> acc(n);
  for (int d = 0; d < n; ++d) { acc[d].location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc[d].location.id = d; acc[d].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE; }
  for (int b = 0; b < 2; ++b) {
    CU(cuMulticastCreate(&mc[b], &mp));
    for (int d = 0; d < n; ++d) CU(cuMulticastAddDevice(mc[b], dev[d]));
    for (int d = 0; d < n; ++d) {
      CK(cudaSetDevice(d));
      ap.location.id = d;
      CUmemGenericAllocationHandle h; CU(cuMemCreate(&h, S, &ap, 0));
      CU(cuMemAddressReserve(&va[b][d], S, gran, 0, 0)); CU(cuMemMap(va[b][d], S, 0, h, 0));
      CU(cuMemSetAccess(va[b][d], S, &acc[d], 1));
      CU(cuMulticastBindMem(mc[b], 0, h, 0, S, 0));
      CK(cudaMemset((void*)va[b][d], 0, S));
    }
    CU(cuMemAddressReserve(&mcva[b], S, gran, 0, 0)); CU(cuMemMap(mcva[b], S, 0, mc[b], 0));
    CU(cuMemSetAccess(mcva[b], S, acc.data(), n));
  }
  // inputs: GPU d holds (d+1)
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    std::vector<float> h(1 << 20, float(d + 1));
    for (size_t off = 0; off < S; off += h.size() * 4) CK(cudaMemcpy((char*)va[0][d] + off, h.data(), std::min(S - off, h.size() * 4), cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());
  }
  const uint64_t nvec = S / 16, per = nvec / n;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<cudaEvent_t> e0(n), e1(n);
  for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]); }
  for (int bps : {2, 4, 8}) {
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
      for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d)); cudaEventRecord(e0[d]);
        nvls_allreduce<<<sms * bps, 256>>>((float*)mcva[0], (float*)mcva[1], per * d, d == n - 1 ? nvec : per * (d + 1));
        cudaEventRecord(e1[d]);
      }
      float worst = 0;
      for (int d = 0; d < n; ++d) { CK(cudaSetDevice(d)); CK(cudaEventSynchronize(e1[d])); float ms; cudaEventElapsedTime(&ms, e0[d], e1[d]); if (ms > worst) worst = ms; }
      if (rep > 0 && worst < best) best = worst;
    }
    float check = 0; CK(cudaSetDevice(n - 1)); CK(cudaMemcpy(&check, (char*)va[1][n - 1] + 16, 4, cudaMemcpyDeviceToHost));
    printf("n=%d bps=%d: 1 GiB allreduce per GPU via NVLS %.3f ms (check %.0f, want %d); per-GPU link bytes/dir S(1+1/n)=%.2f GB -> %.0f GB/s\n",
           n, bps, best, check, n * (n + 1) / 2, S * (1.0 + 1.0 / n) / 1e9, S * (1.0 + 1.0 / n) / (best * 1e6));
  }
  return 0;
}
