/* tests/apps/nccl_app.c -- an ordinary single-process NCCL program (rank 0
 * of NRANKS).  Run as is it needs a real NCCL world; run under
 *   CEMU_CONFIG=job.cfg LD_PRELOAD=libnccl_cemu.so
 * its ncclAllReduce is the emulated collective.  It allreduces COUNT
 * floats x[i] = (i % 97) * 0.25 and writes the result (raw float32) to OUT.
 *   usage: nccl_app NRANKS COUNT OUT */
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { if ((x) != 0) { fprintf(stderr, "%s failed\n", #x); return 1; } } while (0)

int main(int argc, char** argv) {
  if (argc != 4) { fprintf(stderr, "usage: nccl_app NRANKS COUNT OUT\n"); return 2; }
  const int nranks = atoi(argv[1]);
  const size_t count = (size_t)atoll(argv[2]);
  float* h = (float*)malloc(count * sizeof(float));
  for (size_t i = 0; i < count; ++i) h[i] = (float)(i % 97) * 0.25f;
  float* d = NULL;
  CK(cudaSetDevice(0));
  CK(cudaMalloc((void**)&d, count * sizeof(float)));
  CK(cudaMemcpy(d, h, count * sizeof(float), cudaMemcpyHostToDevice));
  ncclUniqueId id;
  ncclComm_t comm;
  int v = 0, n = 0;
  CK(ncclGetVersion(&v));
  CK(ncclGetUniqueId(&id));
  CK(ncclCommInitRank(&comm, nranks, id, 0));
  CK(ncclCommCount(comm, &n));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  CK(ncclAllReduce(d, d, count, ncclFloat32, ncclSum, comm, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaMemcpy(h, d, count * sizeof(float), cudaMemcpyDeviceToHost));
  FILE* f = fopen(argv[3], "wb");
  fwrite(h, sizeof(float), count, f);
  fclose(f);
  printf("nccl_app: version %d, world %d, %zu floats, x[1] = %g\n", v, n, count, (double)h[1]);
  CK(ncclCommDestroy(comm));
  return 0;
}
