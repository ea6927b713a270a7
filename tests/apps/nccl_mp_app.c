/* tests/apps/nccl_mp_app.c -- an ordinary multi-process NCCL program: one
 * process per GPU, the unique id passed through a file.  Run as is it is a
 * real NCCL job; run under
 *   CEMU_CONFIG=job.cfg LD_PRELOAD=libnccl_cemu.so
 * its collectives are the emulated ones (the job config's world contains
 * emulated ranks beside the real ones).
 *
 * MODE selects how the buffers are allocated, as NCCL applications do:
 *   plain     cudaMalloc, not registered
 *   register  cudaMalloc + ncclCommRegister        (nccl.h:243)
 *   window    ncclMemAlloc + ncclCommWindowRegister (nccl.h:130, 251)
 *
 * It allreduces COUNT floats x[i] = ((7i + 13 rank) mod 61 - 30) / 8 out of
 * place, WARM untimed then ITERS timed calls (CUDA events), writes the result
 * (raw float32) to OUT and prints the mean time per call.
 *   usage: nccl_mp_app NRANKS RANK DEVICE COUNT MODE IDFILE OUT ITERS */
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define CK(x) do { if ((x) != 0) { fprintf(stderr, "%s failed: %s\n", #x, ncclGetLastError(NULL)); return 1; } } while (0)
#define CC(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

int main(int argc, char** argv) {
  if (argc != 9) {
    fprintf(stderr, "usage: nccl_mp_app NRANKS RANK DEVICE COUNT MODE IDFILE OUT ITERS\n");
    return 2;
  }
  const int nranks = atoi(argv[1]), rank = atoi(argv[2]), dev = atoi(argv[3]);
  const size_t count = (size_t)atoll(argv[4]);
  const char* mode = argv[5];
  const char* idfile = argv[6];
  const int iters = atoi(argv[8]);
  CC(cudaSetDevice(dev));
  ncclUniqueId id;
  if (rank == 0) {
    CK(ncclGetUniqueId(&id));
    char tmp[4096];
    snprintf(tmp, sizeof tmp, "%s.tmp", idfile);
    FILE* f = fopen(tmp, "wb");
    fwrite(&id, sizeof id, 1, f);
    fclose(f);
    rename(tmp, idfile);
  } else {
    FILE* f = NULL;
    for (int t = 0; t < 6000 && !(f = fopen(idfile, "rb")); ++t) usleep(10000);
    if (!f || fread(&id, sizeof id, 1, f) != 1) { fprintf(stderr, "no unique id in %s\n", idfile); return 1; }
    fclose(f);
  }
  ncclComm_t comm;
  CK(ncclCommInitRank(&comm, nranks, id, rank));
  const size_t bytes = count * sizeof(float);
  float *send = NULL, *recv = NULL;
  void *hs = NULL, *hr = NULL;
  ncclWindow_t ws = NULL, wr = NULL;
  if (!strcmp(mode, "window")) {
    CK(ncclMemAlloc((void**)&send, bytes));
    CK(ncclMemAlloc((void**)&recv, bytes));
    CK(ncclCommWindowRegister(comm, send, bytes, &ws, 0));
    CK(ncclCommWindowRegister(comm, recv, bytes, &wr, 0));
  } else {
    CC(cudaMalloc((void**)&send, bytes));
    CC(cudaMalloc((void**)&recv, bytes));
    if (!strcmp(mode, "register")) {
      CK(ncclCommRegister(comm, send, bytes, &hs));
      CK(ncclCommRegister(comm, recv, bytes, &hr));
    } else if (strcmp(mode, "plain")) {
      fprintf(stderr, "unknown mode %s\n", mode);
      return 2;
    }
  }
  float* h = (float*)malloc(bytes);
  for (size_t i = 0; i < count; ++i) h[i] = (float)((int)((7 * i + 13 * (size_t)rank) % 61) - 30) * 0.125f;
  CC(cudaMemcpy(send, h, bytes, cudaMemcpyHostToDevice));
  cudaStream_t s;
  CC(cudaStreamCreate(&s));
  cudaEvent_t e0, e1;
  CC(cudaEventCreate(&e0));
  CC(cudaEventCreate(&e1));
  for (int i = 0; i < 2; ++i) CK(ncclAllReduce(send, recv, count, ncclFloat32, ncclSum, comm, s));
  CC(cudaStreamSynchronize(s));
  CC(cudaEventRecord(e0, s));
  for (int i = 0; i < iters; ++i) CK(ncclAllReduce(send, recv, count, ncclFloat32, ncclSum, comm, s));
  CC(cudaEventRecord(e1, s));
  CC(cudaStreamSynchronize(s));
  float ms = 0;
  CC(cudaEventElapsedTime(&ms, e0, e1));
  ncclResult_t aerr = ncclSuccess;
  CK(ncclCommGetAsyncError(comm, &aerr));
  CC(cudaMemcpy(h, recv, bytes, cudaMemcpyDeviceToHost));
  FILE* f = fopen(argv[7], "wb");
  fwrite(h, sizeof(float), count, f);
  fclose(f);
  int n = 0;
  CK(ncclCommCount(comm, &n));
  printf("nccl_mp_app: rank %d world %d mode %s bytes %zu ms_per_call %.4f async_error %d\n", rank, n, mode, bytes,
         iters ? ms / iters : 0.0, (int)aerr);
  if (ws) CK(ncclCommWindowDeregister(comm, ws));
  if (wr) CK(ncclCommWindowDeregister(comm, wr));
  if (hs) CK(ncclCommDeregister(comm, hs));
  if (hr) CK(ncclCommDeregister(comm, hr));
  if (!strcmp(mode, "window")) {
    CK(ncclMemFree(send));
    CK(ncclMemFree(recv));
  } else {
    CC(cudaFree(send));
    CC(cudaFree(recv));
  }
  CK(ncclCommDestroy(comm));
  return 0;
}
