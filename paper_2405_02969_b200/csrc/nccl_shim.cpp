// nccl_shim.cpp -- libnccl_cemu.so: NCCL's own symbols, backed by the
// emulator.  The NeuronaBox paper interposes on NCCL; an
// unmodified NCCL application gets the emulated world with
//   CEMU_CONFIG=job.cfg LD_PRELOAD=libnccl_cemu.so ./app
// nranks passed to ncclCommInitRank must equal the config's world_size and
// the rank must be one of its real ranks.  ncclComm_t is the cemuComm_t;
// datatypes, reduction ops and result codes share NCCL's values.  When the
// job puts several real ranks on this box, libcemu_b200 dlopens the real
// libnccl.so.2 for them (a different soname, so it is not this shim).
#include <cuda_runtime.h>
#include <nccl.h>

#include "cemu_b200.h"

#define CEMU_EXPORT extern "C" __attribute__((visibility("default")))

namespace {
inline cemuComm_t C(ncclComm_t c) { return reinterpret_cast<cemuComm_t>(c); }
inline cemuStream_t S(cudaStream_t s) { return reinterpret_cast<cemuStream_t>(s); }
inline ncclResult_t R(cemuResult_t r) { return static_cast<ncclResult_t>(r); }
}  // namespace

CEMU_EXPORT ncclResult_t ncclGetVersion(int* version) { return R(cemuGetVersion(version)); }

CEMU_EXPORT ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  return R(cemuGetUniqueId(reinterpret_cast<cemuUniqueId*>(id)));
}

CEMU_EXPORT ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  cemuUniqueId u;
  static_assert(sizeof u == sizeof id, "unique id size");
  __builtin_memcpy(&u, &id, sizeof u);
  return R(cemuCommInitRank(reinterpret_cast<cemuComm_t*>(comm), nranks, u, rank));
}

CEMU_EXPORT ncclResult_t ncclCommInitAll(ncclComm_t* comms, int ndev, const int* devlist) {
  return R(cemuCommInitAll(reinterpret_cast<cemuComm_t*>(comms), ndev, devlist));
}

CEMU_EXPORT ncclResult_t ncclCommDestroy(ncclComm_t comm) { return R(cemuCommDestroy(C(comm))); }
CEMU_EXPORT ncclResult_t ncclCommFinalize(ncclComm_t) { return ncclSuccess; }
CEMU_EXPORT ncclResult_t ncclCommCount(const ncclComm_t comm, int* count) { return R(cemuCommCount(C(comm), count)); }
CEMU_EXPORT ncclResult_t ncclCommUserRank(const ncclComm_t comm, int* rank) {
  return R(cemuCommUserRank(C(comm), rank));
}
CEMU_EXPORT ncclResult_t ncclCommCuDevice(const ncclComm_t comm, int* device) {
  return R(cemuCommCuDevice(C(comm), device));
}
CEMU_EXPORT const char* ncclGetErrorString(ncclResult_t r) { return cemuGetErrorString(static_cast<cemuResult_t>(r)); }
CEMU_EXPORT const char* ncclGetLastError(ncclComm_t comm) { return cemuGetLastError(C(comm)); }
CEMU_EXPORT ncclResult_t ncclCommGetAsyncError(ncclComm_t comm, ncclResult_t* err) {
  cemuResult_t e = cemuSuccess;
  const cemuResult_t r = cemuCommGetAsyncError(C(comm), &e);
  *err = R(e);
  return R(r);
}

CEMU_EXPORT ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t dt,
                                       ncclRedOp_t op, ncclComm_t comm, cudaStream_t s) {
  return R(cemuAllReduce(send, recv, count, static_cast<cemuDataType_t>(dt), static_cast<cemuRedOp_t>(op), C(comm),
                         S(s)));
}

CEMU_EXPORT ncclResult_t ncclAllGather(const void* send, void* recv, size_t sendcount, ncclDataType_t dt,
                                       ncclComm_t comm, cudaStream_t s) {
  return R(cemuAllGather(send, recv, sendcount, static_cast<cemuDataType_t>(dt), C(comm), S(s)));
}

CEMU_EXPORT ncclResult_t ncclReduceScatter(const void* send, void* recv, size_t recvcount, ncclDataType_t dt,
                                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t s) {
  return R(cemuReduceScatter(send, recv, recvcount, static_cast<cemuDataType_t>(dt), static_cast<cemuRedOp_t>(op),
                             C(comm), S(s)));
}

CEMU_EXPORT ncclResult_t ncclBroadcast(const void* send, void* recv, size_t count, ncclDataType_t dt, int root,
                                       ncclComm_t comm, cudaStream_t s) {
  return R(cemuBroadcast(send, recv, count, static_cast<cemuDataType_t>(dt), root, C(comm), S(s)));
}

CEMU_EXPORT ncclResult_t ncclGroupStart() { return R(cemuGroupStart()); }
CEMU_EXPORT ncclResult_t ncclGroupEnd() { return R(cemuGroupEnd()); }
