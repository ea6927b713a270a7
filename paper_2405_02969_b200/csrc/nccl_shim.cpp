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
// errors raised by the shim itself (entry points the emulated world does
// not provide); ncclGetLastError reports them ahead of the library's
thread_local const char* g_shim_error = nullptr;
ncclResult_t not_emulated(const char* what) {
  g_shim_error = what;
  return ncclInvalidUsage;
}
inline cemuComm_t C(ncclComm_t c) { return reinterpret_cast<cemuComm_t>(c); }
inline cemuStream_t S(cudaStream_t s) { return reinterpret_cast<cemuStream_t>(s); }
inline ncclResult_t R(cemuResult_t r) { return static_cast<ncclResult_t>(r); }
}  // namespace

CEMU_EXPORT ncclResult_t ncclGetVersion(int* version) { return R(cemuGetVersion(version)); }

CEMU_EXPORT ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  return R(cemuGetUniqueId(reinterpret_cast<cemuUniqueId*>(id)));
}

namespace {
// (called by both exports directly: a call through the exported symbol could
// be interposed by an earlier-loaded libnccl)
ncclResult_t init_rank(ncclComm_t* comm, int nranks, const ncclUniqueId& id, int rank) {
  cemuUniqueId u;
  static_assert(sizeof u == sizeof id, "unique id size");
  __builtin_memcpy(&u, &id, sizeof u);
  return R(cemuCommInitRank(reinterpret_cast<cemuComm_t*>(comm), nranks, u, rank));
}
}  // namespace

CEMU_EXPORT ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  return init_rank(comm, nranks, id, rank);
}

// the config's fields (blocking, CTA counts, net name, ...) steer NCCL's own
// resources; the emulated communicator has none of them to tune
CEMU_EXPORT ncclResult_t ncclCommInitRankConfig(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank,
                                                ncclConfig_t*) {
  return init_rank(comm, nranks, id, rank);
}

CEMU_EXPORT ncclResult_t ncclCommInitAll(ncclComm_t* comms, int ndev, const int* devlist) {
  return R(cemuCommInitAll(reinterpret_cast<cemuComm_t*>(comms), ndev, devlist));
}

CEMU_EXPORT ncclResult_t ncclCommDestroy(ncclComm_t comm) { return R(cemuCommDestroy(C(comm))); }
CEMU_EXPORT ncclResult_t ncclCommFinalize(ncclComm_t) { return ncclSuccess; }
CEMU_EXPORT ncclResult_t ncclCommAbort(ncclComm_t comm) { return R(cemuCommDestroy(C(comm))); }
// buffer registration is a no-op here (symmetric buffers come from cemuMemAlloc)
CEMU_EXPORT ncclResult_t ncclCommRegister(const ncclComm_t, void*, size_t, void** handle) {
  if (handle) *handle = nullptr;
  return ncclSuccess;
}
CEMU_EXPORT ncclResult_t ncclCommDeregister(const ncclComm_t, void*) { return ncclSuccess; }
// Entry points the emulated world does not provide fail loudly here rather
// than reaching the real libnccl with an emulated communicator.
CEMU_EXPORT ncclResult_t ncclCommSplit(ncclComm_t, int, int, ncclComm_t* newcomm, ncclConfig_t*) {
  if (newcomm) *newcomm = nullptr;
  return not_emulated("ncclCommSplit: sub-communicators of an emulated world are not provided");
}
CEMU_EXPORT ncclResult_t ncclReduce(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                                    cudaStream_t) {
  return not_emulated("ncclReduce: not emulated (allreduce, allgather, reduce-scatter and broadcast are)");
}
CEMU_EXPORT ncclResult_t ncclSend(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) {
  return not_emulated("ncclSend: point-to-point traffic is not emulated");
}
CEMU_EXPORT ncclResult_t ncclRecv(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) {
  return not_emulated("ncclRecv: point-to-point traffic is not emulated");
}
CEMU_EXPORT ncclResult_t ncclCommCount(const ncclComm_t comm, int* count) { return R(cemuCommCount(C(comm), count)); }
CEMU_EXPORT ncclResult_t ncclCommUserRank(const ncclComm_t comm, int* rank) {
  return R(cemuCommUserRank(C(comm), rank));
}
CEMU_EXPORT ncclResult_t ncclCommCuDevice(const ncclComm_t comm, int* device) {
  return R(cemuCommCuDevice(C(comm), device));
}
CEMU_EXPORT const char* ncclGetErrorString(ncclResult_t r) { return cemuGetErrorString(static_cast<cemuResult_t>(r)); }
CEMU_EXPORT const char* ncclGetLastError(ncclComm_t comm) {
  if (g_shim_error) {
    const char* e = g_shim_error;
    g_shim_error = nullptr;
    return e;
  }
  return cemuGetLastError(C(comm));
}
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
