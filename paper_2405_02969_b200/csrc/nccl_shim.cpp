// nccl_shim.cpp -- libnccl_cemu.so: NCCL's own symbols, backed by the
// emulator.  The NeuronaBox paper interposes on NCCL; an
// unmodified NCCL application gets the emulated world with
//   CEMU_CONFIG=job.cfg LD_PRELOAD=libnccl_cemu.so ./app
// nranks passed to ncclCommInitRank must equal the config's world_size and
// the rank must be one of its real ranks.  ncclComm_t is the cemuComm_t;
// datatypes, reduction ops and result codes share NCCL's values.
//
// When the job puts several real ranks on this box, libcemu_b200 drives the
// real libnccl.so.2 for them (dlopen + dlsym on its handle).  The real
// library calls some of its own public entry points internally -- e.g.
// ncclCommGetAsyncError while a blocking ncclCommInitRank waits -- and with
// this shim preloaded those calls land here.  So every entry point that
// takes a communicator serves only the communicators this shim created and
// forwards any other one to the next definition (RTLD_NEXT: the real NCCL).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <unordered_set>

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

// the communicators this shim handed out
std::mutex g_mu;
std::unordered_set<const void*> g_ours;
void adopt(ncclComm_t c) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_ours.insert(c);
}
void release(ncclComm_t c) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_ours.erase(c);
}
bool ours(const void* c) {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_ours.count(c) != 0;
}

// The next definition of `name` (the real NCCL), looked up once per entry.
template <typename F>
F next(const char* name) {
  return reinterpret_cast<F>(dlsym(RTLD_NEXT, name));
}
}  // namespace

// A foreign communicator goes to the real NCCL (or is an invalid argument
// when none is loaded).
#define FORWARD_FOREIGN(comm, name, ...)                                  \
  do {                                                                    \
    if (comm && !ours(comm)) {                                            \
      static const auto real = next<decltype(&name)>(#name);              \
      return real ? real(__VA_ARGS__) : ncclInvalidArgument;              \
    }                                                                     \
  } while (0)

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
  const ncclResult_t r = R(cemuCommInitRank(reinterpret_cast<cemuComm_t*>(comm), nranks, u, rank));
  if (r == ncclSuccess) adopt(*comm);
  return r;
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
  const ncclResult_t r = R(cemuCommInitAll(reinterpret_cast<cemuComm_t*>(comms), ndev, devlist));
  if (r == ncclSuccess) {
    for (int i = 0; i < ndev; ++i) adopt(comms[i]);
  }
  return r;
}

CEMU_EXPORT ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  FORWARD_FOREIGN(comm, ncclCommDestroy, comm);
  release(comm);
  return R(cemuCommDestroy(C(comm)));
}
CEMU_EXPORT ncclResult_t ncclCommFinalize(ncclComm_t comm) {
  FORWARD_FOREIGN(comm, ncclCommFinalize, comm);
  return ncclSuccess;
}
CEMU_EXPORT ncclResult_t ncclCommAbort(ncclComm_t comm) {
  FORWARD_FOREIGN(comm, ncclCommAbort, comm);
  release(comm);
  return R(cemuCommDestroy(C(comm)));
}
// Buffer registration maps the caller's buffers on every real GPU of the
// box, so an unmodified NCCL job's collectives on registered (or
// window-registered) buffers reach the fused NVLink kernels; unregistered
// buffers take NCCL reduce-scatter + synthesis + NCCL allgather.
CEMU_EXPORT ncclResult_t ncclCommRegister(const ncclComm_t comm, void* buff, size_t size, void** handle) {
  FORWARD_FOREIGN(comm, ncclCommRegister, comm, buff, size, handle);
  return R(cemuCommRegister(C(comm), buff, size, handle));
}
CEMU_EXPORT ncclResult_t ncclCommDeregister(const ncclComm_t comm, void* handle) {
  FORWARD_FOREIGN(comm, ncclCommDeregister, comm, handle);
  return R(cemuCommDeregister(C(comm), handle));
}
CEMU_EXPORT ncclResult_t ncclCommWindowRegister(ncclComm_t comm, void* buff, size_t size, ncclWindow_t* win,
                                                int winFlags) {
  FORWARD_FOREIGN(comm, ncclCommWindowRegister, comm, buff, size, win, winFlags);
  if (!win) return R(cemuCommRegister(C(comm), buff, size, nullptr));  // reports the null argument
  void* h = nullptr;
  const cemuResult_t r = cemuCommRegister(C(comm), buff, size, &h);
  *win = reinterpret_cast<ncclWindow_t>(h);
  return R(r);
}
CEMU_EXPORT ncclResult_t ncclCommWindowDeregister(ncclComm_t comm, ncclWindow_t win) {
  FORWARD_FOREIGN(comm, ncclCommWindowDeregister, comm, win);
  return R(cemuCommDeregister(C(comm), reinterpret_cast<void*>(win)));
}
// ncclMemAlloc / ncclMemFree (nccl.h:130-134) carry no communicator: plain
// device memory, 2 MiB granular like NCCL's cuMem allocations, exportable
// to the box's other real ranks when a communicator registers it.
CEMU_EXPORT ncclResult_t ncclMemAlloc(void** ptr, size_t size) {
  if (!ptr) return ncclInvalidArgument;
  *ptr = nullptr;
  if (size == 0) return ncclSuccess;
  const size_t rounded = (size + (2u << 20) - 1) & ~static_cast<size_t>((2u << 20) - 1);
  if (cudaMalloc(ptr, rounded) != cudaSuccess) {
    g_shim_error = "ncclMemAlloc: cudaMalloc failed";
    return ncclUnhandledCudaError;
  }
  return ncclSuccess;
}
CEMU_EXPORT ncclResult_t ncclMemFree(void* ptr) {
  if (ptr && cudaFree(ptr) != cudaSuccess) {
    g_shim_error = "ncclMemFree: cudaFree failed";
    return ncclUnhandledCudaError;
  }
  return ncclSuccess;
}
// Entry points the emulated world does not provide fail loudly here rather
// than reaching the real libnccl with an emulated communicator.
CEMU_EXPORT ncclResult_t ncclCommSplit(ncclComm_t comm, int color, int key, ncclComm_t* newcomm, ncclConfig_t* config) {
  FORWARD_FOREIGN(comm, ncclCommSplit, comm, color, key, newcomm, config);
  if (newcomm) *newcomm = nullptr;
  return not_emulated("ncclCommSplit: sub-communicators of an emulated world are not provided");
}
CEMU_EXPORT ncclResult_t ncclReduce(const void* send, void* recv, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                                    int root, ncclComm_t comm, cudaStream_t s) {
  FORWARD_FOREIGN(comm, ncclReduce, send, recv, count, dt, op, root, comm, s);
  return not_emulated("ncclReduce: not emulated (allreduce, allgather, reduce-scatter and broadcast are)");
}
CEMU_EXPORT ncclResult_t ncclSend(const void* send, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                                  cudaStream_t s) {
  FORWARD_FOREIGN(comm, ncclSend, send, count, dt, peer, comm, s);
  return not_emulated("ncclSend: point-to-point traffic is not emulated");
}
CEMU_EXPORT ncclResult_t ncclRecv(void* recv, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                                  cudaStream_t s) {
  FORWARD_FOREIGN(comm, ncclRecv, recv, count, dt, peer, comm, s);
  return not_emulated("ncclRecv: point-to-point traffic is not emulated");
}
CEMU_EXPORT ncclResult_t ncclCommCount(const ncclComm_t comm, int* count) {
  FORWARD_FOREIGN(comm, ncclCommCount, comm, count);
  return R(cemuCommCount(C(comm), count));
}
CEMU_EXPORT ncclResult_t ncclCommUserRank(const ncclComm_t comm, int* rank) {
  FORWARD_FOREIGN(comm, ncclCommUserRank, comm, rank);
  return R(cemuCommUserRank(C(comm), rank));
}
CEMU_EXPORT ncclResult_t ncclCommCuDevice(const ncclComm_t comm, int* device) {
  FORWARD_FOREIGN(comm, ncclCommCuDevice, comm, device);
  return R(cemuCommCuDevice(C(comm), device));
}
CEMU_EXPORT const char* ncclGetErrorString(ncclResult_t r) { return cemuGetErrorString(static_cast<cemuResult_t>(r)); }
CEMU_EXPORT const char* ncclGetLastError(ncclComm_t comm) {
  if (comm && !ours(comm)) {
    static const auto real = next<decltype(&ncclGetLastError)>("ncclGetLastError");
    return real ? real(comm) : "";
  }
  if (g_shim_error) {
    const char* e = g_shim_error;
    g_shim_error = nullptr;
    return e;
  }
  return cemuGetLastError(C(comm));
}
CEMU_EXPORT ncclResult_t ncclCommGetAsyncError(ncclComm_t comm, ncclResult_t* err) {
  FORWARD_FOREIGN(comm, ncclCommGetAsyncError, comm, err);
  cemuResult_t e = cemuSuccess;
  const cemuResult_t r = cemuCommGetAsyncError(C(comm), &e);
  *err = R(e);
  return R(r);
}

CEMU_EXPORT ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t dt,
                                       ncclRedOp_t op, ncclComm_t comm, cudaStream_t s) {
  FORWARD_FOREIGN(comm, ncclAllReduce, send, recv, count, dt, op, comm, s);
  return R(cemuAllReduce(send, recv, count, static_cast<cemuDataType_t>(dt), static_cast<cemuRedOp_t>(op), C(comm),
                         S(s)));
}

CEMU_EXPORT ncclResult_t ncclAllGather(const void* send, void* recv, size_t sendcount, ncclDataType_t dt,
                                       ncclComm_t comm, cudaStream_t s) {
  FORWARD_FOREIGN(comm, ncclAllGather, send, recv, sendcount, dt, comm, s);
  return R(cemuAllGather(send, recv, sendcount, static_cast<cemuDataType_t>(dt), C(comm), S(s)));
}

CEMU_EXPORT ncclResult_t ncclReduceScatter(const void* send, void* recv, size_t recvcount, ncclDataType_t dt,
                                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t s) {
  FORWARD_FOREIGN(comm, ncclReduceScatter, send, recv, recvcount, dt, op, comm, s);
  return R(cemuReduceScatter(send, recv, recvcount, static_cast<cemuDataType_t>(dt), static_cast<cemuRedOp_t>(op),
                             C(comm), S(s)));
}

CEMU_EXPORT ncclResult_t ncclBroadcast(const void* send, void* recv, size_t count, ncclDataType_t dt, int root,
                                       ncclComm_t comm, cudaStream_t s) {
  FORWARD_FOREIGN(comm, ncclBroadcast, send, recv, count, dt, root, comm, s);
  return R(cemuBroadcast(send, recv, count, static_cast<cemuDataType_t>(dt), root, C(comm), S(s)));
}

// Groups: the emulated communicators' calls are deferred and replayed by
// cemuGroupEnd, which brackets its own inner-NCCL launches.  (The real
// NCCL's internal grouping does not go through these public symbols.)
CEMU_EXPORT ncclResult_t ncclGroupStart() { return R(cemuGroupStart()); }
CEMU_EXPORT ncclResult_t ncclGroupEnd() { return R(cemuGroupEnd()); }
