// symmetric.cpp -- symmetric memory of the fused multi-GPU path: every real
// GPU's range mapped into every real GPU's process (CUDA IPC), owned
// (cemuMemAlloc, the ncclMemAlloc + window analogue) or registered caller
// memory (cemuCommRegister: ncclCommRegister / ncclCommWindowRegister).
#include "comm_internal.hpp"

namespace cemu_b200 {

// All-gather `rec` (bytes each) among the k real GPUs through the inner NCCL
// comm; synchronous (setup / registration only, never on the hot path).
cudaError_t exchange_records(cemuComm* c, const void* rec, size_t bytes, std::vector<uint8_t>* all, ncclResult_t* nr) {
  const Nccl* n = nccl();
  uint8_t* d = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaMalloc(&d, bytes * c->k);
  if (e != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess) { cudaFree(d); return e; }
  if ((e = cudaMemcpy(d + bytes * c->li, rec, bytes, cudaMemcpyHostToDevice)) == cudaSuccess) {
    *nr = n->AllGather(d + bytes * c->li, d, bytes, ncclUint8, c->inner, st);
    if (*nr == ncclSuccess) {
      e = cudaStreamSynchronize(st);
      all->resize(bytes * c->k);
      if (e == cudaSuccess) e = cudaMemcpy(all->data(), d, bytes * c->k, cudaMemcpyDeviceToHost);
    }
  }
  cudaStreamDestroy(st);
  cudaFree(d);
  return e;
}

// What each real rank publishes for one symmetric range: the IPC handle of
// the allocation holding it, where the range starts inside that allocation
// and how long it is.  `ok` = 0 when this rank could not export its range:
// every rank still takes part in the exchange, so all of them fail together
// instead of one hanging in it.
struct IpcRecord {
  cudaIpcMemHandle_t handle;
  uint64_t offset;
  uint64_t bytes;
  int32_t ok;
  int32_t pad;
};

void* open_peer(cemuComm* c, uint32_t g, const cudaIpcMemHandle_t& h, cudaError_t* err) {
  std::string key(reinterpret_cast<const char*>(&h), sizeof h);
  key.push_back(static_cast<char>(g));
  auto& m = c->ipc_maps[key];
  if (!m.ptr) {
    *err = cudaIpcOpenMemHandle(&m.ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (*err != cudaSuccess) {
      c->ipc_maps.erase(key);
      return nullptr;
    }
  }
  ++m.refs;
  return m.ptr;
}

void close_peer(cemuComm* c, void* ptr) {
  for (auto it = c->ipc_maps.begin(); it != c->ipc_maps.end(); ++it) {
    if (it->second.ptr != ptr) continue;
    if (--it->second.refs == 0) {
      cudaIpcCloseMemHandle(ptr);
      c->ipc_maps.erase(it);
    }
    return;
  }
}

// Collective: every real rank publishes (handle, offset, bytes) of its
// range [alloc_base + offset, + bytes) and maps every peer's.
cemuResult_t map_range(cemuComm* c, void* alloc_base, uint64_t offset, size_t bytes, bool exportable,
                       const std::string& why, uint8_t** peers, uint8_t** peer_maps) {
  IpcRecord mine{};
  mine.offset = offset;
  mine.bytes = bytes;
  mine.ok = exportable ? 1 : 0;
  std::string local_err = why;
  if (exportable) {
    const cudaError_t e = cudaIpcGetMemHandle(&mine.handle, alloc_base);
    if (e != cudaSuccess) {
      mine.ok = 0;
      local_err = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
      cudaGetLastError();
    }
  }
  std::vector<uint8_t> all;
  ncclResult_t nr = ncclSuccess;
  const cudaError_t e = exchange_records(c, &mine, sizeof mine, &all, &nr);
  if (nr != ncclSuccess) return fail(static_cast<cemuResult_t>(nr), "ipc handle exchange: nccl error");
  if (e != cudaSuccess) return fail(cemuUnhandledCudaError, std::string("ipc handle exchange: ") + cudaGetErrorString(e));
  std::vector<IpcRecord> rec(c->k);
  for (uint32_t g = 0; g < c->k; ++g) std::memcpy(&rec[g], all.data() + g * sizeof(IpcRecord), sizeof(IpcRecord));
  for (uint32_t g = 0; g < c->k; ++g) {
    if (!rec[g].ok) {
      return fail(cemuInvalidUsage, g == c->li ? "symmetric range: " + local_err
                                                : "symmetric range: real rank index " + std::to_string(g) +
                                                      " could not export its buffer");
    }
    if (rec[g].bytes != bytes) {
      return fail(cemuInvalidUsage, "symmetric range: real ranks asked for different sizes (" + std::to_string(bytes) +
                                        " vs " + std::to_string(rec[g].bytes) + ")");
    }
  }
  uint8_t* maps[kMaxReal] = {};
  for (uint32_t g = 0; g < c->k; ++g) {
    if (g == c->li) {
      peers[g] = static_cast<uint8_t*>(alloc_base) + offset;
      continue;
    }
    cudaError_t oe = cudaSuccess;
    void* p = open_peer(c, g, rec[g].handle, &oe);
    if (!p) {
      for (uint32_t h = 0; h < g; ++h) {
        if (maps[h]) close_peer(c, maps[h]);
      }
      return fail(cemuUnhandledCudaError, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(oe));
    }
    maps[g] = static_cast<uint8_t*>(p);
    peers[g] = maps[g] + rec[g].offset;
  }
  if (peer_maps) {
    for (uint32_t g = 0; g < c->k; ++g) peer_maps[g] = maps[g];
  }
  return cemuSuccess;
}

// Maps every real GPU's allocation `local` (collectively) into this process.
cemuResult_t map_peers(cemuComm* c, void* local, size_t bytes, uint8_t** peers, uint8_t** peer_maps) {
  return map_range(c, local, 0, bytes, true, "", peers, peer_maps);
}

void unmap_region(cemuComm* c, cemuComm::Region& r) {
  for (uint32_t g = 0; g < c->k; ++g) {
    if (g != c->li && r.peer_map[g]) close_peer(c, r.peer_map[g]);
    r.peer_map[g] = nullptr;
  }
  if (c->k > 1 && c->fused) {  // every peer unmapped before anyone frees
    std::vector<uint8_t> all;
    ncclResult_t nr = ncclSuccess;
    const uint8_t one = 1;
    exchange_records(c, &one, 1, &all, &nr);
  }
}

}  // namespace cemu_b200

extern "C" {

cemuResult_t cemuMemAlloc(cemuComm_t c, size_t bytes, void** ptr) {
  if (!c || !ptr || bytes == 0) return fail(cemuInvalidArgument, "cemuMemAlloc: bad argument");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(cemuUnhandledCudaError, "cemuMemAlloc: cudaSetDevice");
  const size_t rounded = (bytes + (2u << 20) - 1) & ~static_cast<size_t>((2u << 20) - 1);
  void* p = nullptr;
  CUDA_OK(cudaMalloc(&p, rounded));
  cemuComm::Region r;
  r.base = static_cast<uint8_t*>(p);
  r.bytes = rounded;
  r.peer[c->li] = r.base;
  r.id = c->next_region_id++;
  if (c->k > 1 && c->fused) {
    if (auto e = map_peers(c, p, rounded, r.peer, r.peer_map)) {
      cudaFree(p);
      return e;
    }
  }
  c->regions.push_back(r);
  *ptr = p;
  return cemuSuccess;
}

cemuResult_t cemuMemFree(cemuComm_t c, void* ptr) {
  if (!c || !ptr) return fail(cemuInvalidArgument, "cemuMemFree: bad argument");
  for (size_t i = 0; i < c->regions.size(); ++i) {
    auto& r = c->regions[i];
    if (r.base != ptr || !r.owned) continue;
    cudaSetDevice(c->device);
    if (c->order_ev) cudaEventSynchronize(c->order_ev);  // no call of this comm still uses it
    unmap_region(c, r);
    cudaFree(r.base);
    c->regions.erase(c->regions.begin() + static_cast<long>(i));
    return cemuSuccess;
  }
  return fail(cemuInvalidArgument, "cemuMemFree: pointer was not returned by cemuMemAlloc");
}

namespace {
// cuMemGetAddressRange through the runtime's driver entry point (no link
// against libcuda): the allocation holding `p`.
using GetRangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);
bool allocation_of(const void* p, void** base, size_t* bytes) {
  static GetRangeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<GetRangeFn>(nullptr);
    }
    return reinterpret_cast<GetRangeFn>(f);
  }();
  unsigned long long b = 0;
  size_t n = 0;
  if (!fn || fn(&b, &n, reinterpret_cast<unsigned long long>(p)) != 0) return false;
  *base = reinterpret_cast<void*>(b);
  *bytes = n;
  return true;
}
}  // namespace

// ncclCommRegister / ncclCommWindowRegister (nccl.h 2.27.3:243, 251): the
// caller's device range becomes a symmetric range of this communicator, so
// collectives on it (at the same offsets on every real rank) take the fused
// NVLink kernels.  Collective over the job's real ranks on this box, like
// NCCL's window registration: each rank exports the cudaMalloc allocation
// holding its range (CUDA IPC) and maps every peer's.
cemuResult_t cemuCommRegister(cemuComm_t c, void* buff, size_t size, void** handle) {
  if (!c || !handle) return fail(cemuInvalidArgument, "cemuCommRegister: null argument");
  *handle = nullptr;
  if (!buff || size == 0) return cemuSuccess;  // nothing to register (NCCL accepts it too)
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(cemuUnhandledCudaError, "cemuCommRegister: cudaSetDevice");
  cemuComm::Region r;
  r.base = static_cast<uint8_t*>(buff);
  r.bytes = size;
  r.owned = false;
  r.peer[c->li] = r.base;
  r.id = c->next_region_id++;
  if (c->k > 1 && c->fused) {
    void* base = nullptr;
    size_t abytes = 0;
    bool ok = allocation_of(buff, &base, &abytes);
    std::string why;
    if (!ok) {
      why = "cemuCommRegister: the range is not device memory of this process";
    } else if (static_cast<uint8_t*>(buff) + size > static_cast<uint8_t*>(base) + abytes) {
      ok = false;
      why = "cemuCommRegister: the range spans more than one allocation";
    }
    const uint64_t off = ok ? static_cast<uint64_t>(static_cast<uint8_t*>(buff) - static_cast<uint8_t*>(base)) : 0;
    if (auto e = map_range(c, base, off, size, ok, why, r.peer, r.peer_map)) return e;
  }
  c->regions.push_back(r);
  *handle = reinterpret_cast<void*>(static_cast<uintptr_t>(r.id));
  return cemuSuccess;
}

cemuResult_t cemuCommDeregister(cemuComm_t c, void* handle) {
  if (!c) return fail(cemuInvalidArgument, "cemuCommDeregister: comm is null");
  if (!handle) return cemuSuccess;
  const uint64_t id = static_cast<uint64_t>(reinterpret_cast<uintptr_t>(handle));
  for (size_t i = 0; i < c->regions.size(); ++i) {
    auto& r = c->regions[i];
    if (r.id != id || r.owned) continue;
    cudaSetDevice(c->device);
    if (c->order_ev) cudaEventSynchronize(c->order_ev);  // no call of this comm still uses it
    unmap_region(c, r);
    c->regions.erase(c->regions.begin() + static_cast<long>(i));
    return cemuSuccess;
  }
  return fail(cemuInvalidArgument, "cemuCommDeregister: handle was not returned by cemuCommRegister");
}

}  // extern "C"
