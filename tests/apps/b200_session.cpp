// b200_session.cpp -- the INTEGRATION.md recipe, compiled: a C++ drop-in for
// the reference real node's cemu::WorkerSession (proj/include/cemu/
// collective.hpp:50-131) over the C-ABI, on HOST spans like the original.
//
//   b200_session <config file> <rank> <elems> <out.bin>
// runs allreduce_async(span, 4) + wait on an int32 buffer holding i*7+rank,
// then allgather_async(span, 1) on a byte buffer (own block = rank+1), and
// writes both results to out.bin.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <fstream>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "cemu_b200.h"

namespace cemu {
struct TransportError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
}  // namespace cemu

class B200Session {
 public:
  B200Session(const std::string& config_text, uint32_t rank, int device) : rank_(rank) {
    cemuUniqueId id{};  // one real GPU: any bytes
    if (cemuCommInitRankConfig(&comm_, config_text.c_str(), id, static_cast<int>(rank), device) != cemuSuccess)
      throw cemu::TransportError(cemuGetLastError(comm_));
    cudaSetDevice(device);
    cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking);
    int w = 0;
    cemuCommCount(comm_, &w);
    world_ = static_cast<uint32_t>(w);
  }
  // WorkerSession::allreduce_async(span, elem_size): elem_size 4 -> int32
  // lanes, else bytes (collective.cpp:343-350)
  void allreduce_async(std::span<uint8_t> buf, uint32_t elem_size) {
    const bool w = elem_size == 4;
    auto r = cemuAllReduceHost(buf.data(), buf.data(), buf.size() / (w ? 4 : 1), w ? cemuInt32 : cemuUint8, cemuSum,
                               comm_, reinterpret_cast<cemuStream_t>(stream_));
    if (r != cemuSuccess) throw cemu::TransportError(cemuGetLastError(comm_));
  }
  // WorkerSession::allgather_async(full, elem_size): own block already at rank * block
  void allgather_async(std::span<uint8_t> full, uint32_t /*elem_size*/) {
    const size_t blk = full.size() / world_;
    auto r = cemuAllGatherHost(full.data() + rank_ * blk, full.data(), blk, cemuUint8, comm_,
                               reinterpret_cast<cemuStream_t>(stream_));
    if (r != cemuSuccess) throw cemu::TransportError(cemuGetLastError(comm_));
  }
  void wait() { cudaStreamSynchronize(stream_); }  // WorkerSession::wait
  ~B200Session() {
    cemuCommDestroy(comm_);
    cudaStreamDestroy(stream_);
  }

 private:
  cemuComm_t comm_ = nullptr;
  cudaStream_t stream_ = nullptr;
  uint32_t rank_ = 0, world_ = 1;
};

int main(int argc, char** argv) {
  if (argc != 5) {
    std::fprintf(stderr, "usage: %s <config> <rank> <elems> <out.bin>\n", argv[0]);
    return 2;
  }
  std::ifstream in(argv[1]);
  std::stringstream ss;
  ss << in.rdbuf();
  const uint32_t rank = static_cast<uint32_t>(std::stoul(argv[2]));
  const size_t elems = std::stoull(argv[3]);
  try {
    B200Session s(ss.str(), rank, 0);
    std::vector<int32_t> v(elems);
    for (size_t i = 0; i < elems; ++i) v[i] = static_cast<int32_t>(i * 7 + rank);
    cudaHostRegister(v.data(), v.size() * 4, cudaHostRegisterDefault);  // pinned: overlapped pipeline
    s.allreduce_async(std::span<uint8_t>(reinterpret_cast<uint8_t*>(v.data()), v.size() * 4), 4);
    s.wait();
    int w = 0;
    {
      // world size from the config via a throwaway parse of the C-ABI
      cemuJobConfig_t cfg = nullptr;
      char err[256];
      cemuConfigParse(ss.str().c_str(), &cfg, err, sizeof err);
      w = static_cast<int>(cemuConfigWorldSize(cfg));
      cemuConfigFree(cfg);
    }
    const size_t blk = 1000;
    std::vector<uint8_t> full(blk * w, 0);
    for (size_t i = 0; i < blk; ++i) full[rank * blk + i] = static_cast<uint8_t>(rank + 1 + i);
    s.allgather_async(std::span<uint8_t>(full), 1);
    s.wait();
    std::ofstream out(argv[4], std::ios::binary);
    out.write(reinterpret_cast<const char*>(v.data()), v.size() * 4);
    out.write(reinterpret_cast<const char*>(full.data()), full.size());
    cudaHostUnregister(v.data());
    std::printf("b200_session ok rank %u world %d elems %zu\n", rank, w, elems);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
