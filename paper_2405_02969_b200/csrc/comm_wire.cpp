// comm_wire.cpp -- a communicator in wire mode: its
// collectives run the reference worker's op over the CEMU frame protocol
// (wire.cpp) against a reference cemu-emulator.
#include "comm_internal.hpp"

namespace cemu_b200 {

// ---- wire mode -------------------------------------------------------------
// The call runs the reference worker's op (collective.cpp:268-355) with the
// buffer on the GPU: each outgoing chunk is read back from HBM, each incoming
// DATA payload is copied up and folded by launch_wire_fold.  Host-synchronous
// (the protocol is a conversation); results and the per-step arrival times
// land in the call record, next to the device model's floors for the same
// call, so the reference engine's releases can be checked against them.
cemuResult_t wire_call(cemuComm* c, int coll, const void* send, void* recv, uint64_t buf_bytes, uint64_t model_bytes,
                       uint32_t es, cudaStream_t s) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_OK(cudaStreamIsCapturing(s, &cap));
  if (cap != cudaStreamCaptureStatusNone) {
    return fail(cemuInvalidUsage, "wire mode: collectives are host-synchronous and cannot be captured");
  }
  auto* r8 = static_cast<uint8_t*>(recv);
  if (coll == kAllReduce && send != recv) CUDA_OK(cudaMemcpyAsync(recv, send, buf_bytes, cudaMemcpyDeviceToDevice, s));
  if (coll == kAllGather) {
    uint8_t* own = r8 + static_cast<uint64_t>(c->rank) * model_bytes;
    if (send != own) CUDA_OK(cudaMemcpyAsync(own, send, model_bytes, cudaMemcpyDeviceToDevice, s));
  }
  CUDA_OK(cudaStreamSynchronize(s));
  const uint64_t id = c->calls++;
  const uint32_t i = static_cast<uint32_t>(id % cemuComm::kSlots);
  auto& m = c->meta[i];
  m.call_id = id;
  m.coll = coll;
  m.delay = true;  // the record holds the wire arrivals
  m.k = to_real_count(coll, c->W, c->real);
  m.bytes = model_bytes;
  m.latency = call_latency_us(c->delay, coll, c->W, model_bytes, m.k);
  int launches = 0;
  cudaError_t cerr = cudaSuccess;
  auto load = [&](uint64_t off, uint64_t len, uint8_t* host) {
    if (cerr == cudaSuccess) cerr = cudaMemcpy(host, r8 + off, len, cudaMemcpyDeviceToHost);
  };
  auto store = [&](uint64_t off, const uint8_t* host, uint64_t len, bool reduce) {
    if (cerr != cudaSuccess || len == 0) return;
    if (!reduce) {
      cerr = cudaMemcpy(r8 + off, host, len, cudaMemcpyHostToDevice);
      return;
    }
    if (c->wire_buf_bytes < len) {
      if (c->wire_buf) cudaFree(c->wire_buf);
      c->wire_buf = nullptr;
      c->wire_buf_bytes = 0;
      if ((cerr = cudaMalloc(&c->wire_buf, len)) != cudaSuccess) return;
      c->wire_buf_bytes = len;
    }
    if ((cerr = cudaMemcpyAsync(c->wire_buf, host, len, cudaMemcpyHostToDevice, s)) != cudaSuccess) return;
    if ((cerr = launch_wire_fold(r8 + off, c->wire_buf, len, es == 4, s, &launches)) != cudaSuccess) return;
    cerr = cudaStreamSynchronize(s);
  };
  int64_t t_open = 0;
  std::vector<int64_t> arrivals;
  try {
    c->wire->run(coll, buf_bytes, es, load, store, &t_open, &arrivals);
  } catch (const WireError& e) {
    c->launches += launches;
    return fail(cemuRemoteError, e.what());
  }
  c->launches += launches;
  CUDA_OK(cerr);
  // call record: model floors beside the reference engine's observed releases
  const std::vector<double> offs = release_offsets(c->delay, coll, c->W, model_bytes, m.k);
  std::vector<int64_t> rec(slot_words(c->kmax), 0);
  rec[0] = t_open;
  int64_t maxf = 0;
  for (uint32_t j = 0; j < m.k; ++j) {
    const int64_t f = std::llround(offs[j]);
    maxf = std::max(maxf, f);
    rec[kSlotHeader + j] = f;
    rec[kSlotHeader + c->kmax + j] = j < arrivals.size() ? arrivals[j] : 0;
    std::memcpy(&rec[kSlotHeader + 2 * c->kmax + j], &offs[j], 8);
  }
  rec[1] = arrivals.empty() ? t_open : arrivals.back();
  rec[2] = maxf;
  rec[3] = m.k;
  CUDA_OK(cudaMemcpy(c->d_slots + i * slot_words(c->kmax), rec.data(), rec.size() * 8, cudaMemcpyHostToDevice));
  return cemuSuccess;
}

}  // namespace cemu_b200

extern "C" cemuResult_t cemuCommAttachEmulator(cemuComm_t c, const cemuPlanEntry* plan, size_t nplan,
                                               int timeoutMs) {
  if (!c) return fail(cemuInvalidArgument, "cemuCommAttachEmulator: comm is null");
  if (nplan && !plan) return fail(cemuInvalidArgument, "cemuCommAttachEmulator: plan is null");
  if (c->wire) return fail(cemuInvalidUsage, "cemuCommAttachEmulator: already attached");
  if (c->k != 1) return fail(cemuInvalidUsage, "cemuCommAttachEmulator: wire mode serves one real rank per box");
  std::vector<WirePlanEntry> p;
  for (size_t j = 0; j < nplan; ++j) {
    if (plan[j].coll != kAllReduce && plan[j].coll != kAllGather) {
      return fail(cemuInvalidArgument, "cemuCommAttachEmulator: plan entry " + std::to_string(j) +
                                           " is not allreduce/allgather");
    }
    p.push_back(WirePlanEntry{plan[j].coll, plan[j].bytes, plan[j].elemSize});
  }
  try {
    c->wire = std::make_unique<WireSession>(c->cfg, c->rank, std::move(p), timeoutMs > 0 ? timeoutMs : 10000);
  } catch (const WireError& e) {
    return fail(cemuRemoteError, e.what());
  } catch (const std::exception& e) {
    return fail(cemuSystemError, e.what());
  }
  return cemuSuccess;
}

extern "C" cemuResult_t cemuCommDetachEmulator(cemuComm_t c) {
  if (!c) return fail(cemuInvalidArgument, "cemuCommDetachEmulator: comm is null");
  c->wire.reset();
  return cemuSuccess;
}
