// host_pipe.cpp -- host-buffer collectives (cemuAllReduceHost /
// cemuAllGatherHost): the reference WorkerSession's host-span shape
// (proj/include/cemu/collective.hpp:68-78), pipelined through the GPU.
#include "comm_internal.hpp"

namespace cemu_b200 {

// ---- host-buffer collectives -------------------------------------------------
// The reference's WorkerSession takes host spans (collective.hpp:68-78);
// these entry points keep that shape.  One real GPU, hash payload: the
// buffer streams through the pipe in chunks, chunk i's H2D overlapping chunk
// i-1's synthesis and chunk i-2's D2H (PCIe is full duplex; the kernel takes
// ~1% of a chunk's transfer time).  Anything else (several real GPUs, zero
// payload) stages the whole buffer through device scratch and runs the
// device collective.
cemuResult_t ensure_pipe(cemuComm* c) {
  auto& p = c->pipe;
  if (p.ready) return cemuSuccess;
  if (!p.chunk) {
    size_t mib = 32;  // measured: 4 MiB 27.3 ms, 16 MiB 24.8, 32 MiB 22.9 per 1 GiB (full-duplex PCIe floor 22.4)
    if (const char* e = std::getenv("CEMU_HOST_CHUNK_MIB")) mib = std::max(1, std::atoi(e));
    p.chunk = mib << 20;
  }
  // (a retry after a failed attempt creates only what is still missing)
  if (!p.h2d) CUDA_OK(cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking));
  if (!p.comp) CUDA_OK(cudaStreamCreateWithFlags(&p.comp, cudaStreamNonBlocking));
  if (!p.d2h) CUDA_OK(cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking));
  if (!p.start) CUDA_OK(cudaEventCreateWithFlags(&p.start, cudaEventDisableTiming));
  // several real GPUs: the buffers are symmetric (mapped on every real GPU,
  // collective like cemuMemAlloc) so each chunk is one fused kernel
  p.symmetric = c->k > 1;
  for (int b = 0; b < cemuComm::kPipeBufs; ++b) {
    if (!p.buf[b] && p.symmetric) {
      const size_t rounded = (p.chunk + (2u << 20) - 1) & ~static_cast<size_t>((2u << 20) - 1);
      void* d = nullptr;
      CUDA_OK(cudaMalloc(&d, rounded));
      cemuComm::Region r;
      r.base = static_cast<uint8_t*>(d);
      r.bytes = rounded;
      r.peer[c->li] = r.base;
      r.id = c->next_region_id++;
      if (auto e = map_peers(c, d, rounded, r.peer, r.peer_map)) {
        cudaFree(d);
        return e;
      }
      c->regions.push_back(r);  // owns the allocation from here on
      p.buf[b] = d;
      for (uint32_t g = 0; g < c->k; ++g) p.peer[b][g] = r.peer[g];
    } else if (!p.buf[b]) {
      CUDA_OK(cudaMalloc(&p.buf[b], p.chunk));
    }
    if (!p.loaded[b]) CUDA_OK(cudaEventCreateWithFlags(&p.loaded[b], cudaEventDisableTiming));
    if (!p.done[b]) CUDA_OK(cudaEventCreateWithFlags(&p.done[b], cudaEventDisableTiming));
    if (!p.drained[b]) CUDA_OK(cudaEventCreateWithFlags(&p.drained[b], cudaEventDisableTiming));
  }
  p.ready = true;
  return cemuSuccess;
}

// One chunk: optional H2D of `in` into the device buffer, `work` on the
// compute stream, D2H of the buffer into `out`.
struct PipeChunk {
  const void* in = nullptr;  // host source (null: nothing to load)
  void* out = nullptr;       // host destination
  size_t bytes = 0;
  std::function<cudaError_t(int b, void* dbuf, cudaStream_t)> work;
};

cemuResult_t run_pipe(cemuComm* c, cudaStream_t s, const std::vector<PipeChunk>& chunks) {
  auto& p = c->pipe;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_OK(cudaStreamIsCapturing(s, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  CUDA_OK(cudaEventRecord(p.start, s));  // fork: everything after the caller's prior work
  CUDA_OK(cudaStreamWaitEvent(p.h2d, p.start, 0));
  CUDA_OK(cudaStreamWaitEvent(p.comp, p.start, 0));
  CUDA_OK(cudaStreamWaitEvent(p.d2h, p.start, 0));
  for (size_t i = 0; i < chunks.size(); ++i) {
    const int b = static_cast<int>(i % cemuComm::kPipeBufs);
    const PipeChunk& ch = chunks[i];
    // buffer b is free once its previous chunk has drained (a previous
    // call's drain is ordered by the fork unless the caller switched
    // streams; outside capture wait for it explicitly)
    if (i >= static_cast<size_t>(cemuComm::kPipeBufs) || !capturing) {
      CUDA_OK(cudaStreamWaitEvent(p.h2d, p.drained[b], 0));
    }
    if (ch.in) CUDA_OK(cudaMemcpyAsync(p.buf[b], ch.in, ch.bytes, cudaMemcpyHostToDevice, p.h2d));
    CUDA_OK(cudaEventRecord(p.loaded[b], p.h2d));
    CUDA_OK(cudaStreamWaitEvent(p.comp, p.loaded[b], 0));
    CUDA_OK(ch.work(b, p.buf[b], p.comp));
    CUDA_OK(cudaEventRecord(p.done[b], p.comp));
    CUDA_OK(cudaStreamWaitEvent(p.d2h, p.done[b], 0));
    CUDA_OK(cudaMemcpyAsync(ch.out, p.buf[b], ch.bytes, cudaMemcpyDeviceToHost, p.d2h));
    CUDA_OK(cudaEventRecord(p.drained[b], p.d2h));
  }
  // join: the d2h stream is in order, its last event covers every chunk
  if (!chunks.empty()) {
    const int last = static_cast<int>((chunks.size() - 1) % cemuComm::kPipeBufs);
    CUDA_OK(cudaStreamWaitEvent(s, p.drained[last], 0));
  }
  // capture needs every forked stream joined back
  if (capturing) {
    CUDA_OK(cudaEventRecord(p.loaded[0], p.h2d));
    CUDA_OK(cudaStreamWaitEvent(s, p.loaded[0], 0));
    CUDA_OK(cudaEventRecord(p.done[0], p.comp));
    CUDA_OK(cudaStreamWaitEvent(s, p.done[0], 0));
  }
  return cemuSuccess;
}

cemuResult_t host_allreduce(const void* send, void* recv, size_t count, int dt, cemuComm* c, cudaStream_t s) {
  const size_t es = dtype_size(dt);
  const uint64_t bytes = static_cast<uint64_t>(count) * es;
  // several real GPUs: chunks go through the fused kernel over symmetric
  // pipe buffers (rank-independent decision: every real rank pipelines)
  const bool fused = c->k > 1 && c->fused && es <= 4 && c->mode == PayloadMode::kHash && !c->virt.empty();
  if ((c->k > 1 && !fused) || c->mode != PayloadMode::kHash) {  // staged through device scratch
    if (auto r = ensure_scratch(c, bytes)) return r;
    CUDA_OK(cudaMemcpyAsync(c->scratch, send, bytes, cudaMemcpyHostToDevice, s));
    Phases ph;
    if (auto r = do_allreduce(c->scratch, c->scratch, count, dt, c, s, ph)) return r;
    for (auto& f : ph) {
      if (auto r = f()) return r;
    }
    CUDA_OK(cudaMemcpyAsync(recv, c->scratch, bytes, cudaMemcpyDeviceToHost, s));
    return cemuSuccess;
  }
  if (auto r = ensure_pipe(c)) return r;
  auto call = std::make_shared<Call>(c, kAllReduce, bytes, s);
  if (!call->error.empty()) return fail(cemuInvalidArgument, call->error);
  CUDA_OK(call->stamp_now());
  const uint64_t per = c->pipe.chunk / es;  // elements per chunk: a multiple of 4 (payload words)
  std::vector<PipeChunk> chunks;
  for (uint64_t e0 = 0; e0 < count; e0 += per) {
    const uint64_t n = std::min<uint64_t>(per, count - e0);
    PipeChunk ch;
    ch.in = static_cast<const uint8_t*>(send) + e0 * es;
    ch.out = static_cast<uint8_t*>(recv) + e0 * es;
    ch.bytes = n * es;
    const uint32_t nk = static_cast<uint32_t>(c->virt.size());
    if (fused) {
      ch.work = [c, call, dt, n, e0](int b, void*, cudaStream_t st) {
        FusedArgs a = fused_allreduce_args(c, dt, n, e0, c->pipe.peer[b], c->pipe.peer[b]);  // in place
        set_barrier(c, a);
        a.sig = op_sig(kAllReduce, dt, n, static_cast<uint64_t>(b) + 1);
        if (const cudaError_t e = cache_fused(c, dt, a, st, &call->launches)) return e;
        return launch_fused_allreduce(dt, a, st, &call->launches);
      };
    } else {
      ch.work = [c, call, dt, n, e0, nk](int, void* d, cudaStream_t st) {
        return synth_reduce(c, dt, d, d, n, e0, nullptr, st, &call->launches);
      };
    }
    chunks.push_back(std::move(ch));
  }
  if (auto r = run_pipe(c, s, chunks)) return r;
  CUDA_OK(call->finish(kAllReduce));
  return cemuSuccess;
}

cemuResult_t host_allgather(const void* send, void* recv, size_t sc, int dt, cemuComm* c, cudaStream_t s) {
  const size_t es = dtype_size(dt);
  const uint64_t blk = static_cast<uint64_t>(sc) * es;
  auto* r8 = static_cast<uint8_t*>(recv);
  if (c->k > 1 || c->mode != PayloadMode::kHash) {
    if (auto r = ensure_scratch(c, blk * c->W)) return r;
    auto* d8 = static_cast<uint8_t*>(c->scratch);
    CUDA_OK(cudaMemcpyAsync(d8 + c->rank * blk, send, blk, cudaMemcpyHostToDevice, s));
    Phases ph;
    if (auto r = do_allgather(d8 + c->rank * blk, d8, sc, dt, c, s, ph)) return r;
    for (auto& f : ph) {
      if (auto r = f()) return r;
    }
    CUDA_OK(cudaMemcpyAsync(recv, c->scratch, blk * c->W, cudaMemcpyDeviceToHost, s));
    return cemuSuccess;
  }
  if (auto r = ensure_pipe(c)) return r;
  auto call = std::make_shared<Call>(c, kAllGather, blk, s);
  if (!call->error.empty()) return fail(cemuInvalidArgument, call->error);
  CUDA_OK(call->stamp_now());
  // the own block (collective.cpp:289-291: in place it is already there)
  if (send != r8 + c->rank * blk) {
    CUDA_OK(cudaMemcpyAsync(r8 + c->rank * blk, send, blk, cudaMemcpyDefault, s));
  }
  const uint64_t per = c->pipe.chunk / es;
  std::vector<PipeChunk> chunks;
  for (size_t v = 0; v < c->virt.size(); ++v) {
    const uint32_t r = c->virt[v];
    const uint32_t key = payload_key(c->seed, r);
    for (uint64_t e0 = 0; e0 < sc; e0 += per) {
      const uint64_t n = std::min<uint64_t>(per, sc - e0);
      PipeChunk ch;
      ch.out = r8 + r * blk + e0 * es;
      ch.bytes = n * es;
      ch.work = [call, dt, n, e0, key](int, void* d, cudaStream_t st) {
        return launch_synth_fill(dt, d, n, nullptr, nullptr, 1, 0, key, nullptr, 0, nullptr, st, &call->launches,
                                 e0);
      };
      chunks.push_back(std::move(ch));
    }
  }
  if (auto r = run_pipe(c, s, chunks)) return r;
  CUDA_OK(call->finish(kAllGather));
  return cemuSuccess;
}

}  // namespace cemu_b200

extern "C" {

cemuResult_t cemuAllReduceHost(const void* send, void* recv, size_t count, cemuDataType_t dt, cemuRedOp_t op,
                               cemuComm_t c, cemuStream_t stream) {
  if (auto r = check_common(c, dt, "cemuAllReduceHost")) return r;
  if (auto r = check_op(op, "cemuAllReduceHost")) return r;
  if (count && (!send || !recv)) return fail(cemuInvalidArgument, "cemuAllReduceHost: null buffer");
  if (g_group_depth > 0) return fail(cemuInvalidUsage, "cemuAllReduceHost: host-buffer collectives cannot be grouped");
  if (c->wire) return fail(cemuInvalidUsage, "cemuAllReduceHost: not available in wire mode");
  if (count == 0) return cemuSuccess;
  try {
    const auto s = reinterpret_cast<cudaStream_t>(stream);
    if (auto r = order_begin(c, s)) return r;
    if (auto r = host_allreduce(send, recv, count, dt, c, s)) return r;
    return order_end(c, s);
  } catch (const std::exception& e) {
    return fail(cemuInternalError, e.what());
  }
}

cemuResult_t cemuAllGatherHost(const void* send, void* recv, size_t sc, cemuDataType_t dt, cemuComm_t c,
                               cemuStream_t stream) {
  if (auto r = check_common(c, dt, "cemuAllGatherHost")) return r;
  if (sc && (!send || !recv)) return fail(cemuInvalidArgument, "cemuAllGatherHost: null buffer");
  if (g_group_depth > 0) return fail(cemuInvalidUsage, "cemuAllGatherHost: host-buffer collectives cannot be grouped");
  if (c->wire) return fail(cemuInvalidUsage, "cemuAllGatherHost: not available in wire mode");
  if (sc == 0) return cemuSuccess;
  try {
    const auto s = reinterpret_cast<cudaStream_t>(stream);
    if (auto r = order_begin(c, s)) return r;
    if (auto r = host_allgather(send, recv, sc, dt, c, s)) return r;
    return order_end(c, s);
  } catch (const std::exception& e) {
    return fail(cemuInternalError, e.what());
  }
}

}  // extern "C"
