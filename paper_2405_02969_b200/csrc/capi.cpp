// capi.cpp -- C-ABI of the host-side pure functions (job config, schedule,
// delay model, payload generator).  See include/cemu_b200.h.
#include <cstring>
#include <string>
#include <vector>

#include "cemu_b200.h"
#include "config.hpp"
#include "payload.cuh"
#include "schedule.hpp"

using namespace cemu_b200;

struct cemuJobConfig {
  JobConfig cfg;
};

namespace {

void copy_err(char* err, size_t cap, const std::string& s) {
  if (!err || cap == 0) return;
  const size_t n = std::min(cap - 1, s.size());
  std::memcpy(err, s.data(), n);
  err[n] = '\0';
}

int copy_text(const std::string& s, char* out, size_t cap) {
  if (!out || s.size() + 1 > cap) return -static_cast<int>(s.size() + 1);
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

}  // namespace

extern "C" {

cemuResult_t cemuConfigParse(const char* text, cemuJobConfig_t* out, char* err, size_t errcap) {
  if (!text || !out) {
    copy_err(err, errcap, "cemuConfigParse: null argument");
    return cemuInvalidArgument;
  }
  try {
    *out = new cemuJobConfig{parse_job_config(text)};
    return cemuSuccess;
  } catch (const std::exception& e) {
    copy_err(err, errcap, e.what());
    return cemuInvalidArgument;
  }
}

cemuResult_t cemuConfigLoad(const char* path, cemuJobConfig_t* out, char* err, size_t errcap) {
  if (!path || !out) {
    copy_err(err, errcap, "cemuConfigLoad: null argument");
    return cemuInvalidArgument;
  }
  try {
    *out = new cemuJobConfig{load_job_config(path)};
    return cemuSuccess;
  } catch (const std::exception& e) {
    copy_err(err, errcap, e.what());
    return cemuInvalidArgument;
  }
}

void cemuConfigFree(cemuJobConfig_t cfg) { delete cfg; }

int cemuConfigRender(cemuJobConfig_t cfg, char* out, size_t cap) {
  if (!cfg) return 0;
  return copy_text(render_job_config(cfg->cfg), out, cap);
}

uint64_t cemuConfigDigest(cemuJobConfig_t cfg) { return cfg ? config_digest(cfg->cfg) : 0; }

uint32_t cemuConfigWorldSize(cemuJobConfig_t cfg) { return cfg ? cfg->cfg.world_size : 0; }

uint32_t cemuConfigRealRanks(cemuJobConfig_t cfg, uint32_t* out, size_t cap) {
  if (!cfg) return 0;
  size_t i = 0;
  for (uint32_t r : cfg->cfg.real_ranks) {
    if (out && i < cap) out[i] = r;
    ++i;
  }
  return static_cast<uint32_t>(i);
}

uint32_t cemuConfigTopology(cemuJobConfig_t cfg, cemuTopoNode* nodes, cemuTopoEdge* edges, size_t cap) {
  if (!cfg) return 0;
  const JobConfig& c = cfg->cfg;
  for (uint32_t r = 0; r < c.world_size && r < cap; ++r) {
    if (nodes) {
      nodes[r].isReal = c.is_real(r) ? 1 : 0;
      const std::string& nc = c.node_class[r];
      const size_t n = std::min<size_t>(nc.size(), sizeof nodes[r].nodeClass - 1);
      std::memcpy(nodes[r].nodeClass, nc.data(), n);
      nodes[r].nodeClass[n] = '\0';
    }
    if (edges) {
      edges[r].src = r;
      edges[r].dst = (r + 1) % c.world_size;
      edges[r].alphaUs = c.link.alpha_us;
      edges[r].betaUsPerByte = c.link.beta_us_per_byte;
      edges[r].gammaUsPerByte = c.link.gamma_us_per_byte;
    }
  }
  return c.world_size;
}

uint32_t cemuRingSuccessor(uint32_t n, uint32_t rank) { return n ? (rank + 1) % n : 0; }
uint32_t cemuRingPredecessor(uint32_t n, uint32_t rank) { return n ? (rank + n - 1) % n : 0; }

uint64_t cemuChunkBytes(uint32_t n, uint64_t total, uint32_t elem, uint32_t chunk) {
  return chunk_bytes(n, total, elem, chunk);
}

uint64_t cemuChunkOffsetBytes(uint32_t n, uint64_t total, uint32_t elem, uint32_t chunk) {
  return chunk_offset_bytes(n, total, elem, chunk);
}

uint32_t cemuPositions(int coll, uint32_t n) { return positions(coll, n); }

uint32_t cemuSendChunkAt(int coll, uint32_t n, uint32_t rank, uint32_t p) {
  return send_chunk_at(coll, n, rank, p);
}

int cemuBoundaryDump(int coll, uint32_t n, uint64_t bytes, uint32_t elem, uint32_t real, char* out,
                     size_t cap) {
  return copy_text(boundary_dump(coll, n, bytes, elem, real), out, cap);
}

uint32_t cemuToRealCount(int coll, uint32_t n, const uint32_t* real, uint32_t nreal) {
  return to_real_count(coll, n, std::vector<uint32_t>(real, real + nreal));
}

double cemuModelTotalUs(const cemuDelayModel* m, int coll, uint32_t n, uint64_t bytes) {
  return model_total(*m, coll, n, bytes);
}

int cemuReleaseOffsets(const cemuDelayModel* m, int coll, uint32_t n, uint64_t bytes, uint32_t k,
                       double* out) {
  const auto v = release_offsets(*m, coll, n, bytes, k);
  std::memcpy(out, v.data(), v.size() * sizeof(double));
  return static_cast<int>(k);
}

int cemuReleaseFloors(const cemuDelayModel* m, int coll, uint32_t n, uint64_t bytes, uint32_t k,
                      int64_t now_us, int64_t* out) {
  const auto v = release_floors(*m, coll, n, bytes, k, now_us);
  std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
  return static_cast<int>(k);
}

int64_t cemuCallLatencyUs(const cemuDelayModel* m, int coll, uint32_t n, uint64_t bytes, uint32_t k) {
  return call_latency_us(*m, coll, n, bytes, k);
}

uint32_t cemuPayloadKey(uint64_t seed, uint32_t rank) { return payload_key(seed, rank); }

uint32_t cemuPayloadWord(uint32_t key, uint64_t j) { return payload_word(key, j); }

}  // extern "C"

// ---------------------------------------------------------------------------
// harness (proj/src/harness.cpp) and compute emulation
// ---------------------------------------------------------------------------
#include <cuda_runtime.h>

#include "harness.hpp"
#include "kernels.hpp"

struct cemuModelSpec {
  ModelSpec m;
};

extern "C" {

cemuResult_t cemuModelSpecParse(const char* text, cemuModelSpec_t* out, char* err, size_t errcap) {
  if (!text || !out) {
    copy_err(err, errcap, "cemuModelSpecParse: null argument");
    return cemuInvalidArgument;
  }
  try {
    *out = new cemuModelSpec{parse_model_spec(text)};
    return cemuSuccess;
  } catch (const std::exception& e) {
    copy_err(err, errcap, e.what());
    return cemuInvalidArgument;
  }
}

cemuResult_t cemuModelSpecBuiltin(const char* name, cemuModelSpec_t* out) {
  ModelSpec m;
  if (!name || !out || !builtin_model(name, &m)) return cemuInvalidArgument;
  *out = new cemuModelSpec{m};
  return cemuSuccess;
}

void cemuModelSpecFree(cemuModelSpec_t m) { delete m; }

int cemuModelSpecRender(cemuModelSpec_t m, char* out, size_t cap) {
  return m ? copy_text(render_model_spec(m->m), out, cap) : 0;
}

uint32_t cemuModelSpecLayers(cemuModelSpec_t m, int64_t* fwd, int64_t* bwd, uint64_t* grad, size_t cap,
                             uint32_t* iterations, uint32_t* warmup, int64_t* update_us) {
  if (!m) return 0;
  const auto& L = m->m.layers;
  for (size_t i = 0; i < L.size() && i < cap; ++i) {
    if (fwd) fwd[i] = L[i].forward_us;
    if (bwd) bwd[i] = L[i].backward_us;
    if (grad) grad[i] = L[i].grad_bytes;
  }
  if (iterations) *iterations = m->m.iterations;
  if (warmup) *warmup = m->m.warmup_iterations;
  if (update_us) *update_us = m->m.update_us;
  return static_cast<uint32_t>(L.size());
}

uint32_t cemuBucketize(cemuModelSpec_t m, uint64_t bucketBytes, uint32_t* first, uint32_t* last, uint64_t* bytes,
                       size_t cap) {
  if (!m) return 0;
  const auto b = bucketize(m->m, bucketBytes);
  for (size_t i = 0; i < b.size() && i < cap; ++i) {
    if (first) first[i] = b[i].first_layer;
    if (last) last[i] = b[i].last_layer;
    if (bytes) bytes[i] = b[i].bytes;
  }
  return static_cast<uint32_t>(b.size());
}

cemuResult_t cemuRunTrainingLoop(cemuComm_t comm, cemuModelSpec_t m, uint64_t bucketBytes, double* iterStartUs,
                                 double* iterEndUs, double* issueUs, double* completeUs, size_t cap) {
  if (!comm || !m) return cemuInvalidArgument;
  try {
    const auto tr = run_training_loop(comm, m->m, bucketBytes);
    const size_t nb = bucketize(m->m, bucketBytes).size();
    for (size_t it = 0; it < tr.size() && it < cap; ++it) {
      if (iterStartUs) iterStartUs[it] = tr[it].start_us;
      if (iterEndUs) iterEndUs[it] = tr[it].end_us;
      for (size_t b = 0; b < nb; ++b) {
        if (issueUs) issueUs[it * nb + b] = tr[it].issue_us[b];
        if (completeUs) completeUs[it * nb + b] = tr[it].complete_us[b];
      }
    }
    return cemuSuccess;
  } catch (const std::exception& e) {
    (void)e;
    return cemuInternalError;
  }
}

double cemuPredictIterationUs(cemuModelSpec_t m, uint64_t bucketBytes, const double* bucketLatencyUs, size_t n) {
  if (!m) return -1;
  return predicted_iteration_us(m->m, bucketBytes, std::vector<double>(bucketLatencyUs, bucketLatencyUs + n));
}

cemuResult_t cemuSpinUs(cemuStream_t stream, uint64_t us) {
  int l = 0;
  return launch_spin_ns(static_cast<int64_t>(us) * 1000, reinterpret_cast<cudaStream_t>(stream), &l) == cudaSuccess
             ? cemuSuccess
             : cemuUnhandledCudaError;
}

cemuResult_t cemuSpinChainUs(cemuStream_t stream, uint64_t us, int64_t* chain, int resync) {
  if (!chain) return cemuInvalidArgument;
  int l = 0;
  return launch_spin_ns(static_cast<int64_t>(us) * 1000, reinterpret_cast<cudaStream_t>(stream), &l, chain,
                        resync != 0) == cudaSuccess
             ? cemuSuccess
             : cemuUnhandledCudaError;
}

cemuResult_t cemuChainJoin(cemuStream_t stream, int64_t* chain, const int64_t* other) {
  if (!chain || !other) return cemuInvalidArgument;
  int l = 0;
  return launch_chain_join(chain, other, reinterpret_cast<cudaStream_t>(stream), &l) == cudaSuccess
             ? cemuSuccess
             : cemuUnhandledCudaError;
}

}  // extern "C"
