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
