// config.hpp -- the job description (world, real ranks, link model, delay
// injection) in the reference's key=value format, bit-compatible with
// proj/src/config.cpp:153-312: same keys, same validation and error text,
// same canonical render and FNV-1a-64 digest.  New keys (the gaps the
// reference does not cover) are rendered only when they differ from their
// defaults, so every reference config renders -- and digests -- identically.
//
//   collective_algo        ring (reference) | tree | hierarchical   (cost model)
//   topology.gpus_per_node ranks per node for the hierarchical model
//   link.intra.alpha_us / link.intra.beta_us_per_byte   intra-node links
//   payload.mode           hash (default) | zero (the reference's dummy zeros)
//   payload.seed           seed of the counter-based payload hash (default 1)
//   endpoint.R             optional here (all or none): the device path has
//                          no wire; the reference requires them.
#pragma once

#include <cstdint>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace cemu_b200 {

class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};

enum class DelayKind : int32_t { kNone = 0, kAlphaBeta = 1, kFixed = 2 };
enum class CostAlgo : int32_t { kRing = 0, kTree = 1, kHierarchical = 2 };
enum class PayloadMode : int32_t { kHash = 0, kZero = 1 };

struct Link {
  double alpha_us = 0.0;
  double beta_us_per_byte = 0.0;
  double gamma_us_per_byte = 0.0;
  bool operator==(const Link&) const = default;
};

struct Endpoint {
  std::string host;
  uint16_t port = 0;
  bool operator==(const Endpoint&) const = default;
  std::string str() const { return host + ":" + std::to_string(port); }
};

struct JobConfig {
  uint32_t world_size = 0;
  std::set<uint32_t> real_ranks;
  std::vector<std::string> node_class;
  Link link;
  std::string collective_algo = "ring";
  uint64_t bucket_bytes = 0;
  std::string chunk_policy = "one-chunk-per-partition";
  DelayKind delay_kind = DelayKind::kNone;
  double delay_fixed_us = 0.0;
  double delay_inject_us = 0.0;
  int64_t poll_period_us = 10;
  std::vector<Endpoint> endpoints;  // empty = not given (device path)
  // ---- extensions (rendered only when non-default) ----
  uint32_t gpus_per_node = 1;
  bool intra_set = false;
  double intra_alpha_us = 0.0;
  double intra_beta_us_per_byte = 0.0;
  PayloadMode payload_mode = PayloadMode::kHash;
  uint64_t payload_seed = 1;

  bool operator==(const JobConfig&) const = default;
  bool is_real(uint32_t r) const { return real_ranks.count(r) != 0; }
  CostAlgo algo() const;
};

JobConfig parse_job_config(const std::string& text);
JobConfig load_job_config(const std::string& path);
std::string render_job_config(const JobConfig& cfg);
uint64_t config_digest(const JobConfig& cfg);

}  // namespace cemu_b200
