// schedule.cpp -- see schedule.hpp.  Built with -ffp-contract=off.
#include "schedule.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <utility>

#include "delay_math.cuh"

namespace cemu_b200 {

uint64_t chunk_bytes(uint32_t n, uint64_t total, uint32_t elem, uint32_t c) {
  const uint64_t elems = total / elem;
  const uint64_t per = elems / n;
  return (per + (c + 1 == n ? elems % n : 0)) * elem;
}

uint64_t chunk_offset_bytes(uint32_t n, uint64_t total, uint32_t elem, uint32_t c) {
  return static_cast<uint64_t>(c) * ((total / elem) / n) * elem;
}

uint32_t positions(int coll, uint32_t n) { return coll == kAllReduce ? 2 * (n - 1) : n - 1; }

uint32_t send_chunk_at(int coll, uint32_t n, uint32_t rank, uint32_t p) {
  // (rank - p) mod n in the reduce-scatter phase and for allgather;
  // (rank + 1 - t) mod n at gather step t = p - (n - 1) of an allreduce.
  const int64_t nn = n;
  int64_t c;
  if (coll != kAllReduce || p + 1 < n) {
    c = static_cast<int64_t>(rank) - p;
  } else {
    c = static_cast<int64_t>(rank) + 1 - (static_cast<int64_t>(p) - (nn - 1));
  }
  c %= nn;
  return static_cast<uint32_t>(c < 0 ? c + nn : c);
}

// Single real rank R: crossing messages at every position p are
// from_real R->R+1 and to_real R-1->R; within a step the canonical order is
// by src rank.  Reduced edges: to_real@p -> from_real@p+1 (program order of
// the real node) and, for allreduce, from_real@p -> to_real@p+n-1 (the chunk
// travels n-1 hops through the emulated ring before it returns).
std::string boundary_dump(int coll, uint32_t n, uint64_t bytes, uint32_t elem, uint32_t R) {
  const uint32_t P = positions(coll, n);
  const uint32_t prev = (R + n - 1) % n, next = (R + 1) % n;
  const bool from_first = R < prev;
  std::string s = "# boundary ";
  s += coll == kAllReduce ? "allreduce" : "allgather";
  s += " n=" + std::to_string(n) + " side=emulated\n";
  char line[160];
  for (uint32_t p = 0; p < P; ++p) {
    for (int i = 0; i < 2; ++i) {
      const bool from = (i == 0) == from_first;
      const uint32_t src = from ? R : prev;
      const uint32_t c = send_chunk_at(coll, n, src, p);
      const uint64_t sz = coll == kAllReduce ? chunk_bytes(n, bytes, elem, c) : bytes;
      std::snprintf(line, sizeof line, "0 %s %u %u %u %u %llu\n",
                    from ? "from_real:recv" : "to_real:send", p, src, from ? next : R, c,
                    static_cast<unsigned long long>(sz));
      s += line;
    }
  }
  s += "edges\n";
  auto fr = [&](uint32_t p) { return 2 * p + (from_first ? 0u : 1u); };
  auto tr = [&](uint32_t p) { return 2 * p + (from_first ? 1u : 0u); };
  std::vector<std::pair<uint32_t, uint32_t>> e;
  for (uint32_t p = 0; p + 1 < P; ++p) e.emplace_back(tr(p), fr(p + 1));
  if (coll == kAllReduce) {
    for (uint32_t p = 0; p + n - 1 < P; ++p) e.emplace_back(fr(p), tr(p + n - 1));
  }
  std::sort(e.begin(), e.end());
  for (auto [u, v] : e) s += std::to_string(u) + " " + std::to_string(v) + "\n";
  return s;
}

uint32_t to_real_count(int coll, uint32_t n, const std::vector<uint32_t>& real) {
  std::vector<bool> is(n, false);
  for (uint32_t r : real) {
    if (r < n) is[r] = true;
  }
  uint32_t edges = 0;  // ring edges v -> v+1 entering the real set
  for (uint32_t v = 0; v < n; ++v) {
    if (!is[v] && is[(v + 1) % n]) ++edges;
  }
  return edges * positions(coll, n);
}

double model_total(const cemuDelayModel& m, int coll, uint32_t n, uint64_t bytes) {
  return model_total_us(m, coll, n, bytes);
}

std::vector<double> release_offsets(const cemuDelayModel& m, int coll, uint32_t n,
                                    uint64_t bytes, uint32_t k) {
  std::vector<double> out(k);
  const double total = m.kind == 1 ? model_total_us(m, coll, n, bytes) : 0.0;
  for (uint32_t j = 0; j < k; ++j) out[j] = release_offset_us(m, total, j, k);
  return out;
}

std::vector<int64_t> release_floors(const cemuDelayModel& m, int coll, uint32_t n,
                                    uint64_t bytes, uint32_t k, int64_t now_us) {
  std::vector<int64_t> out(k);
  const auto off = release_offsets(m, coll, n, bytes, k);
  for (uint32_t j = 0; j < k; ++j) out[j] = now_us + static_cast<int64_t>(std::llround(off[j]));
  return out;
}

int64_t call_latency_us(const cemuDelayModel& m, int coll, uint32_t n, uint64_t bytes,
                        uint32_t k) {
  int64_t best = 0;
  for (int64_t f : release_floors(m, coll, n, bytes, k, 0)) best = std::max(best, f);
  return best;
}

}  // namespace cemu_b200
