// harness.cpp -- see harness.hpp.
#include "harness.hpp"

#include <algorithm>
#include <cstdlib>
#include <sstream>
#include <stdexcept>

#include "config.hpp"
#include "kernels.hpp"

namespace cemu_b200 {

namespace {

std::string strip(const std::string& s) {
  const char* ws = " \t\r\n";
  const size_t b = s.find_first_not_of(ws);
  if (b == std::string::npos) return {};
  return s.substr(b, s.find_last_not_of(ws) - b + 1);
}

#define CK(expr)                                                                            \
  do {                                                                                      \
    const cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

}  // namespace

// harness.cpp:27-101 of the reference: same keys, same errors.
ModelSpec parse_model_spec(const std::string& text) {
  ModelSpec m;
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  bool have_iters = false;
  while (std::getline(in, line)) {
    ++lineno;
    const size_t hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    line = strip(line);
    if (line.empty()) continue;
    const size_t eq = line.find('=');
    if (eq == std::string::npos) {
      throw ConfigError("model line " + std::to_string(lineno) + ": expected key = value");
    }
    const std::string key = strip(line.substr(0, eq));
    const std::string val = strip(line.substr(eq + 1));
    auto u64 = [&](const std::string& v) {
      char* end = nullptr;
      const unsigned long long r = std::strtoull(v.c_str(), &end, 10);
      if (v.empty() || *end != '\0') {
        throw ConfigError("model " + key + ": expected integer, got '" + v + "'");
      }
      return static_cast<uint64_t>(r);
    };
    if (key == "name") {
      m.name = val;
    } else if (key == "iterations") {
      m.iterations = static_cast<uint32_t>(u64(val));
      have_iters = true;
    } else if (key == "warmup") {
      m.warmup_iterations = static_cast<uint32_t>(u64(val));
    } else if (key == "update_us") {
      m.update_us = static_cast<int64_t>(u64(val));
    } else if (key == "layer") {
      std::istringstream ls(val);
      LayerSpec l;
      if (!(ls >> l.forward_us >> l.backward_us >> l.grad_bytes)) {
        throw ConfigError("model layer: expected 'forward_us backward_us grad_bytes', got '" + val + "'");
      }
      std::string extra;
      if (ls >> extra) throw ConfigError("model layer: trailing token '" + extra + "'");
      if (l.forward_us < 0 || l.backward_us < 0) throw ConfigError("model layer: durations must be >= 0");
      m.layers.push_back(l);
    } else {
      throw ConfigError("model " + key + ": unknown key");
    }
  }
  if (m.layers.empty()) throw ConfigError("model: needs at least one layer");
  if (!have_iters || m.iterations == 0) throw ConfigError("model iterations: must be >= 1");
  if (m.warmup_iterations >= m.iterations) throw ConfigError("model warmup: must be < iterations");
  return m;
}

std::string render_model_spec(const ModelSpec& m) {
  std::ostringstream o;
  o << "name = " << m.name << "\n"
    << "iterations = " << m.iterations << "\n"
    << "warmup = " << m.warmup_iterations << "\n"
    << "update_us = " << m.update_us << "\n";
  for (const auto& l : m.layers) {
    o << "layer = " << l.forward_us << " " << l.backward_us << " " << l.grad_bytes << "\n";
  }
  return o.str();
}

// harness.cpp:116-134: the three built-in profiles
bool builtin_model(const std::string& name, ModelSpec* out) {
  ModelSpec m;
  m.name = name;
  m.iterations = 60;
  m.warmup_iterations = 10;
  if (name == "bert-like") {
    m.layers.assign(4, LayerSpec{1000, 2000, 64 * 1024});
  } else if (name == "small") {
    m.layers.assign(2, LayerSpec{1000, 2000, 32 * 1024});
  } else if (name == "wide") {
    m.layers.assign(16, LayerSpec{1000, 1000, 64 * 1024});
  } else {
    return false;
  }
  *out = m;
  return true;
}

// harness.cpp:152-175: greedy fill in reverse layer order, close on overflow
std::vector<Bucket> bucketize(const ModelSpec& m, uint64_t bucket_bytes) {
  std::vector<Bucket> out;
  Bucket cur;
  bool open = false;
  for (size_t k = m.layers.size(); k-- > 0;) {
    const uint64_t b = m.layers[k].grad_bytes;
    if (open && cur.bytes + b > bucket_bytes) {
      out.push_back(cur);
      open = false;
    }
    if (!open) {
      cur = Bucket{static_cast<uint32_t>(k), static_cast<uint32_t>(k), 0};
      open = true;
    }
    cur.first_layer = static_cast<uint32_t>(k);
    cur.bytes += b;
  }
  if (open) out.push_back(cur);
  return out;
}

std::vector<IterTrace> run_training_loop(cemuComm_t comm, const ModelSpec& m, uint64_t bucket_bytes) {
  int dev = 0;
  if (cemuCommCuDevice(comm, &dev) != cemuSuccess) throw std::runtime_error("harness: bad comm");
  CK(cudaSetDevice(dev));
  const std::vector<Bucket> buckets = bucketize(m, bucket_bytes);
  const size_t nb = buckets.size();
  cudaStream_t compute = nullptr, net = nullptr;
  CK(cudaStreamCreateWithFlags(&compute, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&net, cudaStreamNonBlocking));
  std::vector<uint8_t*> grads(nb, nullptr);
  for (size_t b = 0; b < nb; ++b) {
    CK(cudaMalloc(&grads[b], std::max<uint64_t>(buckets[b].bytes, 1)));
    CK(cudaMemset(grads[b], 0, std::max<uint64_t>(buckets[b].bytes, 1)));
  }
  // events: t0, then per iteration start/end and per bucket issue/complete
  const size_t per_it = 2 + 2 * nb;
  std::vector<cudaEvent_t> ev(1 + per_it * m.iterations);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  int spins = 0;
  // compute timeline chained on absolute device deadlines (see spin_ns_kernel)
  int64_t* chain = nullptr;
  CK(cudaMalloc(&chain, sizeof(int64_t)));
  bool resync = true;
  auto compute_us = [&](int64_t us) {
    if (us <= 0) return;
    CK(launch_spin_ns(us * 1000, compute, &spins, chain, resync));
    resync = false;
  };
  CK(cudaEventRecord(ev[0], compute));
  // The loop enqueues its buckets back to back on one in-order comm stream,
  // so it models that channel: a bucket queued behind the previous one
  // starts on the wire when that one leaves it (cemuCommSetQueueChaining),
  // unless the caller chose a gap of its own.
  struct GapGuard {
    cemuComm_t c;
    int64_t prev;
    ~GapGuard() { exchange_queue_gap_ns(c, prev); }
  } gap_guard{comm, exchange_queue_gap_ns(comm, 0)};
  exchange_queue_gap_ns(comm, gap_guard.prev > 0 ? gap_guard.prev : 10'000);
  const uint32_t L = static_cast<uint32_t>(m.layers.size());
  for (uint32_t it = 0; it < m.iterations; ++it) {
    cudaEvent_t* E = ev.data() + 1 + per_it * it;
    CK(cudaEventRecord(E[0], compute));
    for (const auto& l : m.layers) compute_us(l.forward_us);
    size_t next = 0;
    for (uint32_t i = L; i-- > 0;) {
      compute_us(m.layers[i].backward_us);
      if (next < nb && buckets[next].first_layer == i) {
        // bucket full: hand it to the in-order comm stream
        CK(cudaEventRecord(E[2 + 2 * next], compute));
        CK(cudaStreamWaitEvent(net, E[2 + 2 * next], 0));
        if (buckets[next].bytes) {
          const cemuResult_t r = cemuAllReduce(grads[next], grads[next], buckets[next].bytes, cemuUint8,
                                               cemuSum, comm, reinterpret_cast<cemuStream_t>(net));
          if (r != cemuSuccess) throw std::runtime_error(std::string("harness allreduce: ") + cemuGetLastError(comm));
        }
        CK(cudaEventRecord(E[3 + 2 * next], net));
        ++next;
      }
    }
    // wait-all (harness.cpp:235-247): the comm stream is in order, so its
    // last event implies every bucket
    if (nb) {
      CK(cudaStreamWaitEvent(compute, E[3 + 2 * (nb - 1)], 0));
      // the compute stream may have waited on the network: continue the
      // chain from the later of the two timelines (or from the next
      // kernel's own start when the network end is not on the device)
      if (const int64_t* net_end = resync ? nullptr : stream_release_end(comm, net)) {
        CK(launch_chain_join(chain, net_end, compute, &spins));
      } else {
        resync = true;
      }
    }
    compute_us(m.update_us);
    CK(cudaEventRecord(E[1], compute));
  }
  CK(cudaStreamSynchronize(compute));
  CK(cudaStreamSynchronize(net));
  std::vector<IterTrace> out(m.iterations);
  auto at = [&](cudaEvent_t e) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev[0], e));
    return static_cast<double>(ms) * 1e3;
  };
  for (uint32_t it = 0; it < m.iterations; ++it) {
    cudaEvent_t* E = ev.data() + 1 + per_it * it;
    out[it].start_us = at(E[0]);
    out[it].end_us = at(E[1]);
    for (size_t b = 0; b < nb; ++b) {
      out[it].issue_us.push_back(at(E[2 + 2 * b]));
      out[it].complete_us.push_back(at(E[3 + 2 * b]));
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (auto* g : grads) cudaFree(g);
  cudaFree(chain);
  cudaStreamDestroy(compute);
  cudaStreamDestroy(net);
  return out;
}

double predicted_iteration_us(const ModelSpec& m, uint64_t bucket_bytes,
                              const std::vector<double>& lat) {
  const std::vector<Bucket> buckets = bucketize(m, bucket_bytes);
  double t = 0;
  for (const auto& l : m.layers) t += static_cast<double>(l.forward_us);
  double net_free = 0;  // one op in flight, in issue order
  size_t next = 0;
  for (size_t i = m.layers.size(); i-- > 0;) {
    t += static_cast<double>(m.layers[i].backward_us);
    if (next < buckets.size() && buckets[next].first_layer == i) {
      const double start = std::max(t, net_free);
      net_free = start + (buckets[next].bytes && next < lat.size() ? lat[next] : 0.0);
      ++next;
    }
  }
  return std::max(t, net_free) + static_cast<double>(m.update_us);
}

}  // namespace cemu_b200
