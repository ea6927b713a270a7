// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI driver around the reference `cemu_core` library, compiled from the
// reference sources where they lie (/root/reference/proj/src/*.cpp) by
// oracle/Makefile into oracle/_ref/libcemu_ref.so.  Nothing here is product
// code: only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
// --impl reference) may load it, and only as the checker / the CPU baseline.
//
// Every entry point calls the reference's own API; none restates it:
//   config render/digest ........ proj/src/config.cpp:153-312
//   chunking ..................... proj/src/dag.cpp:32-46
//   DAG / boundary dumps ......... proj/src/dag.cpp:90-137, 232-338, 362-393
//   delay model + offsets ........ proj/src/delay.cpp:5-47
//   OpState floors / release ..... proj/src/engine.cpp:18-126
//   reduce kernels ............... proj/src/reduce.cpp:42-60
//   emulated collective .......... WorkerSession (proj/src/collective.cpp)
//                                  against an in-thread EmulatorServer
//                                  (proj/src/emulator.cpp), the pattern of
//                                  proj/tests/test_transport.cpp:38-54
//   all-real ring ................ n WorkerSessions in threads
//                                  (proj/tests/test_transport.cpp:218-237)
//   emulator server .............. EmulatorServer serving in a thread, for
//                                  the B200 wire-mode interop tests
//                                  (proj/tools/cemu_emulator.cpp's role)
#include <netinet/in.h>
#include <sys/socket.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <set>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "cemu/clock.hpp"
#include "cemu/collective.hpp"
#include "cemu/config.hpp"
#include "cemu/dag.hpp"
#include "cemu/delay.hpp"
#include "cemu/emulator.hpp"
#include "cemu/engine.hpp"
#include "cemu/harness.hpp"
#include "cemu/reduce.hpp"
#include "cemu/trace.hpp"

using namespace cemu;

namespace {

void put_err(char* err, size_t cap, const std::string& s) {
  if (!err || cap == 0) return;
  const size_t n = std::min(cap - 1, s.size());
  std::memcpy(err, s.data(), n);
  err[n] = '\0';
}

int put_text(char* out, size_t cap, const std::string& s) {
  if (s.size() + 1 > cap) return -static_cast<int>(s.size() + 1);
  std::memcpy(out, s.data(), s.size());
  out[s.size()] = '\0';
  return static_cast<int>(s.size());
}

uint16_t free_port() {
  int fd = ::socket(AF_INET, SOCK_STREAM, 0);
  sockaddr_in a{};
  a.sin_family = AF_INET;
  a.sin_addr.s_addr = htonl(INADDR_LOOPBACK);
  a.sin_port = 0;
  ::bind(fd, reinterpret_cast<sockaddr*>(&a), sizeof a);
  socklen_t len = sizeof a;
  ::getsockname(fd, reinterpret_cast<sockaddr*>(&a), &len);
  const uint16_t p = ntohs(a.sin_port);
  ::close(fd);
  return p;
}

CollKind coll_of(int c) {
  return c == 0 ? CollKind::kAllReduce : CollKind::kAllGather;
}

std::set<uint32_t> real_set(const uint32_t* real, int nreal) {
  std::set<uint32_t> s;
  for (int i = 0; i < nreal; ++i) s.insert(real[i]);
  return s;
}

DelayModelParams delay_params(int kind, double a, double b, double g,
                              double fixed, double inject) {
  DelayModelParams p;
  p.kind = static_cast<DelayKind>(kind);  // 0 none, 1 alpha_beta, 2 fixed
  p.link = LinkParams{a, b, g};
  p.fixed_us = fixed;
  p.inject_us = inject;
  return p;
}

// JobConfig for a one-real-rank emulated job (test_transport.cpp:18-30) or an
// all-real baseline job (test_transport.cpp:32-39).
JobConfig make_cfg(uint32_t n, bool emulated, const DelayModelParams& d) {
  JobConfig cfg;
  cfg.world_size = n;
  cfg.real_ranks = {0};
  cfg.node_class.assign(n, "default");
  cfg.bucket_bytes = 1 << 20;
  cfg.link = d.link;
  cfg.delay_kind = d.kind;
  cfg.delay_fixed_us = d.fixed_us;
  cfg.delay_inject_us = d.inject_us;
  const uint16_t p0 = free_port();
  cfg.endpoints.push_back(Endpoint{"127.0.0.1", p0});
  const uint16_t pe = emulated ? free_port() : 0;
  for (uint32_t r = 1; r < n; ++r) {
    cfg.endpoints.push_back(
        Endpoint{"127.0.0.1", emulated ? pe : free_port()});
  }
  return cfg;
}

}  // namespace

extern "C" {

// ---- config (config.cpp:153-312) -----------------------------------------
// Parses `text`, writes the canonical render into `out` and the FNV-1a digest
// into *digest. Returns the render length, or -1 with the ConfigError text in
// `err`, or -(needed) if `out` is too small.
int ref_config_render(const char* text, char* out, size_t cap,
                      uint64_t* digest, char* err, size_t errcap) {
  try {
    const JobConfig cfg = parse_job_config(text);
    *digest = config_digest(cfg);
    return put_text(out, cap, render_job_config(cfg));
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return -1;
  }
}

// ---- chunking (dag.cpp:32-46) ----------------------------------------------
uint64_t ref_chunk_bytes(uint32_t n, uint64_t total, uint32_t elem,
                         uint32_t c) {
  return chunk_bytes(n, total, elem, c);
}
uint64_t ref_chunk_offset_bytes(uint32_t n, uint64_t total, uint32_t elem,
                                uint32_t c) {
  return chunk_offset_bytes(n, total, elem, c);
}

// ---- dumps (dag.cpp:362-393) -----------------------------------------------
int ref_dump_dag(int coll, uint32_t n, uint64_t bytes, uint32_t elem,
                 uint32_t op_id, char* out, size_t cap, char* err,
                 size_t errcap) {
  try {
    return put_text(out, cap,
                    dump_dag(build_collective_dag(coll_of(coll), n, bytes,
                                                  op_id, elem)));
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return -1;
  }
}

int ref_dump_boundary(int coll, uint32_t n, uint64_t bytes, uint32_t elem,
                      const uint32_t* real, int nreal, int side, char* out,
                      size_t cap, char* err, size_t errcap) {
  try {
    const CollectiveDag dag =
        build_collective_dag(coll_of(coll), n, bytes, 0, elem);
    return put_text(
        out, cap,
        dump_boundary(project_boundary(
            dag, real_set(real, nreal),
            side == 0 ? BoundarySide::kEmulated : BoundarySide::kReal)));
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return -1;
  }
}

// ---- delay model (delay.cpp:5-47) ------------------------------------------
double ref_ring_allreduce_delay_us(uint32_t n, uint64_t bytes, double a,
                                   double b, double g) {
  return ring_allreduce_delay_us(n, bytes, LinkParams{a, b, g});
}
double ref_ring_allgather_delay_us(uint32_t n, uint64_t bytes, double a,
                                   double b) {
  return ring_allgather_delay_us(n, bytes, LinkParams{a, b, 0.0});
}

// Offsets for every to-real vertex of the emulated-side boundary. Returns K
// (the to-real count) or -1 on error; writes min(K, cap) offsets.
int ref_release_offsets(int coll, uint32_t n, uint64_t bytes, uint32_t elem,
                        const uint32_t* real, int nreal, int kind, double a,
                        double b, double g, double fixed, double inject,
                        double* out, size_t cap, char* err, size_t errcap) {
  try {
    const CollectiveDag dag =
        build_collective_dag(coll_of(coll), n, bytes, 0, elem);
    const BoundaryDag bd = project_boundary(dag, real_set(real, nreal));
    const auto off =
        release_offsets_us(bd, delay_params(kind, a, b, g, fixed, inject),
                           bytes);
    for (size_t i = 0; i < off.size() && i < cap; ++i) out[i] = off[i];
    return static_cast<int>(off.size());
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return -1;
  }
}

// Release floors exactly as OpState computes them (engine.cpp:36-42):
// now_us + llround(offset).
int ref_opstate_floors(int coll, uint32_t n, uint64_t bytes, uint32_t elem,
                       const uint32_t* real, int nreal, int kind, double a,
                       double b, double g, double fixed, double inject,
                       int64_t now, int64_t* out, size_t cap, char* err,
                       size_t errcap) {
  try {
    const CollectiveDag dag =
        build_collective_dag(coll_of(coll), n, bytes, 0, elem);
    auto bd = std::make_shared<BoundaryDag>(
        project_boundary(dag, real_set(real, nreal)));
    const auto off = release_offsets_us(
        *bd, delay_params(kind, a, b, g, fixed, inject), bytes);
    OpState st(0, bd, off, now);
    for (size_t i = 0; i < off.size() && i < cap; ++i) {
      out[i] = st.release_not_before_us(i);
    }
    return static_cast<int>(off.size());
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return -1;
  }
}

// Drives OpState on a virtual clock against an instantaneous model real node
// (the ModelPeer of tests/test_engine.cpp:28-63): the real node sends its
// from-real message at step p as soon as the to-real reply of step p-1 has
// been released. Returns completion - registration in us (A14), and the
// release time of every to-real message in `release` (K entries).
int64_t ref_simulated_call_latency_us(int coll, uint32_t n, uint64_t bytes,
                                      uint32_t elem, int kind, double a,
                                      double b, double g, double fixed,
                                      double inject, int64_t* release,
                                      size_t cap, char* err, size_t errcap) {
  try {
    const CollectiveDag dag =
        build_collective_dag(coll_of(coll), n, bytes, 0, elem);
    auto bd = std::make_shared<BoundaryDag>(project_boundary(dag, {0}));
    const auto off = release_offsets_us(
        *bd, delay_params(kind, a, b, g, fixed, inject), bytes);
    std::vector<MsgDesc> sends, expected;
    for (const auto& v : bd->vertices) {
      (v.dir == BoundaryDir::kFromReal ? sends : expected).push_back(v.msg);
    }
    OpState st(0, bd, off, 0);
    int64_t now = 0;
    size_t sent = 0, received = 0;
    auto received_step = [&](uint32_t step) {
      for (size_t i = 0; i < received; ++i) {
        if (expected[i].step == step) return true;
      }
      return false;
    };
    for (int guard = 0; guard < 10000000; ++guard) {
      bool progressed = false;
      while (sent < sends.size() &&
             (sends[sent].step == 0 || received_step(sends[sent].step - 1))) {
        if (st.on_receive_from_real(sends[sent])) {
          throw std::runtime_error("protocol error in model peer");
        }
        ++sent;
        progressed = true;
      }
      while (auto m = st.try_send_to_real(now)) {
        if (received < cap) release[received] = now;
        ++received;
        progressed = true;
      }
      if (st.is_complete()) return now;
      if (!progressed) {
        const auto next = st.next_release_at_us();
        if (!next) throw std::runtime_error("deadlock in model run");
        now = std::max(now, *next);
      }
    }
    throw std::runtime_error("model run did not terminate");
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return -1;
  }
}

// ---- reduce kernels (reduce.cpp:42-60) -------------------------------------
void ref_reduce_add_i32(int32_t* dst, const int32_t* src, size_t count) {
  reduce_add_i32(dst, src, count);
}
void ref_reduce_add_u8(uint8_t* dst, const uint8_t* src, size_t count) {
  reduce_add_u8(dst, src, count);
}
const char* ref_reduce_backend() { return reduce_backend(); }

// ---- emulated collective over loopback -------------------------------------
// Rank 0 is the only real rank; ranks 1..n-1 are served by an in-thread
// EmulatorServer. `buf` is the real rank's buffer (plan bytes for allreduce,
// n * plan bytes for allgather). Runs warmup+reps synchronous calls on the
// same buffer, the way tools/cemu_coll.cpp:136-146 times them, and writes the
// per-call wall time (us) of the timed reps into `times_us`. The last call's
// result is left in `buf`. Returns 0, or -1 with the error in `err`.
int ref_emulated_collective(uint32_t n, int coll, uint8_t* buf,
                            uint64_t plan_bytes, uint32_t elem, int kind,
                            double a, double b, double g, double fixed,
                            double inject, int warmup, int reps,
                            double* times_us, char* err, size_t errcap) {
  // Concurrent callers (the bench's multi-session reference arm): choosing
  // loopback ports, binding the emulator and the worker's listener, and the
  // handshake happen under one process-wide lock, so two sessions can never
  // pick the same port; the timed calls run unlocked.
  static std::mutex setup_mu;
  std::unique_lock<std::mutex> setup(setup_mu);
  try {
    const DelayModelParams d = delay_params(kind, a, b, g, fixed, inject);
    const JobConfig cfg = make_cfg(n, /*emulated=*/true, d);
    EmulatorServer::Options o;
    o.once = true;
    EmulatorServer server(cfg, o);
    std::thread th([&] { server.serve(); });
    std::string failure;
    try {
      std::vector<CollectivePlanEntry> plan = {
          {coll_of(coll), plan_bytes, elem}};
      WorkerSession s(cfg, 0, plan);
      setup.unlock();
      const uint64_t len = coll == 0 ? plan_bytes : plan_bytes * n;
      std::span<uint8_t> sp(buf, len);
      for (int i = 0; i < warmup + reps; ++i) {
        const int64_t t0 = now_us();
        if (coll == 0) {
          s.allreduce(sp, elem);
        } else {
          s.allgather(sp, elem);
        }
        const int64_t t1 = now_us();
        if (i >= warmup && times_us) {
          times_us[i - warmup] = static_cast<double>(t1 - t0);
        }
      }
      s.close();
    } catch (const std::exception& e) {
      failure = e.what();
    }
    if (setup.owns_lock()) setup.unlock();
    server.request_stop();
    th.join();
    if (!failure.empty()) throw std::runtime_error(failure);
    return 0;
  } catch (const std::exception& e) {
    if (setup.owns_lock()) setup.unlock();
    put_err(err, errcap, e.what());
    return -1;
  }
}

// ---- all-real ring ---------------------------------------------------------
// n real WorkerSessions in threads, one buffer per rank, one call each.
int ref_real_ring(uint32_t n, int coll, uint8_t** bufs, uint64_t plan_bytes,
                  uint32_t elem, char* err, size_t errcap) {
  try {
    // Baseline mode of test_transport.cpp:32-39: the config keeps
    // real_ranks = {0} (validate() wants a strict subset) and real workers
    // simply answer at every endpoint; WorkerSession never consults the set.
    const JobConfig cfg = make_cfg(n, /*emulated=*/false, DelayModelParams{});
    std::vector<CollectivePlanEntry> plan = {
        {coll_of(coll), plan_bytes, elem}};
    const uint64_t len = coll == 0 ? plan_bytes : plan_bytes * n;
    std::vector<std::string> errors(n);
    std::vector<std::thread> ths;
    for (uint32_t r = 0; r < n; ++r) {
      ths.emplace_back([&, r] {
        try {
          WorkerSession s(cfg, r, plan);
          std::span<uint8_t> sp(bufs[r], len);
          if (coll == 0) {
            s.allreduce(sp, elem);
          } else {
            s.allgather(sp, elem);
          }
          s.close();
        } catch (const std::exception& e) {
          errors[r] = e.what();
        }
      });
    }
    for (auto& t : ths) t.join();
    for (uint32_t r = 0; r < n; ++r) {
      if (!errors[r].empty()) {
        throw std::runtime_error("rank " + std::to_string(r) + ": " +
                                 errors[r]);
      }
    }
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return -1;
  }
}

// ---- EventLog (trace.cpp:9-46) ----------------------------------------------
void ref_trace_open(const char* path) { global_event_log().open(path ? path : ""); }

// ---- model spec + bucketing (harness.cpp:27-189) ---------------------------
int ref_model_render(const char* text, char* out, size_t cap, char* err, size_t errcap) {
  try {
    return put_text(out, cap, render_model_spec(parse_model_spec(text)));
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return -1;
  }
}

// Returns the bucket count (or -1); writes (first, last, bytes) triples.
int ref_bucketize(const char* text, uint64_t bucket_bytes, uint64_t* out, size_t cap, char* err,
                  size_t errcap) {
  try {
    const auto b = bucketize(parse_model_spec(text), bucket_bytes);
    for (size_t i = 0; i < b.size() && 3 * i + 2 < cap; ++i) {
      out[3 * i] = b[i].first_layer;
      out[3 * i + 1] = b[i].last_layer;
      out[3 * i + 2] = b[i].bytes;
    }
    return static_cast<int>(b.size());
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return -1;
  }
}

// ---- the reference's synthetic DDP loop (harness.cpp:191-254) -----------
// run_training_loop on WorkerSession(rank 0) against an in-thread emulator,
// world n, bucket_bytes from the caller, delay params as above.  Writes each
// iteration's wall time (us) to iter_us and returns the iteration count, or
// -1 with the error in `err`.
int ref_run_training_loop(const char* model_text, uint32_t n, uint64_t bucket_bytes, int kind, double a,
                          double b, double g, double fixed, double inject, double* iter_us, size_t cap,
                          char* err, size_t errcap) {
  try {
    const ModelSpec model = parse_model_spec(model_text);
    JobConfig cfg = make_cfg(n, /*emulated=*/true, delay_params(kind, a, b, g, fixed, inject));
    cfg.bucket_bytes = bucket_bytes;
    EmulatorServer::Options o;
    o.once = true;
    EmulatorServer server(cfg, o);
    std::thread th([&] { server.serve(); });
    std::string failure;
    std::vector<IterationTrace> traces;
    try {
      WorkerSession s(cfg, 0, harness_plan(model, bucket_bytes));
      traces = run_training_loop(cfg, model, s);
      s.close();
    } catch (const std::exception& e) {
      failure = e.what();
    }
    server.request_stop();
    th.join();
    if (!failure.empty()) throw std::runtime_error(failure);
    for (size_t i = 0; i < traces.size() && i < cap; ++i) {
      iter_us[i] = static_cast<double>(traces[i].iteration_time_us());
    }
    return static_cast<int>(traces.size());
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return -1;
  }
}



// ---- a reference emulator process, in a thread ------------------------------
// Parses `cfg_text` with the reference parser, binds the emulator endpoint
// (emulator.cpp:14-39) and serves sessions until ref_emulator_stop.  Returns
// a handle, or null with the ConfigError/NetError text in `err`.
struct RefEmulator {
  std::unique_ptr<EmulatorServer> server;
  std::thread th;
};

void* ref_emulator_start(const char* cfg_text, char* err, size_t errcap) {
  try {
    const JobConfig cfg = parse_job_config(cfg_text);
    auto* h = new RefEmulator;
    h->server = std::make_unique<EmulatorServer>(cfg);
    h->th = std::thread([h] { h->server->serve(); });
    return h;
  } catch (const std::exception& e) {
    put_err(err, errcap, e.what());
    return nullptr;
  }
}

uint64_t ref_emulator_sessions(void* h) {
  return h ? static_cast<RefEmulator*>(h)->server->sessions_served() : 0;
}

void ref_emulator_stop(void* hv) {
  auto* h = static_cast<RefEmulator*>(hv);
  if (!h) return;
  h->server->request_stop();  // serve() polls the flag every 200 ms
  if (h->th.joinable()) h->th.join();
  delete h;
}

// config_digest of the reference parser (for the interop tests)
uint64_t ref_config_digest(const char* cfg_text) {
  try {
    return config_digest(parse_job_config(cfg_text));
  } catch (const std::exception&) {
    return 0;
  }
}

}  // extern "C"
