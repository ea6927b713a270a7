// harness.hpp -- the synthetic data-parallel training loop on the B200
// (the DDP bucket what-if curve).
//
// Same model-spec format and bucketing as the reference
// (proj/src/harness.cpp:27-189): layers of (forward_us, backward_us,
// grad_bytes), gradients bucketed greedily in reverse layer order, one
// allreduce (elem_size 1) per bucket.  The loop itself is re-expressed on
// the device: layer compute is a %globaltimer spin kernel on a compute
// stream (the analogue of emulate_compute_us, clock.hpp:29-37), each filled
// bucket's emulated allreduce goes to an in-order comm stream (the
// reference's one-op-in-flight engine, collective.cpp:357-404) after an
// event from the compute stream, and the wait-all joins the streams.  All
// timestamps are device events, so the measured timeline contains no host
// jitter.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "cemu_b200.h"

namespace cemu_b200 {

struct LayerSpec {
  int64_t forward_us = 0;
  int64_t backward_us = 0;
  uint64_t grad_bytes = 0;
  bool operator==(const LayerSpec&) const = default;
};

struct ModelSpec {
  std::string name = "model";
  std::vector<LayerSpec> layers;
  uint32_t iterations = 1;
  uint32_t warmup_iterations = 0;
  int64_t update_us = 0;
  bool operator==(const ModelSpec&) const = default;
};

struct Bucket {
  uint32_t first_layer = 0;
  uint32_t last_layer = 0;
  uint64_t bytes = 0;
};

ModelSpec parse_model_spec(const std::string& text);
std::string render_model_spec(const ModelSpec& m);
bool builtin_model(const std::string& name, ModelSpec* out);
std::vector<Bucket> bucketize(const ModelSpec& m, uint64_t bucket_bytes);

// One iteration's device timeline, microseconds from the loop's first event.
struct IterTrace {
  double start_us = 0, end_us = 0;
  std::vector<double> issue_us, complete_us;  // per bucket (issue order)
};

// Runs model.iterations iterations on `comm`; returns one trace per
// iteration (warm-up included).  Throws std::runtime_error on failure.
std::vector<IterTrace> run_training_loop(cemuComm_t comm, const ModelSpec& m,
                                         uint64_t bucket_bytes);

// The ideal timeline of the same loop: compute exactly as specified, each
// bucket's collective taking exactly its modelled latency (A14) in issue
// order.  Returns the iteration time in us.
double predicted_iteration_us(const ModelSpec& m, uint64_t bucket_bytes,
                              const std::vector<double>& bucket_latency_us);

// Device word holding the end (%globaltimer ns) of the last delayed call
// `comm` enqueued on `stream`, or null (delay off, or another stream).
const int64_t* stream_release_end(cemuComm_t comm, cudaStream_t stream);
// Sets the communicator's queue-chaining gap and returns the previous one.
int64_t exchange_queue_gap_ns(cemuComm_t comm, int64_t gap_ns);

}  // namespace cemu_b200
