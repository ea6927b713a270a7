// schedule.hpp -- host-side ring schedule arithmetic of one emulated call.
//
// The reference materialises a send/recv DAG per call (proj/src/dag.cpp:
// 90-137, n*2(n-1)*2 vertices) and projects it onto the real/emulated
// boundary with an O(n^3) reachability + transitive reduction (232-338).
// Here every quantity the hot path needs is a closed form, O(1) per step:
// chunk sizes/offsets (dag.cpp:32-46), the chunk each rank sends at each
// position (73-82), the boundary's vertex/edge structure for a single real
// rank, and K = the number of to-real messages for any real set.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "cemu_b200.h"

namespace cemu_b200 {

uint64_t chunk_bytes(uint32_t n, uint64_t total, uint32_t elem, uint32_t c);
uint64_t chunk_offset_bytes(uint32_t n, uint64_t total, uint32_t elem, uint32_t c);
uint32_t positions(int coll, uint32_t n);
uint32_t send_chunk_at(int coll, uint32_t n, uint32_t rank, uint32_t p);
std::string boundary_dump(int coll, uint32_t n, uint64_t bytes, uint32_t elem, uint32_t real);
uint32_t to_real_count(int coll, uint32_t n, const std::vector<uint32_t>& real);

// Delay model, host evaluation (delay_math.cuh is shared with the device).
double model_total(const cemuDelayModel& m, int coll, uint32_t n, uint64_t bytes);
std::vector<double> release_offsets(const cemuDelayModel& m, int coll, uint32_t n,
                                    uint64_t bytes, uint32_t k);
std::vector<int64_t> release_floors(const cemuDelayModel& m, int coll, uint32_t n,
                                    uint64_t bytes, uint32_t k, int64_t now_us);
int64_t call_latency_us(const cemuDelayModel& m, int coll, uint32_t n, uint64_t bytes,
                        uint32_t k);

}  // namespace cemu_b200
