// wire.hpp -- the CEMU wire protocol, spoken by a B200 communicator to a
// reference `cemu-emulator` (wire-format interop).
//
// The device path has no wire; this is the optional cross-check mode in
// which a real rank's collectives travel as the reference WorkerSession's
// would, so the reference engine (proj/src/emulator.cpp) schedules and
// releases the emulated peers' frames, and this side records when each
// arrived against the device delay model's floors.
//
// Protocol (re-stated from the reference's behaviour, not its code):
//   frame   24-byte little-endian header (frame.hpp:24-45, frame.cpp:40-58)
//             "CEMU" | version 1 | type u8 | op_id u32 | seq u32 |
//             src u16 | dst u16 | chunk u16 | payload_len u32
//           then payload_len bytes (cap 64 MiB, frame.hpp:43)
//   types   HELLO 1, TOPO 2, OPEN_OP 3, DATA 4, ERROR 5, BYE 6
//   session the real rank dials endpoint[successor]; HELLO carries JSON
//           {rank, world_size, config_digest, plan[{op, bytes, elem_size}]}
//           (transport.cpp:9-41); the emulator answers TOPO with its own
//           identity (rank -1) after checking the digest (transport.cpp:
//           105-159).  One connection carries every emulated peer; the
//           emulator's DATA comes back on it (emulator.cpp:110-140).
//   op      OPEN_OP {op_id, seq = plan index, src = rank, dst = successor},
//           then per ring position p: DATA out (own scheduled chunk), DATA
//           in (the predecessor's), checked field by field and folded --
//           int32 lanes when elem_size is 4, bytes otherwise -- in the
//           reduce phase, copied in the gather phase (collective.cpp:268-355).
//           The emulator mirrors OPEN_OP; BYE closes (collective.cpp:406-442).
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "config.hpp"

namespace cemu_b200 {

class WireError : public std::runtime_error {
 public:
  explicit WireError(const std::string& what) : std::runtime_error(what) {}
};

struct WirePlanEntry {
  int coll = 0;  // 0 allreduce, 1 allgather (the reference protocol's two kinds)
  uint64_t bytes = 0;  // allgather: per-rank block
  uint32_t elem_size = 1;
  bool operator==(const WirePlanEntry&) const = default;
};

struct WireFrame {
  uint8_t type = 4;
  uint32_t op_id = 0, seq = 0;
  uint16_t src = 0, dst = 0, chunk = 0;
  std::vector<uint8_t> payload;
  int64_t arrival_ns = 0;  // CLOCK_REALTIME when the reader finished it
};

constexpr uint32_t kWireMaxPayload = 64u << 20;

std::vector<uint8_t> wire_encode_header(const WireFrame& f, uint32_t payload_len);
std::string wire_encode_hello(int32_t rank, uint32_t world, uint64_t digest,
                              const std::vector<WirePlanEntry>& plan);

struct WireHello {
  int64_t rank = -1;
  uint64_t world = 0, digest = 0;
  std::vector<WirePlanEntry> plan;
};
WireHello wire_decode_hello(const std::string& json);

class WireSession {
 public:
  // Dials endpoint[successor(rank)] and performs the HELLO/TOPO handshake.
  WireSession(const JobConfig& cfg, uint32_t rank, std::vector<WirePlanEntry> plan, int timeout_ms = 10000);
  ~WireSession();  // BYE, shutdown, join the reader

  // One collective on the caller's buffer, through callbacks (the buffer
  // lives on the GPU):
  //   load(offset, len, host_dst)          local bytes -> outgoing DATA
  //   store(offset, host_src, len, reduce) incoming DATA -> local buffer
  // `buffer_bytes` as WorkerSession::submit checks it (plan bytes, or
  // world * plan bytes for allgather).  Fills t_open_ns and the arrival
  // time of each received DATA (one per ring position).
  void run(int coll, uint64_t buffer_bytes, uint32_t elem_size,
           const std::function<void(uint64_t, uint64_t, uint8_t*)>& load,
           const std::function<void(uint64_t, const uint8_t*, uint64_t, bool)>& store,
           int64_t* t_open_ns, std::vector<int64_t>* arrival_ns);

  uint32_t ops() const { return next_op_; }

 private:
  void reader_main();
  WireFrame await(uint32_t op_id);
  void write_frame(const WireFrame& f, const uint8_t* payload, uint32_t len);
  void fail(const std::string& why);

  JobConfig cfg_;
  uint32_t rank_ = 0;
  std::vector<WirePlanEntry> plan_;
  int fd_ = -1;
  uint32_t next_op_ = 0;
  std::thread reader_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<WireFrame> inbox_;
  bool failed_ = false, closing_ = false, eof_ = false, reader_done_ = false;
  std::string fail_reason_;
  std::vector<uint8_t> out_;  // staging for outgoing DATA payloads
};

}  // namespace cemu_b200
