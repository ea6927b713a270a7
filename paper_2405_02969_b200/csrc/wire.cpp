// wire.cpp -- CEMU wire-protocol client (see wire.hpp for the format and the
// reference behaviour each piece follows).
#include "wire.hpp"

#include <arpa/inet.h>
#include <netdb.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <sys/time.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cstring>
#include <ctime>
#include <map>

#include "schedule.hpp"

namespace cemu_b200 {
namespace {

constexpr uint8_t kHello = 1, kTopo = 2, kOpenOp = 3, kData = 4, kError = 5, kBye = 6;
constexpr int kAwaitTimeoutMs = 30000;  // collective.cpp:15

const char* type_name(uint8_t t) {
  static const char* names[] = {"UNKNOWN", "HELLO", "TOPO", "OPEN_OP", "DATA", "ERROR", "BYE"};
  return t >= 1 && t <= 6 ? names[t] : names[0];
}

int64_t realtime_ns() {
  timespec ts{};
  clock_gettime(CLOCK_REALTIME, &ts);
  return static_cast<int64_t>(ts.tv_sec) * 1000000000LL + ts.tv_nsec;
}

void put16(uint8_t* p, uint16_t v) {
  p[0] = static_cast<uint8_t>(v);
  p[1] = static_cast<uint8_t>(v >> 8);
}
void put32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}
uint16_t get16(const uint8_t* p) { return static_cast<uint16_t>(p[0] | (p[1] << 8)); }
uint32_t get32(const uint8_t* p) {
  return static_cast<uint32_t>(p[0]) | static_cast<uint32_t>(p[1]) << 8 | static_cast<uint32_t>(p[2]) << 16 |
         static_cast<uint32_t>(p[3]) << 24;
}

void write_all(int fd, const uint8_t* p, size_t n) {
  while (n) {
    const ssize_t k = ::send(fd, p, n, MSG_NOSIGNAL);
    if (k < 0) {
      if (errno == EINTR) continue;
      throw WireError(std::string("send: ") + std::strerror(errno));
    }
    p += k;
    n -= static_cast<size_t>(k);
  }
}

// false on clean EOF before the first byte
bool read_exact(int fd, uint8_t* p, size_t n) {
  size_t got = 0;
  while (got < n) {
    const ssize_t k = ::recv(fd, p + got, n - got, 0);
    if (k == 0) {
      if (got == 0) return false;
      throw WireError("connection closed mid-frame");
    }
    if (k < 0) {
      if (errno == EINTR) continue;
      if (errno == EAGAIN || errno == EWOULDBLOCK) throw WireError("timed out");
      throw WireError(std::string("recv: ") + std::strerror(errno));
    }
    got += static_cast<size_t>(k);
  }
  return true;
}

bool read_frame(int fd, WireFrame* f) {
  uint8_t h[24];
  if (!read_exact(fd, h, sizeof h)) return false;
  if (std::memcmp(h, "CEMU", 4) != 0) throw WireError("bad magic");
  if (h[4] != 1) throw WireError("unsupported wire version " + std::to_string(h[4]));
  f->type = h[5];
  if (f->type < kHello || f->type > kBye) throw WireError("unknown frame type " + std::to_string(h[5]));
  f->op_id = get32(h + 6);
  f->seq = get32(h + 10);
  f->src = get16(h + 14);
  f->dst = get16(h + 16);
  f->chunk = get16(h + 18);
  const uint32_t len = get32(h + 20);
  if (len > kWireMaxPayload) {
    throw WireError("payload_len " + std::to_string(len) + " exceeds cap " + std::to_string(kWireMaxPayload));
  }
  f->payload.resize(len);
  if (len && !read_exact(fd, f->payload.data(), len)) throw WireError("connection closed mid-frame");
  f->arrival_ns = realtime_ns();
  return true;
}

void set_recv_timeout(int fd, int ms) {
  timeval tv{};
  tv.tv_sec = ms / 1000;
  tv.tv_usec = (ms % 1000) * 1000;
  ::setsockopt(fd, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof tv);
}

int dial(const Endpoint& ep, int timeout_ms) {
  sockaddr_in addr{};
  addr.sin_family = AF_INET;
  addr.sin_port = htons(ep.port);
  if (::inet_pton(AF_INET, ep.host.c_str(), &addr.sin_addr) != 1) {
    addrinfo hints{}, *res = nullptr;
    hints.ai_family = AF_INET;
    if (::getaddrinfo(ep.host.c_str(), nullptr, &hints, &res) != 0 || !res) {
      throw WireError("cannot resolve " + ep.host);
    }
    addr.sin_addr = reinterpret_cast<sockaddr_in*>(res->ai_addr)->sin_addr;
    ::freeaddrinfo(res);
  }
  // retry until the listener is up (net.cpp:198-216 does the same)
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  int err = 0;
  do {
    const int fd = ::socket(AF_INET, SOCK_STREAM, 0);
    if (fd < 0) throw WireError(std::string("socket: ") + std::strerror(errno));
    if (::connect(fd, reinterpret_cast<sockaddr*>(&addr), sizeof addr) == 0) {
      int one = 1;
      ::setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
      return fd;
    }
    err = errno;
    ::close(fd);
    std::this_thread::sleep_for(std::chrono::milliseconds(20));
  } while (std::chrono::steady_clock::now() < deadline);
  throw WireError("connect " + ep.str() + ": " + std::strerror(err));
}

// ---- a small JSON reader: enough for the HELLO/TOPO payloads ----------------
struct Json {
  enum Kind { kNull, kBool, kNum, kStr, kArr, kObj } kind = kNull;
  bool neg = false;
  uint64_t mag = 0;  // integer magnitude (the handshake holds integers only)
  bool integral = true;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;
  int64_t as_i64() const { return neg ? -static_cast<int64_t>(mag) : static_cast<int64_t>(mag); }
  const Json& at(const std::string& k) const {
    auto it = obj.find(k);
    if (kind != kObj || it == obj.end()) throw WireError("malformed handshake payload: missing '" + k + "'");
    return it->second;
  }
};

struct JsonParser {
  const std::string& s;
  size_t i = 0;
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r')) ++i;
  }
  [[noreturn]] void bad() { throw WireError("malformed handshake payload at byte " + std::to_string(i)); }
  char peek() {
    ws();
    if (i >= s.size()) bad();
    return s[i];
  }
  void expect(char c) {
    if (peek() != c) bad();
    ++i;
  }
  std::string string() {
    expect('"');
    std::string out;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\') {
        if (++i >= s.size()) bad();
        const char e = s[i];
        out.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e);  // the handshake carries plain ASCII
      } else {
        out.push_back(s[i]);
      }
      ++i;
    }
    if (i >= s.size()) bad();
    ++i;
    return out;
  }
  Json value() {
    Json v;
    const char c = peek();
    if (c == '{') {
      v.kind = Json::kObj;
      ++i;
      if (peek() == '}') {
        ++i;
        return v;
      }
      while (true) {
        std::string k = string();
        expect(':');
        v.obj[k] = value();
        if (peek() == ',') {
          ++i;
          continue;
        }
        expect('}');
        return v;
      }
    }
    if (c == '[') {
      v.kind = Json::kArr;
      ++i;
      if (peek() == ']') {
        ++i;
        return v;
      }
      while (true) {
        v.arr.push_back(value());
        if (peek() == ',') {
          ++i;
          continue;
        }
        expect(']');
        return v;
      }
    }
    if (c == '"') {
      v.kind = Json::kStr;
      v.str = string();
      return v;
    }
    if (s.compare(i, 4, "true") == 0 || s.compare(i, 5, "false") == 0 || s.compare(i, 4, "null") == 0) {
      v.kind = s[i] == 'n' ? Json::kNull : Json::kBool;
      i += s[i] == 'f' ? 5 : 4;
      return v;
    }
    v.kind = Json::kNum;
    if (s[i] == '-') {
      v.neg = true;
      ++i;
    }
    if (i >= s.size() || s[i] < '0' || s[i] > '9') bad();
    while (i < s.size() && s[i] >= '0' && s[i] <= '9') v.mag = v.mag * 10 + static_cast<uint64_t>(s[i++] - '0');
    while (i < s.size() && (s[i] == '.' || s[i] == 'e' || s[i] == 'E' || s[i] == '+' || s[i] == '-' ||
                            (s[i] >= '0' && s[i] <= '9'))) {
      v.integral = false;
      ++i;
    }
    return v;
  }
};

}  // namespace

std::vector<uint8_t> wire_encode_header(const WireFrame& f, uint32_t len) {
  if (len > kWireMaxPayload) {
    throw WireError("payload_len " + std::to_string(len) + " exceeds cap " + std::to_string(kWireMaxPayload));
  }
  std::vector<uint8_t> h(24);
  std::memcpy(h.data(), "CEMU", 4);
  h[4] = 1;
  h[5] = f.type;
  put32(&h[6], f.op_id);
  put32(&h[10], f.seq);
  put16(&h[14], f.src);
  put16(&h[16], f.dst);
  put16(&h[18], f.chunk);
  put32(&h[20], len);
  return h;
}

std::string wire_encode_hello(int32_t rank, uint32_t world, uint64_t digest, const std::vector<WirePlanEntry>& plan) {
  std::string s = "{\"config_digest\":" + std::to_string(digest) + ",\"plan\":[";
  for (size_t k = 0; k < plan.size(); ++k) {
    if (k) s += ",";
    s += "{\"bytes\":" + std::to_string(plan[k].bytes) + ",\"elem_size\":" + std::to_string(plan[k].elem_size) +
         ",\"op\":\"" + (plan[k].coll == 0 ? "allreduce" : "allgather") + "\"}";
  }
  s += "],\"rank\":" + std::to_string(rank) + ",\"world_size\":" + std::to_string(world) + "}";
  return s;
}

WireHello wire_decode_hello(const std::string& text) {
  JsonParser p{text};
  const Json j = p.value();
  WireHello h;
  h.rank = j.at("rank").as_i64();
  h.world = j.at("world_size").mag;
  h.digest = j.at("config_digest").mag;
  const Json& plan = j.at("plan");
  if (plan.kind != Json::kArr) throw WireError("malformed handshake payload: plan is not an array");
  for (const Json& e : plan.arr) {
    WirePlanEntry pe;
    const std::string& op = e.at("op").str;
    if (op != "allreduce" && op != "allgather") throw WireError("unknown collective kind '" + op + "'");
    pe.coll = op == "allreduce" ? 0 : 1;
    pe.bytes = e.at("bytes").mag;
    pe.elem_size = static_cast<uint32_t>(e.at("elem_size").mag);
    h.plan.push_back(pe);
  }
  return h;
}

WireSession::WireSession(const JobConfig& cfg, uint32_t rank, std::vector<WirePlanEntry> plan, int timeout_ms)
    : cfg_(cfg), rank_(rank), plan_(std::move(plan)) {
  const uint32_t n = cfg_.world_size;
  if (cfg_.endpoints.size() != n) throw WireError("endpoint: the wire mode needs endpoint.R for every rank");
  if (rank_ >= n) throw WireError("rank " + std::to_string(rank_) + " out of range");
  const uint32_t succ = (rank_ + 1) % n;
  if (cfg_.is_real(succ)) throw WireError("wire mode: the successor of rank " + std::to_string(rank_) +
                                          " must be emulated (one real rank per ring segment)");
  fd_ = dial(cfg_.endpoints[succ], timeout_ms);
  try {
    set_recv_timeout(fd_, timeout_ms);
    const std::string hello = wire_encode_hello(static_cast<int32_t>(rank_), n, config_digest(cfg_), plan_);
    WireFrame f;
    f.type = kHello;
    write_frame(f, reinterpret_cast<const uint8_t*>(hello.data()), static_cast<uint32_t>(hello.size()));
    WireFrame t;
    if (!read_frame(fd_, &t)) throw WireError("handshake: connection closed");
    if (t.type == kError) {
      throw WireError("handshake rejected by peer: " + std::string(t.payload.begin(), t.payload.end()));
    }
    if (t.type != kTopo) {
      throw WireError(std::string("handshake: expected TOPO, got ") + type_name(t.type));
    }
    const WireHello peer = wire_decode_hello(std::string(t.payload.begin(), t.payload.end()));
    if (peer.digest != config_digest(cfg_) || peer.world != n) {
      throw WireError("handshake: config digest mismatch");
    }
    set_recv_timeout(fd_, 0);
  } catch (...) {
    ::close(fd_);
    fd_ = -1;
    throw;
  }
  reader_ = std::thread([this] { reader_main(); });
}

WireSession::~WireSession() {
  bool ok;
  {
    std::lock_guard<std::mutex> lk(mu_);
    closing_ = true;
    ok = !failed_;
  }
  if (fd_ >= 0) {
    if (ok) {
      try {
        WireFrame bye;
        bye.type = kBye;
        bye.src = static_cast<uint16_t>(rank_);
        write_frame(bye, nullptr, 0);
      } catch (const std::exception&) {
      }
    }
    // the BYE sits ahead of the FIN; the emulator answers BYE and closes,
    // which ends the reader -- unless it is gone: then, after a grace
    // period, shutting the read side down wakes the blocked recv
    ::shutdown(fd_, SHUT_WR);
    std::unique_lock<std::mutex> lk(mu_);
    if (!cv_.wait_for(lk, std::chrono::seconds(2), [this] { return reader_done_; })) {
      ::shutdown(fd_, SHUT_RDWR);
    }
  }
  if (reader_.joinable()) reader_.join();
  if (fd_ >= 0) ::close(fd_);
}

void WireSession::write_frame(const WireFrame& f, const uint8_t* payload, uint32_t len) {
  const std::vector<uint8_t> h = wire_encode_header(f, len);
  write_all(fd_, h.data(), h.size());
  if (len) write_all(fd_, payload, len);
}

void WireSession::fail(const std::string& why) {
  std::lock_guard<std::mutex> lk(mu_);
  if (!failed_) {
    failed_ = true;
    fail_reason_ = why;
  }
  cv_.notify_all();
}

void WireSession::reader_main() {
  struct Done {  // tells the destructor the reader has left, however it leaves
    WireSession* w;
    ~Done() {
      std::lock_guard<std::mutex> lk(w->mu_);
      w->reader_done_ = true;
      w->cv_.notify_all();
    }
  } done{this};
  try {
    while (true) {
      WireFrame f;
      if (!read_frame(fd_, &f)) {
        std::lock_guard<std::mutex> lk(mu_);
        eof_ = true;
        if (!closing_ && !failed_) {
          failed_ = true;
          fail_reason_ = "peer closed connection unexpectedly";
        }
        cv_.notify_all();
        return;
      }
      if (f.type == kData || f.type == kOpenOp) {
        std::lock_guard<std::mutex> lk(mu_);
        inbox_.push_back(std::move(f));
        cv_.notify_all();
      } else if (f.type == kBye) {
        return;
      } else if (f.type == kError) {
        fail("peer reported error: " + std::string(f.payload.begin(), f.payload.end()));
        return;
      } else {
        fail(std::string("unexpected frame type ") + type_name(f.type));
        return;
      }
    }
  } catch (const std::exception& e) {
    bool closing;
    {
      std::lock_guard<std::mutex> lk(mu_);
      closing = closing_;
    }
    if (!closing) fail(std::string("transport failure: ") + e.what());
  }
}

WireFrame WireSession::await(uint32_t op_id) {
  std::unique_lock<std::mutex> lk(mu_);
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(kAwaitTimeoutMs);
  while (true) {
    for (auto it = inbox_.begin(); it != inbox_.end(); ++it) {
      if (it->op_id == op_id) {
        WireFrame f = std::move(*it);
        inbox_.erase(it);
        return f;
      }
    }
    if (failed_) throw WireError(fail_reason_);
    if (cv_.wait_until(lk, deadline) == std::cv_status::timeout) {
      failed_ = true;
      fail_reason_ = "timed out waiting for collective traffic";
      throw WireError(fail_reason_);
    }
  }
}

void WireSession::run(int coll, uint64_t buffer_bytes, uint32_t elem_size,
                      const std::function<void(uint64_t, uint64_t, uint8_t*)>& load,
                      const std::function<void(uint64_t, const uint8_t*, uint64_t, bool)>& store,
                      int64_t* t_open_ns, std::vector<int64_t>* arrival_ns) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    if (failed_) throw WireError(fail_reason_);
  }
  // WorkerSession::submit's checks (collective.cpp:181-211)
  if (plan_.empty()) throw WireError("no collectives were declared for this session");
  const uint32_t op_id = next_op_;
  const uint32_t pi = op_id % static_cast<uint32_t>(plan_.size());
  const WirePlanEntry& e = plan_[pi];
  if (e.coll != coll || e.elem_size != elem_size) {
    throw WireError("collective call does not match the declared plan");
  }
  const uint32_t n = cfg_.world_size;
  const uint64_t want = coll == 0 ? e.bytes : e.bytes * n;
  if (buffer_bytes != want) {
    throw WireError("buffer size " + std::to_string(buffer_bytes) + " does not match plan entry (" +
                    std::to_string(want) + ")");
  }
  ++next_op_;
  const uint32_t succ = (rank_ + 1) % n, pred = (rank_ + n - 1) % n;
  auto span_of = [&](uint32_t c, uint64_t* off, uint64_t* len) {
    if (coll == 0) {
      *off = chunk_offset_bytes(n, e.bytes, e.elem_size, c);
      *len = chunk_bytes(n, e.bytes, e.elem_size, c);
    } else {
      *off = static_cast<uint64_t>(c) * e.bytes;
      *len = e.bytes;
    }
  };
  WireFrame open;
  open.type = kOpenOp;
  open.op_id = op_id;
  open.seq = pi;
  open.src = static_cast<uint16_t>(rank_);
  open.dst = static_cast<uint16_t>(succ);
  *t_open_ns = realtime_ns();
  write_frame(open, nullptr, 0);
  const uint32_t P = positions(coll, n);
  arrival_ns->assign(P, 0);
  for (uint32_t p = 0; p < P; ++p) {
    const uint32_t sc = send_chunk_at(coll, n, rank_, p);
    uint64_t off = 0, len = 0;
    span_of(sc, &off, &len);
    if (len > kWireMaxPayload) {
      throw WireError("payload_len " + std::to_string(len) + " exceeds cap " + std::to_string(kWireMaxPayload));
    }
    out_.resize(len);
    load(off, len, out_.data());
    WireFrame d;
    d.type = kData;
    d.op_id = op_id;
    d.seq = p;
    d.src = static_cast<uint16_t>(rank_);
    d.dst = static_cast<uint16_t>(succ);
    d.chunk = static_cast<uint16_t>(sc);
    write_frame(d, out_.data(), static_cast<uint32_t>(len));

    const uint32_t rc = send_chunk_at(coll, n, pred, p);
    uint64_t roff = 0, rlen = 0;
    span_of(rc, &roff, &rlen);
    WireFrame r;
    while (true) {
      r = await(op_id);
      if (r.type == kOpenOp) {
        if (r.seq != pi) {
          const std::string why = "peer opened op " + std::to_string(op_id) + " with plan index " +
                                  std::to_string(r.seq) + ", expected " + std::to_string(pi);
          fail(why);
          throw WireError(why);
        }
        continue;  // the emulator's mirror of the announcement
      }
      break;
    }
    if (r.seq != p || r.src != pred || r.dst != rank_ || r.chunk != rc || r.payload.size() != rlen) {
      const std::string why =
          "protocol mismatch: expected {op=" + std::to_string(op_id) + " step=" + std::to_string(p) +
          " src=" + std::to_string(pred) + " dst=" + std::to_string(rank_) + " chunk=" + std::to_string(rc) +
          " size=" + std::to_string(rlen) + "}, got {op=" + std::to_string(r.op_id) + " step=" +
          std::to_string(r.seq) + " src=" + std::to_string(r.src) + " dst=" + std::to_string(r.dst) +
          " chunk=" + std::to_string(r.chunk) + " size=" + std::to_string(r.payload.size()) + "}";
      fail(why);
      throw WireError(why);
    }
    (*arrival_ns)[p] = r.arrival_ns;
    store(roff, r.payload.data(), rlen, coll == 0 && p + 2 <= n);
  }
}

}  // namespace cemu_b200
