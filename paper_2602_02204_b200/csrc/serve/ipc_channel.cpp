// Cross-process DEVICE transport: control frames over a connected AF_UNIX
// stream socket (see omni/ipc_channel.hpp).
#include "omni/ipc_channel.hpp"

#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cstring>
#include <thread>

namespace omni {

namespace {

[[noreturn]] void sys_fail(const std::string& what) {
  throw TransportDown(what + ": " + std::strerror(errno));
}

sockaddr_un unix_addr(const std::string& path) {
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  if (path.size() >= sizeof(a.sun_path)) throw ConfigInvalid("unix socket path too long: " + path);
  std::memcpy(a.sun_path, path.c_str(), path.size() + 1);
  return a;
}

int ms_left(std::chrono::steady_clock::time_point deadline) {
  const auto d = std::chrono::duration_cast<std::chrono::milliseconds>(deadline - std::chrono::steady_clock::now());
  return d.count() > 0 ? static_cast<int>(d.count()) : 0;
}

}  // namespace

IpcChannel& IpcChannel::operator=(IpcChannel&& o) noexcept {
  if (this != &o) {
    if (fd_ >= 0) ::close(fd_);
    fd_ = std::exchange(o.fd_, -1);
    rx_ = std::move(o.rx_);
    sent_ = o.sent_;
  }
  return *this;
}

IpcChannel::~IpcChannel() {
  if (fd_ >= 0) ::close(fd_);
}

std::pair<IpcChannel, IpcChannel> IpcChannel::pair() {
  int sv[2];
  if (::socketpair(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0, sv) != 0) sys_fail("socketpair");
  return {IpcChannel(sv[0]), IpcChannel(sv[1])};
}

IpcChannel IpcChannel::listen_accept(const std::string& path, uint64_t timeout_ms) {
  const int s = ::socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
  if (s < 0) sys_fail("socket");
  ::unlink(path.c_str());
  sockaddr_un a = unix_addr(path);
  if (::bind(s, reinterpret_cast<sockaddr*>(&a), sizeof(a)) != 0) {
    ::close(s);
    if (errno == EADDRINUSE) throw PortInUse("unix socket in use: " + path);
    sys_fail("bind " + path);
  }
  if (::listen(s, 1) != 0) {
    ::close(s);
    sys_fail("listen");
  }
  pollfd p{s, POLLIN, 0};
  const int r = ::poll(&p, 1, static_cast<int>(timeout_ms));
  if (r <= 0) {
    ::close(s);
    ::unlink(path.c_str());
    throw TimeoutError("no connection on " + path);
  }
  const int c = ::accept4(s, nullptr, nullptr, SOCK_CLOEXEC);
  ::close(s);
  ::unlink(path.c_str());
  if (c < 0) sys_fail("accept");
  return IpcChannel(c);
}

IpcChannel IpcChannel::connect(const std::string& path, uint64_t timeout_ms) {
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  sockaddr_un a = unix_addr(path);
  for (;;) {
    const int s = ::socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (s < 0) sys_fail("socket");
    if (::connect(s, reinterpret_cast<sockaddr*>(&a), sizeof(a)) == 0) return IpcChannel(s);
    ::close(s);
    if (std::chrono::steady_clock::now() >= deadline) throw TimeoutError("cannot connect to " + path);
    std::this_thread::sleep_for(std::chrono::milliseconds(2));
  }
}

void IpcChannel::send(const ControlMessage& m) {
  if (fd_ < 0) throw TransportDown("ipc channel closed");
  const std::vector<uint8_t> f = encode_control_frame(m);
  size_t at = 0;
  while (at < f.size()) {
    const ssize_t n = ::send(fd_, f.data() + at, f.size() - at, MSG_NOSIGNAL);
    if (n < 0) {
      if (errno == EINTR) continue;
      sys_fail("ipc send");
    }
    at += static_cast<size_t>(n);
  }
  ++sent_;
}

bool IpcChannel::fill(int timeout_ms) {
  if (fd_ < 0) throw TransportDown("ipc channel closed");
  pollfd p{fd_, POLLIN, 0};
  const int r = ::poll(&p, 1, timeout_ms);
  if (r < 0) {
    if (errno == EINTR) return false;
    sys_fail("ipc poll");
  }
  if (r == 0) return false;
  uint8_t buf[1 << 16];
  const ssize_t n = ::recv(fd_, buf, sizeof(buf), MSG_DONTWAIT);
  if (n < 0) {
    if (errno == EAGAIN || errno == EWOULDBLOCK || errno == EINTR) return false;
    sys_fail("ipc recv");
  }
  if (n == 0) throw TransportDown("ipc peer closed the channel");
  rx_.insert(rx_.end(), buf, buf + n);
  return true;
}

std::optional<std::vector<uint8_t>> IpcChannel::take_frame() {
  if (rx_.size() < 5) return std::nullopt;
  const uint32_t len = uint32_t(rx_[0]) | uint32_t(rx_[1]) << 8 | uint32_t(rx_[2]) << 16 | uint32_t(rx_[3]) << 24;
  if (rx_.size() < 5ull + len) return std::nullopt;
  std::vector<uint8_t> f(rx_.begin(), rx_.begin() + 5 + len);
  rx_.erase(rx_.begin(), rx_.begin() + 5 + len);
  return f;
}

std::optional<ControlMessage> IpcChannel::try_recv() {
  if (auto f = take_frame()) return decode_control_frame(*f);
  while (fill(0))
    if (auto f = take_frame()) return decode_control_frame(*f);
  return std::nullopt;
}

ControlMessage IpcChannel::recv(uint64_t timeout_ms) {
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  for (;;) {
    if (auto f = take_frame()) return decode_control_frame(*f);
    const int left = ms_left(deadline);
    if (!fill(left) && left == 0) throw TimeoutError("ipc recv timed out");
  }
}

ControlMessage handoff_frame(const std::string& key, const void* bytes, size_t n) {
  ControlMessage m;
  m.kind = ControlMessage::Kind::HANDOFF;
  m.key = key;
  m.locator.kind = Locator::Kind::INLINE;
  const auto* b = static_cast<const uint8_t*>(bytes);
  m.locator.inline_bytes.assign(b, b + n);
  return m;
}

std::vector<uint8_t> handoff_bytes(const ControlMessage& m, const std::string& key) {
  if (m.kind != ControlMessage::Kind::HANDOFF || m.key != key || m.locator.kind != Locator::Kind::INLINE)
    throw ProtocolViolation("expected HANDOFF " + key);
  return m.locator.inline_bytes;
}

// ---- producer -------------------------------------------------------------

void IpcStreamSender::send(const StreamChunk& c) {
  if (!c.payload.is_device()) throw BadDtype("ipc device stream carries device payloads only");
  const uint64_t a = c.payload.dev.blob, n = c.payload.dev.nbytes;
  if (a < base_ || a + n > base_ + bytes_) throw ProtocolViolation("payload blob outside the exported arena");
  St& s = st_[c.request_id];
  if (s.eos) throw ProtocolViolation("chunk after eos");
  if (c.seq != s.next)
    throw ProtocolViolation("out-of-order chunk seq " + std::to_string(c.seq) + " (expected " +
                            std::to_string(s.next) + ")");
  ControlMessage m;
  m.kind = c.eos ? ControlMessage::Kind::EOS : ControlMessage::Kind::CHUNK_NOTICE;
  m.request_id = c.request_id;
  m.edge = edge_;
  m.seq = c.seq;
  m.locator = device_locator(c.payload);
  m.locator.arena = arena_;
  m.locator.offset = a - base_;
  ch_->send(m);
  ++s.next;
  s.eos = c.eos;
}

void IpcStreamSender::poll_acks() {
  while (auto m = ch_->try_recv()) {
    if (m->kind != ControlMessage::Kind::ACK || m->edge != edge_)
      throw ProtocolViolation("unexpected frame on the producer side of " + edge_);
    St& s = st_[m->request_id];
    if (m->seq >= s.next) throw ProtocolViolation("ack of a chunk never sent");
    s.acked = std::max<uint64_t>(s.acked, uint64_t(m->seq) + 1);
  }
}

uint64_t IpcStreamSender::acked(uint64_t rid) const {
  auto it = st_.find(rid);
  return it == st_.end() ? 0 : it->second.acked;
}

// ---- consumer -------------------------------------------------------------

void IpcStreamReceiver::accept(const ControlMessage& m) {
  const bool chunk = m.kind == ControlMessage::Kind::CHUNK_NOTICE || m.kind == ControlMessage::Kind::EOS;
  if (!chunk || m.edge != edge_) {
    other_.push_back(m);
    return;
  }
  const Locator& l = m.locator;
  if (l.kind != Locator::Kind::DEVICE) throw ProtocolViolation("ipc chunk without a device locator");
  if (l.arena != arena_) throw ProtocolViolation("chunk names an unknown arena");
  if (l.offset % 16 != 0 || l.offset > bytes_ || l.length > bytes_ - l.offset)
    throw ProtocolViolation("device locator outside the arena");
  St& s = st_[m.request_id];
  if (s.eos) throw ProtocolViolation("chunk after eos");
  if (m.seq != s.next)
    throw ProtocolViolation("out-of-order chunk seq " + std::to_string(m.seq) + " (expected " +
                            std::to_string(s.next) + ")");
  StreamChunk c;
  c.request_id = m.request_id;
  const auto arrow = edge_.find("->");
  if (arrow != std::string::npos) {
    c.from = edge_.substr(0, arrow);
    c.to = edge_.substr(arrow + 2);
  }
  c.seq = m.seq;
  c.eos = m.kind == ControlMessage::Kind::EOS;
  c.payload = payload_from_locator(l);
  c.payload.dev.device = dev_;
  c.payload.dev.arena = 0;  // re-based: a local address from here on
  c.payload.dev.blob = base_ + l.offset;
  s.q.push_back(std::move(c));
  ++s.next;
  s.eos = m.kind == ControlMessage::Kind::EOS;
}

std::optional<StreamChunk> IpcStreamReceiver::try_recv(uint64_t rid) {
  while (auto m = ch_->try_recv()) accept(*m);
  auto it = st_.find(rid);
  if (it == st_.end() || it->second.q.empty()) return std::nullopt;
  StreamChunk c = std::move(it->second.q.front());
  it->second.q.pop_front();
  return c;
}

StreamChunk IpcStreamReceiver::recv(uint64_t rid, uint64_t timeout_ms) {
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  for (;;) {
    if (auto c = try_recv(rid)) return std::move(*c);
    accept(ch_->recv(static_cast<uint64_t>(std::max(1, ms_left(deadline)))));
    auto it = st_.find(rid);
    if (it != st_.end() && !it->second.q.empty()) continue;
    if (ms_left(deadline) == 0) throw TimeoutError("ipc stream recv timed out");
  }
}

void IpcStreamReceiver::ack(uint64_t rid, uint32_t seq) {
  ControlMessage m;
  m.kind = ControlMessage::Kind::ACK;
  m.key = ConnectorKey{rid, edge_, "chunk", seq}.canonical();
  m.request_id = rid;
  m.edge = edge_;
  m.seq = seq;
  ch_->send(m);
}

}  // namespace omni
