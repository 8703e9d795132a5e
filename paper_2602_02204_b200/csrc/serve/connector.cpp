// Connector streams: same ordering / exactly-once / protocol-violation
// contract as the reference (connector.hpp:95-321).
#include "omni/connector.hpp"

#include <chrono>

#include "omni/control.hpp"

namespace omni {

std::string ConnectorKey::canonical() const {
  return "req:" + std::to_string(request_id) + "/edge:" + edge + "/" + name + "/" + std::to_string(index);
}

Connector::Connector(std::string edge, TransportConfig cfg, const std::string&)
    : edge_(std::move(edge)), cfg_(std::move(cfg)) {
  if (cfg_.kind == TransportKind::TCP && cfg_.tcp_endpoint.empty())
    throw ConfigInvalid("tcp transport needs an endpoint on edge " + edge_);
  const auto arrow = edge_.find("->");
  if (arrow != std::string::npos) {
    from_ = edge_.substr(0, arrow);
    to_ = edge_.substr(arrow + 2);
  }
}

uint64_t Connector::payload_bytes(const Payload& p) {
  return p.is_device() ? p.dev.nbytes : payload_header_bytes(p.shape.size()) + p.bytes.size();
}

void Connector::put(const ConnectorKey& key, const Payload& p) {
  const uint64_t h = p.is_device() ? p.dev.blob : fnv1a64(encode_payload(p));
  std::lock_guard lk(mu_);
  const std::string k = key.canonical();
  auto it = kv_.find(k);
  if (it != kv_.end()) {
    const Payload& held = it->second.frame.empty()
                              ? it->second.payload
                              : payload_from_locator(decode_control_frame(it->second.frame).locator);
    if (it->second.hash == h && held == p) return;  // idempotent re-put
    throw WriteConflict(k);
  }
  Slot slot{p, {}, h, false, key.request_id};
  if (p.is_device()) {
    ControlMessage m;
    m.kind = ControlMessage::Kind::PUT_NOTICE;
    m.key = k;
    m.request_id = key.request_id;
    m.edge = edge_;
    m.locator = device_locator(p);
    slot.frame = encode_control_frame(m);
    slot.payload = Payload{};
    ++frames_;
  }
  kv_.emplace(k, std::move(slot));
  cv_.notify_all();
}

Payload Connector::get(const ConnectorKey& key, uint64_t timeout_ms) {
  std::unique_lock lk(mu_);
  const std::string k = key.canonical();
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  for (;;) {
    auto it = kv_.find(k);
    if (it != kv_.end() && !it->second.consumed) {
      it->second.consumed = true;
      if (it->second.frame.empty()) return it->second.payload;
      const ControlMessage m = decode_control_frame(it->second.frame);
      if (m.kind != ControlMessage::Kind::PUT_NOTICE || m.key != k)
        throw ProtocolViolation("put notice does not match key " + k);
      return payload_from_locator(m.locator);
    }
    if (cv_.wait_until(lk, deadline) == std::cv_status::timeout) throw TimeoutError("get timed out on " + k);
  }
}

StreamSender Connector::open_stream(uint64_t rid) {
  std::lock_guard lk(mu_);
  auto& s = streams_[rid];
  if (s.sender_open) throw AlreadyOpen("stream sender for request " + std::to_string(rid));
  s.sender_open = true;
  return StreamSender(this, rid);
}

StreamReceiver Connector::subscribe(uint64_t rid) {
  std::lock_guard lk(mu_);
  auto& s = streams_[rid];
  if (s.receiver_open) throw AlreadyOpen("stream receiver for request " + std::to_string(rid));
  s.receiver_open = true;
  return StreamReceiver(this, rid);
}

uint64_t Connector::cleanup(uint64_t rid) {
  std::lock_guard lk(mu_);
  uint64_t freed = 0;
  for (auto it = kv_.begin(); it != kv_.end();) {
    if (it->second.request_id == rid) {
      if (!it->second.consumed)
        freed += it->second.frame.empty() ? payload_bytes(it->second.payload)
                                          : decode_control_frame(it->second.frame).locator.length;
      it = kv_.erase(it);
    } else {
      ++it;
    }
  }
  auto st = streams_.find(rid);
  if (st != streams_.end()) {
    for (const auto& b : st->second.q)
      freed += b.frame.empty() ? payload_bytes(b.payload) : decode_control_frame(b.frame).locator.length;
    streams_.erase(st);
  }
  return freed;
}

void Connector::stream_send(uint64_t rid, const StreamChunk& c) {
  std::lock_guard lk(mu_);
  auto& s = streams_[rid];
  if (s.eos_sent) throw ProtocolViolation("chunk after eos");
  if (c.seq != s.next_seq)
    throw ProtocolViolation("out-of-order chunk seq " + std::to_string(c.seq) + " (expected " +
                            std::to_string(s.next_seq) + ")");
  if (c.payload.is_device()) {
    ControlMessage m;
    m.kind = c.eos ? ControlMessage::Kind::EOS : ControlMessage::Kind::CHUNK_NOTICE;
    m.request_id = rid;
    m.edge = edge_;
    m.seq = c.seq;
    m.locator = device_locator(c.payload);
    s.q.push_back(Buffered{c.seq, c.eos, Payload{}, encode_control_frame(m)});
    ++frames_;
  } else {
    s.q.push_back(Buffered{c.seq, c.eos, c.payload, {}});
  }
  ++s.next_seq;
  ++chunks_sent_;
  s.eos_sent = c.eos;
  cv_.notify_all();
}

std::optional<StreamChunk> Connector::stream_try_recv(uint64_t rid) {
  std::lock_guard lk(mu_);
  auto it = streams_.find(rid);
  if (it == streams_.end() || it->second.q.empty()) return std::nullopt;
  Buffered b = std::move(it->second.q.front());
  it->second.q.pop_front();
  StreamChunk c;
  c.request_id = rid;
  c.from = from_;
  c.to = to_;
  c.seq = b.seq;
  c.eos = b.eos;
  if (b.frame.empty()) {
    c.payload = std::move(b.payload);
    return c;
  }
  const ControlMessage m = decode_control_frame(b.frame);
  const auto want = b.eos ? ControlMessage::Kind::EOS : ControlMessage::Kind::CHUNK_NOTICE;
  if (m.kind != want || m.request_id != rid || m.seq != b.seq || m.edge != edge_)
    throw ProtocolViolation("chunk notice does not match its stream slot on edge " + edge_);
  c.payload = payload_from_locator(m.locator);
  return c;
}

StreamChunk Connector::stream_recv(uint64_t rid, uint64_t timeout_ms) {
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  for (;;) {
    if (auto c = stream_try_recv(rid)) return std::move(*c);
    std::unique_lock lk(mu_);
    auto it = streams_.find(rid);
    if (it != streams_.end() && !it->second.q.empty()) continue;
    if (cv_.wait_until(lk, deadline) == std::cv_status::timeout) throw TimeoutError("stream recv timed out");
  }
}

void StreamSender::send(const StreamChunk& c) { conn_->stream_send(rid_, c); }
std::optional<StreamChunk> StreamReceiver::try_recv() { return conn_->stream_try_recv(rid_); }
StreamChunk StreamReceiver::recv(uint64_t timeout_ms) { return conn_->stream_recv(rid_, timeout_ms); }

}  // namespace omni
