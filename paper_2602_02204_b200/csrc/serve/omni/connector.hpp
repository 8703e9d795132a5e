// Per-edge data plane: keyed put/get plus exactly-once, in-order SPSC
// streams per request (reference connector.hpp:23-348). Host payloads are
// queued by value (INPROC / SHM / TCP all stay in-process here — the SHM and
// TCP byte stores are out of scope); DEVICE payloads
// are queued as locators while their blobs stay in HBM.
#pragma once
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <mutex>
#include <optional>
#include <string>

#include "omni/graph.hpp"
#include "omni/payload.hpp"

namespace omni {

struct TransportConfig {
  TransportKind kind = TransportKind::INPROC;
  uint64_t inline_threshold = 4096;
  uint64_t shm_region_bytes = 64ull << 20;
  std::string tcp_endpoint;
  std::string shm_name;
  uint64_t default_timeout_ms = 5000;
};

struct StreamChunk {
  uint64_t request_id = 0;
  std::string from;
  std::string to;
  uint32_t seq = 0;
  Payload payload;
  bool eos = false;
};

class Connector;

class StreamSender {
 public:
  StreamSender() = default;
  void send(const StreamChunk& c);
  bool valid() const { return conn_ != nullptr; }

 private:
  friend class Connector;
  StreamSender(Connector* c, uint64_t rid) : conn_(c), rid_(rid) {}
  Connector* conn_ = nullptr;
  uint64_t rid_ = 0;
};

class StreamReceiver {
 public:
  StreamReceiver() = default;
  std::optional<StreamChunk> try_recv();
  StreamChunk recv(uint64_t timeout_ms);
  bool valid() const { return conn_ != nullptr; }

 private:
  friend class Connector;
  StreamReceiver(Connector* c, uint64_t rid) : conn_(c), rid_(rid) {}
  Connector* conn_ = nullptr;
  uint64_t rid_ = 0;
};

struct ConnectorKey {
  uint64_t request_id = 0;
  std::string edge;
  std::string name;
  uint32_t index = 0;
  // req:{id}/edge:{from->to}/{name}/{index}   (control.hpp:13-23)
  std::string canonical() const;
};

class Connector {
 public:
  Connector(std::string edge, TransportConfig cfg, const std::string& server_id = "0");

  const std::string& edge() const { return edge_; }
  const TransportConfig& config() const { return cfg_; }

  void put(const ConnectorKey& key, const Payload& p);
  Payload get(const ConnectorKey& key, uint64_t timeout_ms);
  StreamSender open_stream(uint64_t request_id);
  StreamReceiver subscribe(uint64_t request_id);
  // Drops everything of a request; returns payload bytes released.
  uint64_t cleanup(uint64_t request_id);
  uint64_t chunks_sent() const { return chunks_sent_; }
  uint64_t frames_encoded() const { return frames_; }

 private:
  friend class StreamSender;
  friend class StreamReceiver;
  // Device payloads travel as encoded DEVICE control frames (control.hpp):
  // the frame is what a cross-process DEVICE transport puts on the wire, and
  // decoding it on the receive side re-checks the locator.
  struct Slot {
    Payload payload;
    std::vector<uint8_t> frame;
    uint64_t hash = 0;
    bool consumed = false;
    uint64_t request_id = 0;
  };
  struct Buffered {
    uint32_t seq;
    bool eos;
    Payload payload;
    std::vector<uint8_t> frame;
  };
  struct Stream {
    bool sender_open = false, receiver_open = false, eos_sent = false;
    uint32_t next_seq = 0;
    std::deque<Buffered> q;
  };
  void stream_send(uint64_t rid, const StreamChunk& c);
  std::optional<StreamChunk> stream_try_recv(uint64_t rid);
  StreamChunk stream_recv(uint64_t rid, uint64_t timeout_ms);
  static uint64_t payload_bytes(const Payload& p);

  std::string edge_, from_, to_;
  TransportConfig cfg_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::map<std::string, Slot> kv_;
  std::map<uint64_t, Stream> streams_;
  uint64_t chunks_sent_ = 0;
  uint64_t frames_ = 0;
};

}  // namespace omni
