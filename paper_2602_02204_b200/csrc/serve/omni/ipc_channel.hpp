// Cross-process DEVICE transport: the multi-process role the
// reference gives its SHM and TCP transports (connector.hpp:23-30, 77-90,
// shm_region.hpp, tcp_store.hpp), re-designed for payloads that stay in HBM.
//
//   * the consumer process owns the connector arena and exports it with CUDA
//     IPC (omni_arena_export); the producer maps it (omni_arena_import) and
//     its pack kernel stores the blob straight into it -- over NVLink when the
//     two processes drive different GPUs, no staging copy on either side;
//   * ordering is an interprocess CUDA event the producer records right after
//     each pack and the consumer's stage waits on (omni_stage_wait_event);
//   * the control plane is a byte stream (a connected AF_UNIX socket) carrying
//     the reference's control frames (control.hpp): HANDOFF frames for the
//     arena / event handles (INLINE locator = the raw handle bytes),
//     CHUNK_NOTICE / EOS frames with DEVICE locators whose `arena` is the
//     arena id and `offset` is relative to the arena base, ACK frames back.
//
// The stream contract is the connector's (connector.hpp:213-321): per request
// exactly-once, in order, seq == next expected, nothing after eos, checked on
// BOTH sides (the receiver cannot trust a remote sender), plus bounds checks of
// every locator against the arena it names.
#pragma once
#include <cstdint>
#include <deque>
#include <map>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "omni/connector.hpp"
#include "omni/control.hpp"

namespace omni {

class IpcChannel {
 public:
  IpcChannel() = default;
  explicit IpcChannel(int fd) : fd_(fd) {}
  IpcChannel(IpcChannel&& o) noexcept : fd_(std::exchange(o.fd_, -1)), rx_(std::move(o.rx_)) {}
  IpcChannel& operator=(IpcChannel&& o) noexcept;
  IpcChannel(const IpcChannel&) = delete;
  IpcChannel& operator=(const IpcChannel&) = delete;
  ~IpcChannel();

  // A connected pair (socketpair) -- create before fork(), keep one end per side.
  static std::pair<IpcChannel, IpcChannel> pair();
  // Rendezvous over a filesystem AF_UNIX socket path.
  static IpcChannel listen_accept(const std::string& path, uint64_t timeout_ms);
  static IpcChannel connect(const std::string& path, uint64_t timeout_ms);

  int fd() const { return fd_; }
  void send(const ControlMessage& m);
  // Non-blocking: a whole frame if one has fully arrived.
  std::optional<ControlMessage> try_recv();
  ControlMessage recv(uint64_t timeout_ms);
  uint64_t frames_sent() const { return sent_; }

 private:
  bool fill(int timeout_ms);  // reads what is available; false on timeout
  std::optional<std::vector<uint8_t>> take_frame();
  int fd_ = -1;
  std::vector<uint8_t> rx_;
  uint64_t sent_ = 0;
};

// HANDOFF frames for the handles (key "arena:<id>" / "event:<id>").
ControlMessage handoff_frame(const std::string& key, const void* bytes, size_t n);
std::vector<uint8_t> handoff_bytes(const ControlMessage& m, const std::string& key);

// Producer side of one edge: device payloads whose blobs lie inside the
// imported arena [base, base + bytes) become DEVICE locators relative to it.
class IpcStreamSender {
 public:
  IpcStreamSender(IpcChannel& ch, std::string edge, uint64_t arena_id, uint64_t arena_base, uint64_t arena_bytes)
      : ch_(&ch), edge_(std::move(edge)), arena_(arena_id), base_(arena_base), bytes_(arena_bytes) {}
  void send(const StreamChunk& c);
  // Consumer ACKs received so far (arena space of acked chunks may be reused).
  void poll_acks();
  uint64_t acked(uint64_t rid) const;

 private:
  struct St {
    uint32_t next = 0;
    bool eos = false;
    uint64_t acked = 0;
  };
  IpcChannel* ch_;
  std::string edge_;
  uint64_t arena_, base_, bytes_;
  std::map<uint64_t, St> st_;
};

// Consumer side of one edge: decodes, validates and re-bases DEVICE locators
// onto the local arena, demultiplexes per request.
class IpcStreamReceiver {
 public:
  IpcStreamReceiver(IpcChannel& ch, std::string edge, uint64_t arena_id, uint64_t local_base, uint64_t arena_bytes,
                    int32_t device)
      : ch_(&ch), edge_(std::move(edge)), arena_(arena_id), base_(local_base), bytes_(arena_bytes), dev_(device) {}
  // Drains the channel (non-blocking), then the next chunk of `rid` if any.
  std::optional<StreamChunk> try_recv(uint64_t rid);
  StreamChunk recv(uint64_t rid, uint64_t timeout_ms);
  void ack(uint64_t rid, uint32_t seq);
  // Frames that arrived for a different edge or of another kind (HANDOFF ...).
  std::deque<ControlMessage>& other() { return other_; }

 private:
  void accept(const ControlMessage& m);
  struct St {
    uint32_t next = 0;
    bool eos = false;
    std::deque<StreamChunk> q;
  };
  IpcChannel* ch_;
  std::string edge_;
  uint64_t arena_, base_, bytes_;
  int32_t dev_;
  std::map<uint64_t, St> st_;
  std::deque<ControlMessage> other_;
};

}  // namespace omni
