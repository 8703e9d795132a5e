// Streaming front end: the reference's HttpService
// (http_service.hpp:88-212) without cpp-httplib -- a small HTTP/1.1 server on
// POSIX sockets in front of the Orchestrator, same routes and bodies:
//
//   POST /v1/generate  {"prompt_tokens": [...], "request_id"?, "seed"?, "stream"?}
//        stream=false -> {"text_tokens", "codec_tokens", "waveform_b64", "metrics"}
//        stream=true  -> chunked application/x-ndjson: one
//                        {"type":"waveform_chunk","seq","data_b64"} line per
//                        ResultHandle::next_chunk(), then {"type":"done","metrics"}
//                        or {"type":"error","error"}
//        400 malformed JSON / empty prompt / OmniError, 429 Overloaded, 500 failed request
//   GET  /v1/health    {"<stage>": "UP", ...}
//   GET  /v1/metrics   {"requests_seen", "requests_done", "requests_failed"}
//
// Waveform chunks are produced on the device (the DiT's Euler epilogue stores
// int32 samples straight into pinned host memory) and leave the process as
// base64 of little-endian int32 (http_service.hpp:45-58). One thread per
// connection, `Connection: close` after each response.
#pragma once
#include <atomic>
#include <cstdint>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "omni/orchestrator.hpp"

namespace omni {

std::string base64_encode(const uint8_t* data, size_t len);
std::string waveform_b64(const std::vector<int32_t>& samples);

class HttpService {
 public:
  explicit HttpService(Orchestrator& orch) : orch_(orch) {}
  ~HttpService() { stop(); }
  HttpService(const HttpService&) = delete;
  HttpService& operator=(const HttpService&) = delete;

  // Binds "host:port" (port 0 = any free port) and starts accepting on a
  // background thread. Throws PortInUse / TransportDown.
  void start(const std::string& listen);
  int port() const { return port_; }
  void stop();

 private:
  void accept_loop();
  void serve(int fd);
  void handle_generate(int fd, const std::string& body);

  Orchestrator& orch_;
  int listen_fd_ = -1;
  int port_ = 0;
  std::atomic<bool> running_{false};
  std::atomic<uint64_t> next_id_{1};
  std::thread accept_thread_;
  struct Conn {
    std::thread t;
    std::shared_ptr<std::atomic<bool>> done;
  };
  void reap(bool all);  // joins finished connection threads (all: every one)
  std::mutex conn_mu_;
  std::list<Conn> conns_;
};

}  // namespace omni
