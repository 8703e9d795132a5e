// Stage worker processes (multi-process stage placement).
//
// A worker process owns stages on its GPU and runs their steps for an
// orchestrator in another process. Requests and replies are the reference's
// control frames (control.hpp) over an AF_UNIX stream (ipc_channel.hpp): a
// request is a PUT_NOTICE whose key names the operation and whose INLINE
// locator carries the arguments, a reply is an ACK on the same key. The data
// plane stays on the GPU: a consumer stage's connector arena is allocated by
// its worker and exported with CUDA IPC, the producer (a Thinker in the
// orchestrator process) packs hidden rows straight into it and records an
// interprocess event the worker's step waits on before it runs.
//
// Operations (request body -> reply body; integers little-endian):
//   create      model desc, limits, dev i32, seed u64      -> stage u64, weight bytes u64
//   destroy     (stage in request_id)                      -> -
//   sm_share    sms i32                                    -> status
//   arena       dev i32, bytes u64                         -> arena u64, omni_ipc_handle, base u64
//   event       dev i32, omni_ipc_event_handle             -> event u64
//   ar_step     events, entries (seq, phase, span, pos0,
//               out_index), tokens, [cond_src, cond_row]   -> status, error, tokens, margins, step us
//   dit_step    jobs (rid, offset, n), tokens              -> status, error, samples, step us
//   release     rid u64                                    -> -
//   shutdown                                               -> -
// Steps are asynchronous for the client: it sends the request at launch and
// polls for the reply (one outstanding step per stage).
#pragma once
#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "omni/ipc_channel.hpp"
#include "omni_dev.h"

namespace omni {

// Serves one orchestrator connection until it sends shutdown or closes.
void run_stage_worker(IpcChannel& ch);

class WorkerClient {
 public:
  explicit WorkerClient(IpcChannel ch) : ch_(std::move(ch)) {}
  ~WorkerClient();
  WorkerClient(const WorkerClient&) = delete;
  WorkerClient& operator=(const WorkerClient&) = delete;

  struct StepReply {
    int32_t status = 0;
    std::string error;
    std::vector<int32_t> tokens;  // ar: per entry; dit: samples
    std::vector<float> margins;
    float step_us = 0.f;
  };

  uint64_t create_stage(const omni_model_desc& m, const omni_stage_limits& lim, int dev, uint64_t seed,
                        uint64_t* weight_bytes);
  void destroy_stage(uint64_t stage);
  void set_sm_share(uint64_t stage, int sms);
  // arena on the worker's GPU, exported: returns its id + IPC handle + the worker-local base
  uint64_t create_arena(int dev, uint64_t bytes, omni_ipc_handle* h, uint64_t* remote_base);
  uint64_t open_event(int dev, const omni_ipc_event_handle& h);
  void ar_step(uint64_t stage, const std::vector<uint64_t>& events, const omni_ar_batch& b, int n_tokens);
  void dit_step(uint64_t stage, const omni_dit_batch& b);
  void release(uint64_t stage, uint64_t rid);
  // the outstanding step reply of `stage`, if it has arrived
  std::optional<StepReply> poll(uint64_t stage);
  StepReply wait(uint64_t stage);

 private:
  ControlMessage call(const std::string& op, uint64_t id, std::vector<uint8_t> body);  // synchronous
  void send(const std::string& op, uint64_t id, std::vector<uint8_t> body);
  void pump(bool block);
  IpcChannel ch_;
  std::map<uint64_t, StepReply> done_;  // step replies by stage
  std::vector<ControlMessage> sync_;    // replies of synchronous calls
};

}  // namespace omni
