// Continuous-batching autoregressive stage engine (reference ar_engine.hpp).
//
// Scheduling, admission, preemption and chunk emission reproduce the
// reference bit for bit (ar_engine.hpp:66-374; checked against golden traces
// of the reference in tests/golden). The forward work is either the
// reference's per-entry hook loop (plugins without launch_batch) or ONE
// asynchronous batched device step: begin_iteration applies the value-
// independent bookkeeping and launches; complete_iteration collects the
// device tokens, then emits chunks exactly like the reference.
#pragma once
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "omni/clock.hpp"
#include "omni/connector.hpp"
#include "omni/context.hpp"
#include "omni/metrics.hpp"
#include "omni/registry.hpp"

namespace omni {

struct EmitPlan {
  std::string edge_key;
  EdgeMode mode = EdgeMode::FULL;
  uint32_t chunk_size = 0;
  StreamSender sender;
  size_t sent_tokens = 0;
  uint32_t next_seq = 0;
  bool tokens_i32 = false;  // diffusion consumer: ship emitted ids as I32 (per-edge pack)
};

struct ArAdmission {
  ArSubmission sub;
  std::shared_ptr<RequestContext> ctx;
  std::optional<StreamReceiver> upstream;
  std::vector<EmitPlan> emits;
};

struct StepReport {
  IterationBatch batch;
  uint64_t cost_us = 0;
  std::vector<uint64_t> finished;
  std::vector<std::pair<uint64_t, std::string>> failed;
  uint64_t chunks_emitted = 0;
};

class ArEngine {
 public:
  ArEngine(StageId stage, EngineConfig cfg, StageModel model, PreprocessFn preprocess = nullptr,
           MetricsCollector* metrics = nullptr);

  const StageId& stage() const { return stage_; }
  const EngineConfig& config() const { return cfg_; }

  void admit(ArAdmission a);
  bool has_work() const { return !waiting_.empty() || !residents_.empty(); }
  bool computing() const { return computing_; }
  uint64_t end_time() const { return end_time_; }
  size_t resident_count() const { return residents_.size(); }
  size_t waiting_count() const { return waiting_.size(); }
  uint64_t resident_tokens() const;

  bool begin_iteration(uint64_t now);
  StepReport complete_iteration(uint64_t now);
  // Device-paced mode: has the launched iteration's device work finished?
  bool ready() const;

  IterationBatch schedule_iteration() const;
  const SeqState* finished_seq(uint64_t rid) const;
  void drop_finished(uint64_t rid) { finished_.erase(rid); }
  std::vector<uint64_t> abort_all();
  uint64_t iterations() const { return iterations_; }
  uint64_t preemptions() const { return preemptions_; }

 private:
  struct Resident {
    SeqState seq;
    std::shared_ptr<RequestContext> ctx;
    std::optional<StreamReceiver> upstream;
    std::vector<EmitPlan> emits;
    uint32_t seed = 0;
    bool prompt_streams = false;
    bool stalled = false;
  };

  Resident* find(uint64_t rid);
  void admit_waiting();
  void run_preprocess();
  bool decode_blocked_by_budget() const;
  bool preempt_youngest();
  void run_entries_host();
  void run_entries_batched();
  void collect_batched();
  size_t emit_output(Resident& r);
  void send_chunk(Resident& r, EmitPlan& plan, size_t b, size_t e, bool eos);
  void fail(uint64_t rid, const std::string& why) { failures_.emplace_back(rid, why); }
  void prune_failed();

  StageId stage_;
  EngineConfig cfg_;
  StageModel model_;
  PreprocessFn preprocess_;
  MetricsCollector* metrics_;

  std::deque<ArAdmission> waiting_;
  std::vector<Resident> residents_;  // admission order
  std::map<uint64_t, SeqState> finished_;
  bool computing_ = false;
  uint64_t end_time_ = 0;
  StepReport pending_;
  std::vector<BatchSlot> slots_;  // launched device step (batched plugins)
  std::vector<std::pair<uint64_t, std::string>> failures_;
  uint64_t iterations_ = 0, preemptions_ = 0;
};

}  // namespace omni
