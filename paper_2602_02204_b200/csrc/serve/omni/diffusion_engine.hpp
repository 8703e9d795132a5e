// Job-granularity engine for DIFFUSION stage nodes (reference
// diffusion_engine.hpp:68-143): FIFO batches of up to max_resident_requests
// jobs, cost = the slowest member, deterministic (request, chunk) delivery.
// The denoiser is a registered DiffusionModel (B200: one batched DiT step per
// iteration) instead of the reference's built-in closed form.
#pragma once
#include <cstdint>
#include <deque>
#include <functional>
#include <vector>

#include "omni/metrics.hpp"
#include "omni/registry.hpp"

namespace omni {

struct DiffusionOutput {
  uint64_t request_id = 0;
  uint32_t chunk_seq = 0;
  Payload waveform;
  bool eos = false;
};

class DiffusionEngine {
 public:
  using OutputSink = std::function<void(const DiffusionOutput&, uint64_t now_us)>;

  DiffusionEngine(StageId stage, EngineConfig cfg, DiffusionModel model,
                  MetricsCollector* metrics = nullptr);

  const StageId& stage() const { return stage_; }
  const EngineConfig& config() const { return cfg_; }
  void set_output_sink(OutputSink s) { sink_ = std::move(s); }
  void submit(DiffusionJob job) { queue_.push_back(std::move(job)); }
  bool has_work() const { return !queue_.empty(); }
  bool computing() const { return computing_; }
  uint64_t end_time() const { return end_time_; }
  size_t queued_jobs() const { return queue_.size(); }
  bool ready() const;

  std::vector<DiffusionJob> batch_jobs(size_t max_jobs);
  bool begin_iteration(uint64_t now);
  uint64_t complete_iteration(uint64_t now);
  void abort_all() { queue_.clear(); }
  uint64_t iterations() const { return iterations_; }

 private:
  StageId stage_;
  EngineConfig cfg_;
  DiffusionModel model_;
  MetricsCollector* metrics_;
  OutputSink sink_;
  std::deque<DiffusionJob> queue_;
  std::vector<DiffusionJob> launched_;
  std::vector<DiffusionOutput> pending_;
  bool computing_ = false;
  uint64_t end_time_ = 0, cost_us_ = 0, iterations_ = 0;
};

}  // namespace omni
