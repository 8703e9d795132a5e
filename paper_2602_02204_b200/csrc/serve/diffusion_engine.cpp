#include "omni/diffusion_engine.hpp"

#include <algorithm>

namespace omni {

DiffusionEngine::DiffusionEngine(StageId stage, EngineConfig cfg, DiffusionModel model,
                                 MetricsCollector* metrics)
    : stage_(std::move(stage)), cfg_(std::move(cfg)), model_(std::move(model)), metrics_(metrics) {
  cfg_.check();
  if (!model_.denoise && !model_.batched())
    throw ConfigInvalid("diffusion stage " + stage_ + " has no denoiser");
}

std::vector<DiffusionJob> DiffusionEngine::batch_jobs(size_t max_jobs) {
  std::vector<DiffusionJob> b;
  while (!queue_.empty() && b.size() < max_jobs) {
    b.push_back(std::move(queue_.front()));
    queue_.pop_front();
  }
  return b;
}

bool DiffusionEngine::ready() const {
  if (!computing_ || launched_.empty() || !model_.batch_ready) return true;
  return model_.batch_ready();
}

bool DiffusionEngine::begin_iteration(uint64_t now) {
  if (computing_) throw OmniError("begin_iteration while computing");
  auto batch = batch_jobs(cfg_.max_resident_requests);
  if (batch.empty()) return false;
  pending_.clear();
  uint64_t cost = 0;
  for (const auto& job : batch) {
    if (metrics_) metrics_->on_stage_scheduled(job.request_id, stage_, now);
    cost = std::max(cost, iteration_cost_us(job.steps, cfg_));  // co-execution: slowest member
  }
  if (model_.batched()) {
    model_.launch_batch(batch);  // device errors propagate like the reference's denoise throw
    launched_ = std::move(batch);
  } else {
    for (auto& job : batch) {
      DiffusionOutput o;
      o.request_id = job.request_id;
      o.chunk_seq = job.chunk_seq;
      o.waveform = model_.denoise(job);
      o.eos = job.eos;
      pending_.push_back(std::move(o));
    }
  }
  computing_ = true;
  end_time_ = now + cost;
  cost_us_ = cost;
  ++iterations_;
  return true;
}

uint64_t DiffusionEngine::complete_iteration(uint64_t now) {
  if (!computing_) throw OmniError("complete_iteration while idle");
  computing_ = false;
  if (!launched_.empty()) {
    auto waves = model_.collect_batch();
    if (waves.size() != launched_.size()) throw ForwardError("denoiser returned a wrong job count");
    for (size_t i = 0; i < launched_.size(); ++i) {
      DiffusionOutput o;
      o.request_id = launched_[i].request_id;
      o.chunk_seq = launched_[i].chunk_seq;
      o.waveform = std::move(waves[i]);
      o.eos = launched_[i].eos;
      pending_.push_back(std::move(o));
    }
    launched_.clear();
  }
  // deterministic delivery order within a batch (diffusion_engine.hpp:102-107)
  std::sort(pending_.begin(), pending_.end(), [](const DiffusionOutput& a, const DiffusionOutput& b) {
    return a.request_id != b.request_id ? a.request_id < b.request_id : a.chunk_seq < b.chunk_seq;
  });
  for (const auto& o : pending_) {
    if (metrics_) {
      const uint64_t samples = o.waveform.element_count();
      if (samples > 0) metrics_->on_stage_tokens(o.request_id, stage_, samples, now);
      if (o.eos) metrics_->on_stage_finished(o.request_id, stage_, now);
    }
    if (sink_) sink_(o, now);
  }
  pending_.clear();
  return cost_us_;
}

}  // namespace omni
