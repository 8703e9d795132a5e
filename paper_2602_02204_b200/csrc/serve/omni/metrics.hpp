// Per-request event timelines and the serving metrics derived from them
// (reference metrics.hpp:16-143: JCT, TTFT, RTF, TPS).
#pragma once
#include <cstdint>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "omni/errors.hpp"

namespace omni {

inline constexpr uint64_t kTimeUnset = std::numeric_limits<uint64_t>::max();

struct StageTiming {
  uint64_t first_scheduled_at = kTimeUnset;
  uint64_t first_token_at = kTimeUnset;
  uint64_t finished_at = kTimeUnset;
  uint64_t tokens = 0;
};

struct MetricsRecord {
  uint64_t request_id = 0;
  uint64_t submitted_at = kTimeUnset;
  std::map<std::string, StageTiming> stages;
  uint64_t first_final_chunk_at = kTimeUnset;
  uint64_t done_at = kTimeUnset;
  uint64_t text_token_count = 0;
  uint64_t codec_token_count = 0;
  uint64_t waveform_sample_count = 0;
  uint32_t sample_rate = 16000;
  std::string status = "DONE";
};

uint64_t jct_us(const MetricsRecord& r);
uint64_t ttft_us(const MetricsRecord& r);
double rtf(const MetricsRecord& r);
double tps(const MetricsRecord& r, const std::string& stage);

class MetricsCollector {
 public:
  void on_submitted(uint64_t rid, uint64_t t);
  void on_stage_scheduled(uint64_t rid, const std::string& stage, uint64_t t);
  void on_stage_tokens(uint64_t rid, const std::string& stage, uint64_t n, uint64_t t);
  void on_stage_finished(uint64_t rid, const std::string& stage, uint64_t t);
  void on_final_chunk(uint64_t rid, uint64_t t);
  void on_done(uint64_t rid, uint64_t t, const std::string& status);
  void set_counts(uint64_t rid, uint64_t text, uint64_t codec, uint64_t wave);
  MetricsRecord record(uint64_t rid) const;
  std::vector<MetricsRecord> all() const;

 private:
  mutable std::mutex mu_;
  std::map<uint64_t, MetricsRecord> rec_;
};

}  // namespace omni
