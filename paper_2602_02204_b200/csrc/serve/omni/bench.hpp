// Synthetic workload + serving statistics (reference bench.hpp:23-312),
// with p99 added (nearest rank, same rule as p50/p95).
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "omni/metrics.hpp"
#include "omni/orchestrator.hpp"

namespace omni::bench {

struct WorkloadSpec {
  uint64_t n = 100;
  std::string arrival = "closed-loop";  // closed-loop | poisson
  double rate = 1.0;
  uint64_t seed = 0;
  uint32_t prompt_min = 16;
  uint32_t prompt_max = 128;
  bool stream = true;
};

// Deterministic under a seed; bit-identical to the reference generator with
// libstdc++ (mt19937_64 + uniform_int / exponential distributions).
std::vector<Request> gen_workload(const WorkloadSpec& spec);

struct BenchRow {
  uint64_t request_id = 0, submitted_at = 0, jct_us = 0, ttft_us = 0;
  double rtf = 0, thinker_tps = 0, talker_tps = 0;
  uint64_t text_tokens = 0, codec_tokens = 0, waveform_samples = 0;
  std::string status = "DONE";
};

struct SummaryStats {
  double jct_us = 0, ttft_us = 0, rtf = 0, thinker_tps = 0, talker_tps = 0;
  double text_tokens = 0, codec_tokens = 0, waveform_samples = 0;
};

struct BenchReport {
  std::string mode;
  std::vector<BenchRow> rows;
  SummaryStats mean, p50, p95, p99;
  std::map<StageId, double> stage_share;
  std::string csv;
  uint64_t makespan_us = 0;     // first admission -> last completion
  double requests_per_s = 0;
  uint64_t completed = 0;
};

double nearest_rank(std::vector<double> v, double q);
void summarize(const std::vector<BenchRow>& rows, SummaryStats& mean, SummaryStats& p50,
               SummaryStats& p95, SummaryStats* p99 = nullptr);
// Missing stages (e.g. a single-stage graph has no talker) leave tps at 0.
BenchRow row_from_record(const MetricsRecord& rec, const StageId& thinker, const StageId& talker);
std::string render_csv(const BenchReport& rep, const WorkloadSpec& spec);
void finish_report(BenchReport& rep, const std::vector<MetricsRecord>& recs, const WorkloadSpec& spec);

struct BenchOptions {
  uint64_t concurrency = 16;
  StageId thinker_stage = "thinker";
  StageId talker_stage = "talker";
};

// Closed-loop / poisson driver over an Orchestrator (bench.hpp:225-269).
// Keeps the plan's clock kind (virtual for parity, device for performance).
BenchReport run_bench_disaggregated(DeploymentPlan plan, const FunctionRegistry& reg,
                                    std::vector<Request> workload, const WorkloadSpec& spec,
                                    const BenchOptions& opt = {});

}  // namespace omni::bench
