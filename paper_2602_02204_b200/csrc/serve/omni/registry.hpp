// Model plugin API of a stage (reference registry.hpp:20-168), extended with
// the B200 batched-forward hooks. The four per-sequence hooks keep their
// reference signatures so reference-style plugins (and the reference's mock
// pipeline, restated under oracle/) run unchanged; a plugin that also sets
// launch_batch/collect_batch gets ONE asynchronous device step per engine
// iteration instead of one host call per entry (ar_engine.hpp:308-337).
#pragma once
#include <cstdint>
#include <functional>
#include <map>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "omni/connector.hpp"
#include "omni/context.hpp"
#include "omni/graph.hpp"
#include "omni/payload.hpp"

namespace omni {

enum class Phase { PREFILL, DECODE, FINISHED };

struct EngineConfig {
  StageId stage;
  uint64_t max_batch_tokens = 256;
  uint64_t max_resident_requests = 64;
  uint64_t kv_budget_tokens = 4096;
  uint64_t workers = 1;
  uint64_t prefill_chunk = 64;
  uint64_t step_latency_us = 1000;
  void check() const;
};

// Simulated iteration cost (virtual-clock parity mode): ceil(tokens*lat/workers).
inline uint64_t iteration_cost_us(uint64_t tokens, const EngineConfig& c) {
  return (tokens * c.step_latency_us + c.workers - 1) / c.workers;
}

struct SeqState {
  uint64_t request_id = 0;
  Phase phase = Phase::PREFILL;
  std::vector<uint8_t> prompt;
  bool prompt_complete = true;
  size_t consumed_prompt = 0;
  std::vector<int32_t> emitted;
  std::vector<HiddenState> hidden;
  uint32_t rng_state = 0;
  size_t target_len = 0;
  // B200: device address of the upstream hidden row feeding prompt token j
  // (talker conditioning; parallel to `prompt`, empty for host plugins).
  std::vector<uint64_t> prompt_rows;
};

struct IterationEntry {
  uint64_t request_id = 0;
  Phase phase = Phase::PREFILL;
  uint32_t token_span = 0;
};

struct IterationBatch {
  std::vector<IterationEntry> entries;
  uint64_t total_tokens() const {
    uint64_t n = 0;
    for (const auto& e : entries) n += e.token_span;
    return n;
  }
};

struct DecodeStep {
  int32_t token = 0;
  HiddenState hidden{};
  bool has_hidden = false;
};

// One entry of a batched device step, with the value-independent bookkeeping
// already applied by the engine.
struct BatchSlot {
  uint64_t request_id = 0;
  Phase phase = Phase::PREFILL;  // phase the entry was SCHEDULED in
  uint32_t span = 0;
  size_t pos0 = 0;               // first KV position written by the entry
  int32_t out_index = -1;        // DECODE: index of the emitted token
  SeqState* seq = nullptr;
  RequestContext* ctx = nullptr;
};

struct StageModel {
  // ---- reference hooks (registry.hpp:79-89) ----
  std::function<void(RequestContext&, SeqState&, std::span<const uint8_t>)> prefill;
  std::function<void(RequestContext&, SeqState&)> on_prompt_consumed;
  std::function<DecodeStep(RequestContext&, SeqState&)> decode;
  std::function<Payload(const SeqState&, size_t, size_t)> pack_chunk;
  // ---- B200 batched path (optional) ----
  std::function<void(std::vector<BatchSlot>&)> launch_batch;         // enqueue, return
  std::function<bool()> batch_ready;                                   // non-blocking
  std::function<void(std::vector<BatchSlot>&, std::vector<int32_t>&)> collect_batch;  // tokens per slot
  // Per-entry device admission before the batched launch (KV pages for
  // [pos0, pos0+span)); throwing fails that request alone (ar_engine.hpp:
  // 332-334 semantics) instead of the whole step.
  std::function<void(const BatchSlot&)> reserve;
  std::function<void(uint64_t)> release;  // drop device state (finish / preempt / fail)
  std::function<void()> flush;            // after an iteration's chunks are packed
  std::function<void(uint64_t)> cleanup;  // request left the pipeline
  bool batched() const { return static_cast<bool>(launch_batch); }
};

enum class PreprocessStatus { READY, STALL };
using PreprocessFn = std::function<PreprocessStatus(RequestContext&, SeqState&, StreamReceiver*)>;

struct ArSubmission {
  uint64_t request_id = 0;
  std::vector<uint8_t> prompt;
  bool prompt_streams = false;
  uint32_t seed = 0;
  std::vector<uint64_t> prompt_rows;  // B200 device rows (FULL edges)
};

struct DiffusionWiring {
  uint32_t steps = 4;
  uint32_t samples_per_token = 16;
};

struct TransferEnv {
  RequestContext& ctx;
  const TransferEdge& edge;
  const Request& request;
  std::optional<Payload> upstream_final;
  std::function<void(ArSubmission)> submit_ar;
  std::function<void(DiffusionWiring)> wire_diffusion;
};
using TransferFn = std::function<void(TransferEnv&)>;

// Diffusion job and the (B200) denoiser plugin. The reference has no hook
// here: denoise() is a built-in free function (diffusion_engine.hpp:28-43,98).
struct DiffusionJob {
  uint64_t request_id = 0;
  uint32_t chunk_seq = 0;
  Payload input;              // I32 conditioning tokens, rank 1
  uint32_t steps = 4;
  uint32_t samples_per_token = 16;
  bool eos = false;
  uint32_t token_offset = 0;  // B200: global position of input[0] (noise key)
};

struct DiffusionModel {
  // Synchronous per-job path (reference semantics).
  std::function<Payload(const DiffusionJob&)> denoise;
  // Batched asynchronous device path.
  std::function<void(const std::vector<DiffusionJob>&)> launch_batch;
  std::function<bool()> batch_ready;
  std::function<std::vector<Payload>()> collect_batch;  // one waveform per job, job order
  bool batched() const { return static_cast<bool>(launch_batch); }
};

// Replica router of a stage placed on several devices: request
// ids are dense from 1 (bench.hpp:31-56), so (rid - 1) mod R spreads a closed
// loop evenly and is decided once, at admission to the stage.
inline size_t replica_for(uint64_t request_id, size_t replicas) {
  return replicas <= 1 || request_id == 0 ? 0 : static_cast<size_t>((request_id - 1) % replicas);
}
// Name a stage replica's model is registered under: replica 0 keeps the
// reference name (registry.hpp:127-129), replica r > 0 is "name#r".
inline std::string replica_name(const std::string& n, size_t r) {
  return r == 0 ? n : n + "#" + std::to_string(r);
}

class FunctionRegistry final : public FunctionResolver {
 public:
  void register_forward(const std::string& n, StageModel m) { fwd_[n] = std::move(m); }
  void register_preprocess(const std::string& n, PreprocessFn f) { pre_[n] = std::move(f); }
  void register_transfer(const std::string& n, TransferFn f) { xfer_[n] = std::move(f); }
  // Diffusion nodes without a forward ref resolve the denoiser "denoise".
  void register_denoiser(const std::string& n, DiffusionModel m) { den_[n] = std::move(m); }

  bool has_forward(const std::string& n) const override { return fwd_.count(n) != 0; }
  bool has_preprocess(const std::string& n) const override { return pre_.count(n) != 0; }
  bool has_transfer(const std::string& n) const override { return xfer_.count(n) != 0; }
  bool has_denoiser(const std::string& n) const { return den_.count(n) != 0; }

  const StageModel& forward(const std::string& n) const { return find(fwd_, n, "forward"); }
  const PreprocessFn& preprocess(const std::string& n) const { return find(pre_, n, "preprocess"); }
  const TransferFn& transfer(const std::string& n) const { return find(xfer_, n, "transfer"); }
  const DiffusionModel& denoiser(const std::string& n) const { return find(den_, n, "denoiser"); }
  // Replica r's model: its own registration when present (device plugins
  // register one per replica), else the shared one (stateless host plugins).
  const StageModel& forward_for(const std::string& n, size_t r) const {
    auto it = fwd_.find(replica_name(n, r));
    return it != fwd_.end() ? it->second : forward(n);
  }
  const DiffusionModel& denoiser_for(const std::string& n, size_t r) const {
    auto it = den_.find(replica_name(n, r));
    return it != den_.end() ? it->second : denoiser(n);
  }

 private:
  template <typename M>
  static const typename M::mapped_type& find(const M& m, const std::string& n, const char* what) {
    auto it = m.find(n);
    if (it == m.end()) throw ConfigInvalid(std::string("unknown ") + what + ": " + n);
    return it->second;
  }
  std::map<std::string, StageModel> fwd_;
  std::map<std::string, PreprocessFn> pre_;
  std::map<std::string, TransferFn> xfer_;
  std::map<std::string, DiffusionModel> den_;
};

}  // namespace omni
