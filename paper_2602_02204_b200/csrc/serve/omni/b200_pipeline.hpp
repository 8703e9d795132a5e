// The B200 stage plugins: Thinker / Talker StageModels with batched device
// steps, the device-resident hidden-state connector, the Talker preprocess
// and transfers, and the DiT denoiser — registered under the reference's
// function-table names (reference_pipeline.hpp:237-247) so the reference's
// configs run unchanged on the GPU.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "omni/clock.hpp"
#include "omni/registry.hpp"
#include "omni_dev.h"

namespace omni {

// Optional event log in the reference-harness trace format (oracle/ref_harness.cpp).
struct Tracer {
  const Clock* clock = nullptr;
  std::string out;
  uint64_t now() const { return clock ? clock->now_us() : 0; }
};

struct B200Options {
  uint64_t weight_seed = 1234;
  // forward / denoiser name -> CUDA ordinals of its replicas (placement;
  // one engine + one device stage per entry, routed by replica_for)
  std::map<std::string, std::vector<int>> devices;
  bool small_models = false;               // reduced dims (tests)
  uint64_t arena_bytes = 256ull << 20;     // hidden-state connector arena per producer
  std::map<std::string, EngineConfig> engines;  // stage limits keyed by forward name
  std::set<std::string> needed;                 // forward / denoiser names to build (empty = all)
  // forward / denoiser name -> AF_UNIX socket of the stage worker process that
  // hosts its stages (stage_worker.hpp); absent = this process
  std::map<std::string, std::string> workers;
};

class B200Pipeline {
 public:
  explicit B200Pipeline(B200Options opt);
  ~B200Pipeline();
  B200Pipeline(const B200Pipeline&) = delete;
  B200Pipeline& operator=(const B200Pipeline&) = delete;

  // Registers thinker_forward / talker_forward / ar_forward / process_input /
  // Thinker2Talker / Talker2Vocoder / denoise (+ dit_image) into `reg`.
  void register_into(FunctionRegistry& reg);
  void set_tracer(Tracer* t);
  // Parity capture (tests): keep every thinker hidden row a step writes
  // (bf16 bits, [index][d]) per request id, read back after the run.
  void set_capture(bool on);
  const std::vector<uint16_t>* captured_hidden(uint64_t rid) const;
  // Device milliseconds spent in steps, per stage kind (diagnostics).
  std::map<std::string, double> device_ms() const;
  std::map<std::string, uint64_t> step_counts() const;
  // per stage: (host ms inside launches, mean ms from result collection to next launch)
  std::map<std::string, std::pair<double, double>> host_ms() const;
  uint64_t weight_bytes() const;
  void reset_counters();

  struct Impl;

 private:
  std::unique_ptr<Impl> impl_;
};

}  // namespace omni
