// Control plane: one engine per stage node, per-edge connectors, transfer
// functions fired on edge crossings, request lifecycle and final-output
// assembly (reference orchestrator.hpp:28-765).
//
// Three pacing modes share one event loop:
//   virtual — discrete-event clock + cost model (bit-exact parity mode; the
//             device work of an iteration is collected at its virtual end)
//   wall    — reference wall-clock semantics (sleep until the modelled end)
//   device  — B200 performance mode: an iteration completes when its CUDA
//             work does (engines poll their events), timestamps are wall µs.
#pragma once
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "omni/ar_engine.hpp"
#include "omni/clock.hpp"
#include "omni/connector.hpp"
#include "omni/context.hpp"
#include "omni/diffusion_engine.hpp"
#include "omni/graph.hpp"
#include "omni/metrics.hpp"
#include "omni/registry.hpp"

namespace omni {

struct ServerOptions {
  std::string listen = "127.0.0.1:8080";
  uint64_t admission_cap = 256;
};

struct DeploymentPlan {
  StageGraph graph;
  std::map<StageId, EngineConfig> engines;
  std::map<std::string, TransportConfig> transports;  // keyed "from->to"
  // B200 placement: stage -> "cuda:N" or a comma list "cuda:1,cuda:2" of
  // replica devices. The reference declares this map and never
  // reads it (orchestrator.hpp:37); here R devices = R engine replicas of the
  // stage, requests routed by replica_for(rid, R).
  std::map<StageId, std::string> placement;
  // B200 multi-process placement: stage -> AF_UNIX socket of the stage worker
  // process (omni_worker_serve) that hosts its device stages
  std::map<StageId, std::string> workers;
  std::string clock_kind = "virtual";                 // virtual | wall | device
  ServerOptions server;
  std::string server_id = "0";
};

// Parsed placement of one stage: CUDA ordinals of its replicas, or
// {default_dev} when the plan does not place it.
std::vector<int> placement_devices(const DeploymentPlan& plan, const StageId& stage, int default_dev = 0);

struct FinalOutput {
  std::vector<int32_t> text_tokens;
  std::vector<int32_t> codec_tokens;
  std::vector<int32_t> waveform;                            // first diffusion exit
  std::map<StageId, std::vector<int32_t>> exit_waveforms;   // every diffusion exit (branching)
  MetricsRecord metrics;
  std::string status = "DONE";
  std::string error;
};

class ResultHandle {
 public:
  struct WaveChunk {
    uint32_t seq = 0;
    Payload payload;
    bool eos = false;
  };
  const FinalOutput& wait();
  bool is_done() const;
  std::optional<WaveChunk> next_chunk();

 private:
  friend class Orchestrator;
  void push_chunk(WaveChunk c);
  void finish(FinalOutput out);
  mutable std::mutex mu_;
  std::condition_variable cv_;
  bool done_ = false, closed_ = false;
  FinalOutput out_;
  std::deque<WaveChunk> chunks_;
};

struct ShutdownReport {
  uint64_t drained = 0;
  uint64_t aborted = 0;
};

class Orchestrator {
 public:
  Orchestrator(DeploymentPlan plan, const FunctionRegistry* registry, std::unique_ptr<Clock> clock = nullptr);
  ~Orchestrator();

  Clock& clock() { return *clock_; }
  MetricsCollector& metrics() { return metrics_; }
  const DeploymentPlan& plan() const { return plan_; }

  void start();
  void serve_async();
  std::map<StageId, std::string> health() const;
  std::shared_ptr<ResultHandle> submit(Request req);
  std::shared_ptr<ResultHandle> submit_at(Request req, uint64_t at_us);
  const FinalOutput& collect(const std::shared_ptr<ResultHandle>& h) { return h->wait(); }
  void run_until_drained();
  void set_on_done(std::function<void(uint64_t, uint64_t)> cb) { on_done_ = std::move(cb); }
  ShutdownReport shutdown(bool drain);

  // introspection (bench / tests)
  uint64_t iterations(const StageId& s) const;
  uint64_t preemptions(const StageId& s) const;
  size_t replicas(const StageId& s) const;
  // per-replica iteration counts (router balance)
  std::vector<uint64_t> replica_iterations(const StageId& s) const;

 private:
  struct Pending {
    Request req;
    std::shared_ptr<ResultHandle> handle;
    std::optional<uint64_t> at_us;
  };
  struct DiffWiring {
    DiffusionWiring params;
    StageId to_stage;
    std::string edge_key;
    bool eos_seen = false;
    uint32_t tokens_seen = 0;  // global position of the next chunk's first token
  };
  struct ExitWave {
    std::map<uint32_t, Payload> parts;
    std::optional<uint32_t> expected;
  };
  struct InFlight {
    Request req;
    std::shared_ptr<RequestContext> ctx;
    std::shared_ptr<ResultHandle> handle;
    std::map<StageId, std::vector<EmitPlan>> stage_plans;
    std::map<std::string, StreamReceiver> pending_receivers;
    std::map<std::string, StreamReceiver> held_receivers;
    std::vector<DiffWiring> diff_wirings;
    std::map<std::string, int> transfer_count;
    std::map<StageId, std::vector<int32_t>> stage_tokens;
    std::set<StageId> exits_done;
    std::map<StageId, ExitWave> waves;
    bool streaming_status = false;
  };

  void validate_plan();
  void loop();
  void stop_loop();
  bool tick();
  bool drain_due(uint64_t now);
  void admit_request(Pending s, uint64_t now);
  void apply_transfer(InFlight& f, const TransferEdge& e, std::optional<Payload> upstream_final);
  void pump_diffusion_inflows();
  void handle_ar_report(const StageId& stage, ArEngine& eng, const StepReport& rep, uint64_t now);
  void on_diffusion_output(const StageId& stage, const DiffusionOutput& out, uint64_t now);
  bool is_exit(const StageId& s) const;
  InFlight* find_inflight(uint64_t rid);
  void maybe_finalize(uint64_t rid, uint64_t now);
  void fail_request(uint64_t rid, const StageId& stage, const std::string& why);
  void fail_all_locked(const std::string& why);
  void cleanup_request(uint64_t rid);
  void complete_engine(const StageId& id, size_t replica, bool diffusion, uint64_t t);
  ArEngine& ar_for(const StageId& id, uint64_t rid);
  DiffusionEngine& diff_for(const StageId& id, uint64_t rid);

  DeploymentPlan plan_;
  const FunctionRegistry* registry_;
  std::unique_ptr<Clock> clock_;
  MetricsCollector metrics_;
  std::map<std::string, std::unique_ptr<Connector>> connectors_;
  // one engine per replica; replica r of a request = replica_for(rid, R)
  std::map<StageId, std::vector<std::unique_ptr<ArEngine>>> ar_;
  std::map<StageId, std::vector<std::unique_ptr<DiffusionEngine>>> diff_;
  std::vector<StageModel> models_;  // for cleanup hooks
  std::vector<StageId> topo_;
  StageId text_stage_, codec_stage_, wave_stage_;

  std::mutex loop_mu_, state_mu_, wake_mu_;
  std::condition_variable wake_cv_;
  std::condition_variable_any drained_cv_;
  std::map<uint64_t, InFlight> inflight_;
  std::set<uint64_t> diff_active_;  // requests with a not-yet-eos diffusion wiring
  std::deque<Pending> submissions_;
  std::function<void(uint64_t, uint64_t)> on_done_;
  std::thread loop_thread_;
  std::atomic<bool> loop_running_{false};
  bool started_ = false, accepting_ = false;
  uint64_t completed_ = 0;
};

}  // namespace omni
