// Orchestrator: request admission and edge wiring, the discrete-event tick,
// transfers, diffusion inflow pump, output assembly and fail-fast handling.
// Event order and state transitions follow the reference
// (orchestrator.hpp:125-734) so virtual-clock runs reproduce its traces.
#include <cstdlib>
#include "omni/orchestrator.hpp"

#include <algorithm>

namespace omni {

// ---- ResultHandle -------------------------------------------------------------
const FinalOutput& ResultHandle::wait() {
  std::unique_lock lk(mu_);
  cv_.wait(lk, [&] { return done_; });
  return out_;
}
bool ResultHandle::is_done() const {
  std::lock_guard lk(mu_);
  return done_;
}
std::optional<ResultHandle::WaveChunk> ResultHandle::next_chunk() {
  std::unique_lock lk(mu_);
  cv_.wait(lk, [&] { return !chunks_.empty() || closed_; });
  if (chunks_.empty()) return std::nullopt;
  WaveChunk c = std::move(chunks_.front());
  chunks_.pop_front();
  return c;
}
void ResultHandle::push_chunk(WaveChunk c) {
  std::lock_guard lk(mu_);
  chunks_.push_back(std::move(c));
  cv_.notify_all();
}
void ResultHandle::finish(FinalOutput out) {
  std::lock_guard lk(mu_);
  out_ = std::move(out);
  done_ = closed_ = true;
  cv_.notify_all();
}

// ---- lifecycle ------------------------------------------------------------------
std::vector<int> placement_devices(const DeploymentPlan& plan, const StageId& stage, int default_dev) {
  auto it = plan.placement.find(stage);
  if (it == plan.placement.end() || it->second.empty()) return {default_dev};
  std::vector<int> devs;
  size_t at = 0;
  const std::string& v = it->second;
  while (at <= v.size()) {
    size_t end = v.find(',', at);
    if (end == std::string::npos) end = v.size();
    std::string tok = v.substr(at, end - at);
    while (!tok.empty() && tok.front() == ' ') tok.erase(tok.begin());
    while (!tok.empty() && tok.back() == ' ') tok.pop_back();
    if (tok.rfind("cuda:", 0) == 0) tok = tok.substr(5);
    if (tok.empty() || tok.find_first_not_of("0123456789") != std::string::npos)
      throw ConfigInvalid("placement." + stage + ": expected \"cuda:N[,cuda:M...]\", got \"" + v + "\"");
    devs.push_back(std::stoi(tok));
    at = end + 1;
  }
  return devs;
}

namespace {
std::unique_ptr<Clock> clock_for(const std::string& kind) {
  if (kind == "virtual") return std::make_unique<VirtualClock>();
  if (kind == "wall") return std::make_unique<WallClock>();
  if (kind == "device") return std::make_unique<DeviceClock>();
  throw ConfigInvalid("unknown clock kind: " + kind);
}
}  // namespace

Orchestrator::Orchestrator(DeploymentPlan plan, const FunctionRegistry* registry, std::unique_ptr<Clock> clock)
    : plan_(std::move(plan)), registry_(registry), clock_(clock ? std::move(clock) : clock_for(plan_.clock_kind)) {}

Orchestrator::~Orchestrator() {
  if (started_) shutdown(false);
}

void Orchestrator::validate_plan() {
  const auto v = validate_graph(plan_.graph, *registry_);
  if (!v.empty()) {
    std::string msg = "invalid stage graph:";
    for (const auto& x : v) msg += " " + violation_to_string(x);
    throw ConfigInvalid(msg);
  }
  for (const auto& n : plan_.graph.nodes) {
    auto it = plan_.engines.find(n.id);
    if (it == plan_.engines.end()) throw ConfigInvalid("missing engine config for stage " + n.id);
    it->second.check();
    if (n.kind == StageKind::DIFFUSION && !plan_.graph.edges_from(n.id).empty())
      throw ConfigInvalid("diffusion stage " + n.id + " cannot have outgoing edges");
  }
  for (const auto& [stage, _] : plan_.placement) {
    if (!plan_.graph.find_node(stage)) throw ConfigInvalid("placement names unknown stage " + stage);
    placement_devices(plan_, stage);  // throws ConfigInvalid on a malformed device list
  }
  std::set<std::string> endpoints;
  for (const auto& e : plan_.graph.edges) {
    auto it = plan_.transports.find(e.key());
    if (it != plan_.transports.end() && it->second.kind == TransportKind::TCP &&
        !endpoints.insert(it->second.tcp_endpoint).second)
      throw PortInUse("duplicate tcp endpoint " + it->second.tcp_endpoint);
  }
}

void Orchestrator::start() {
  if (started_) throw OmniError("orchestrator already started");
  validate_plan();
  topo_ = topo_order(plan_.graph);
  for (const auto& e : plan_.graph.edges) {
    TransportConfig tc;
    auto it = plan_.transports.find(e.key());
    if (it != plan_.transports.end()) tc = it->second;
    connectors_[e.key()] = std::make_unique<Connector>(e.key(), tc, plan_.server_id);
  }
  for (const auto& n : plan_.graph.nodes) {
    const EngineConfig& cfg = plan_.engines.at(n.id);
    const size_t R = placement_devices(plan_, n.id).size();
    try {
      for (size_t r = 0; r < R; ++r) {
        if (n.kind == StageKind::AR) {
          PreprocessFn pre = n.preprocess_ref.empty() ? nullptr : registry_->preprocess(n.preprocess_ref);
          const StageModel& m = registry_->forward_for(n.forward_ref, r);
          models_.push_back(m);
          ar_[n.id].push_back(std::make_unique<ArEngine>(n.id, cfg, m, pre, &metrics_));
        } else {
          const std::string den = n.forward_ref.empty() ? "denoise" : n.forward_ref;
          auto eng = std::make_unique<DiffusionEngine>(n.id, cfg, registry_->denoiser_for(den, r), &metrics_);
          eng->set_output_sink([this, id = n.id](const DiffusionOutput& o, uint64_t now) {
            on_diffusion_output(id, o, now);
          });
          diff_[n.id].push_back(std::move(eng));
        }
      }
    } catch (const ConfigInvalid&) {
      throw;
    } catch (const OmniError& e) {
      throw EngineSpawnFailed("stage " + n.id + ": " + e.what());
    }
  }
  std::vector<StageId> ar_topo, diff_topo;
  for (const auto& id : topo_) (ar_.count(id) ? ar_topo : diff_topo).push_back(id);
  text_stage_ = ar_topo.empty() ? StageId{} : ar_topo.front();
  codec_stage_ = ar_topo.empty() ? StageId{} : ar_topo.back();
  wave_stage_.clear();
  for (const auto& id : diff_topo)
    if (is_exit(id)) {
      wave_stage_ = id;
      break;
    }
  started_ = accepting_ = true;
}

void Orchestrator::serve_async() {
  if (loop_thread_.joinable()) return;
  loop_running_ = true;
  loop_thread_ = std::thread([this] { loop(); });
}

std::map<StageId, std::string> Orchestrator::health() const {
  std::map<StageId, std::string> h;
  for (const auto& n : plan_.graph.nodes) h[n.id] = started_ ? "UP" : "DOWN";
  return h;
}

std::shared_ptr<ResultHandle> Orchestrator::submit(Request req) {
  {
    std::lock_guard lk(state_mu_);
    if (!accepting_) throw Rejected("server not accepting requests");
    if (inflight_.size() + submissions_.size() >= plan_.server.admission_cap)
      throw Overloaded("admission cap reached");
    if (req.prompt_tokens.empty()) throw Rejected("empty prompt");
    if (req.prompt_tokens.size() > plan_.engines.at(plan_.graph.entry).kv_budget_tokens)
      throw Rejected("prompt exceeds entry-stage kv budget");
  }
  auto h = std::make_shared<ResultHandle>();
  {
    std::lock_guard lk(state_mu_);
    submissions_.push_back({std::move(req), h, std::nullopt});
  }
  wake_cv_.notify_all();
  return h;
}

std::shared_ptr<ResultHandle> Orchestrator::submit_at(Request req, uint64_t at_us) {
  auto h = std::make_shared<ResultHandle>();
  std::lock_guard lk(state_mu_);
  submissions_.push_back({std::move(req), h, at_us});
  return h;
}

void Orchestrator::run_until_drained() {
  std::lock_guard lk(loop_mu_);
  for (;;) {
    if (tick()) continue;
    std::lock_guard slk(state_mu_);
    if (inflight_.empty() && submissions_.empty()) break;
    fail_all_locked("pipeline stalled: no runnable engine event");
    break;
  }
}

ShutdownReport Orchestrator::shutdown(bool drain) {
  ShutdownReport rep;
  if (!started_) return rep;
  {
    std::lock_guard lk(state_mu_);
    accepting_ = false;
  }
  if (drain) {
    if (loop_thread_.joinable()) {
      std::unique_lock lk(state_mu_);
      drained_cv_.wait(lk, [&] { return inflight_.empty() && submissions_.empty(); });
    } else {
      run_until_drained();
    }
    rep.drained = completed_;
  } else {
    std::lock_guard lk(loop_mu_);
    std::lock_guard slk(state_mu_);
    rep.aborted = inflight_.size();
    fail_all_locked("shutdown");
  }
  stop_loop();
  // let in-flight device work of every engine settle before tearing down
  for (auto& [_, v] : ar_)
    for (auto& e : v)
      if (e->computing()) e->complete_iteration(clock_->now_us());
  for (auto& [_, v] : diff_)
    for (auto& e : v)
      if (e->computing()) e->complete_iteration(clock_->now_us());
  for (auto& [_, v] : ar_)
    for (auto& e : v) e->abort_all();
  for (auto& [_, v] : diff_)
    for (auto& e : v) e->abort_all();
  ar_.clear();
  diff_.clear();
  connectors_.clear();
  models_.clear();
  started_ = false;
  return rep;
}

std::vector<uint64_t> Orchestrator::replica_iterations(const StageId& s) const {
  std::vector<uint64_t> v;
  if (auto it = ar_.find(s); it != ar_.end())
    for (const auto& e : it->second) v.push_back(e->iterations());
  if (auto it = diff_.find(s); it != diff_.end())
    for (const auto& e : it->second) v.push_back(e->iterations());
  return v;
}
uint64_t Orchestrator::iterations(const StageId& s) const {
  uint64_t n = 0;
  for (uint64_t x : replica_iterations(s)) n += x;
  return n;
}
uint64_t Orchestrator::preemptions(const StageId& s) const {
  uint64_t n = 0;
  if (auto it = ar_.find(s); it != ar_.end())
    for (const auto& e : it->second) n += e->preemptions();
  return n;
}
size_t Orchestrator::replicas(const StageId& s) const {
  if (auto it = ar_.find(s); it != ar_.end()) return it->second.size();
  if (auto it = diff_.find(s); it != diff_.end()) return it->second.size();
  return 0;
}
ArEngine& Orchestrator::ar_for(const StageId& id, uint64_t rid) {
  auto& v = ar_.at(id);
  return *v[replica_for(rid, v.size())];
}
DiffusionEngine& Orchestrator::diff_for(const StageId& id, uint64_t rid) {
  auto& v = diff_.at(id);
  return *v[replica_for(rid, v.size())];
}

void Orchestrator::loop() {
  while (loop_running_) {
    bool progressed;
    {
      std::lock_guard lk(loop_mu_);
      progressed = tick();
    }
    if (!progressed) {
      {
        std::lock_guard slk(state_mu_);
        if (inflight_.empty() && submissions_.empty()) drained_cv_.notify_all();
      }
      std::unique_lock lk(wake_mu_);
      wake_cv_.wait_for(lk, std::chrono::milliseconds(5));
    }
  }
}

void Orchestrator::stop_loop() {
  loop_running_ = false;
  wake_cv_.notify_all();
  if (loop_thread_.joinable()) loop_thread_.join();
}

// ---- event loop -------------------------------------------------------------------
void Orchestrator::complete_engine(const StageId& id, size_t replica, bool diffusion, uint64_t t) {
  if (diffusion) {
    diff_[id][replica]->complete_iteration(t);
  } else {
    ArEngine& eng = *ar_[id][replica];
    StepReport rep = eng.complete_iteration(t);
    handle_ar_report(id, eng, rep, t);
  }
  pump_diffusion_inflows();
}

bool Orchestrator::tick() {
  const uint64_t now = clock_->now_us();
  if (drain_due(now)) return true;
  pump_diffusion_inflows();

  for (const auto& id : topo_) {
    if (auto a = ar_.find(id); a != ar_.end())
      for (auto& e : a->second)
        if (!e->computing() && e->has_work()) e->begin_iteration(now);
    if (auto d = diff_.find(id); d != diff_.end())
      for (auto& e : d->second)
        if (!e->computing() && e->has_work()) e->begin_iteration(now);
  }

  uint64_t next_arrival = kTimeUnset;
  {
    std::lock_guard lk(state_mu_);
    for (const auto& s : submissions_)
      if (s.at_us && *s.at_us < next_arrival) next_arrival = *s.at_us;
  }

  if (clock_->device_paced()) {
    // Complete the first engine (topo order) whose device work has finished,
    // then relaunch THAT engine at once: its next step is on the request's
    // critical path (AR decode chains), the other idle engines start on the
    // next tick. Device-paced batches are timing-dependent by nature; the
    // virtual-clock (parity) path below keeps the reference's order.
    static const bool eager = [] {
      const char* e = std::getenv("OMNI_EAGER_BEGIN");
      return !(e && e[0] == '0');
    }();
    bool busy = false;
    for (const auto& id : topo_) {
      if (auto a = ar_.find(id); a != ar_.end())
        for (size_t r = 0; r < a->second.size(); ++r) {
          ArEngine& e = *a->second[r];
          if (!e.computing()) continue;
          busy = true;
          if (!e.ready()) continue;
          complete_engine(id, r, false, clock_->now_us());
          if (eager && !e.computing() && e.has_work()) {
            pump_diffusion_inflows();
            e.begin_iteration(clock_->now_us());
          }
          return true;
        }
      if (auto d = diff_.find(id); d != diff_.end())
        for (size_t r = 0; r < d->second.size(); ++r) {
          DiffusionEngine& e = *d->second[r];
          if (!e.computing()) continue;
          busy = true;
          if (!e.ready()) continue;
          complete_engine(id, r, true, clock_->now_us());
          if (eager && !e.computing() && e.has_work()) e.begin_iteration(clock_->now_us());
          return true;
        }
    }
    if (busy) {
      std::this_thread::yield();
      return true;
    }
    if (next_arrival != kTimeUnset) {
      std::this_thread::sleep_until(std::chrono::steady_clock::now() +
                                    std::chrono::microseconds(next_arrival > now ? next_arrival - now : 0));
      return true;
    }
    return false;
  }

  uint64_t best = kTimeUnset;
  StageId best_stage;
  size_t best_rep = 0;
  bool best_diff = false;
  for (const auto& id : topo_) {
    if (auto a = ar_.find(id); a != ar_.end())
      for (size_t r = 0; r < a->second.size(); ++r)
        if (a->second[r]->computing() && a->second[r]->end_time() < best) {
          best = a->second[r]->end_time();
          best_stage = id;
          best_rep = r;
          best_diff = false;
        }
    if (auto d = diff_.find(id); d != diff_.end())
      for (size_t r = 0; r < d->second.size(); ++r)
        if (d->second[r]->computing() && d->second[r]->end_time() < best) {
          best = d->second[r]->end_time();
          best_stage = id;
          best_rep = r;
          best_diff = true;
        }
  }
  if (next_arrival < best) {
    clock_->advance_to_us(next_arrival);
    drain_due(clock_->now_us());
    return true;
  }
  if (best == kTimeUnset) return false;
  clock_->advance_to_us(best);
  complete_engine(best_stage, best_rep, best_diff, clock_->now_us());
  return true;
}

bool Orchestrator::drain_due(uint64_t now) {
  std::vector<Pending> due;
  {
    std::lock_guard lk(state_mu_);
    for (auto it = submissions_.begin(); it != submissions_.end();) {
      if (!it->at_us || *it->at_us <= now) {
        due.push_back(std::move(*it));
        it = submissions_.erase(it);
      } else {
        ++it;
      }
    }
  }
  for (auto& s : due) {
    const uint64_t at = s.at_us ? std::max(*s.at_us, now) : now;
    admit_request(std::move(s), at);
  }
  return !due.empty();
}

void Orchestrator::admit_request(Pending s, uint64_t now) {
  const uint64_t rid = s.req.request_id;
  InFlight fl;
  fl.req = std::move(s.req);
  fl.req.submitted_at_us = now;
  fl.handle = std::move(s.handle);
  fl.ctx = std::make_shared<RequestContext>(rid);
  fl.ctx->set_current_stage(plan_.graph.entry);
  fl.ctx->set_status(RequestStatus::RUNNING);
  metrics_.on_submitted(rid, now);
  InFlight* f;
  {
    std::lock_guard lk(state_mu_);
    f = &inflight_.emplace(rid, std::move(fl)).first->second;
  }
  try {
    // wire every edge: stream pair, upstream emit plan, receiver ownership;
    // STREAMING transfers fire now, FULL ones at upstream finish
    std::vector<const TransferEdge*> fire;
    for (const auto& e : plan_.graph.edges) {
      Connector& conn = *connectors_.at(e.key());
      const EdgeMode mode = (f->req.stream && e.mode == EdgeMode::STREAMING) ? EdgeMode::STREAMING : EdgeMode::FULL;
      EmitPlan plan;
      plan.edge_key = e.key();
      plan.mode = mode;
      plan.chunk_size = e.streaming_chunk_size ? e.streaming_chunk_size : 1;
      plan.sender = conn.open_stream(rid);
      // per-edge payload: a diffusion consumer conditions on the token ids
      // (I32, the reference's AR pack, reference_pipeline.hpp:227-234) even
      // when the producer's model packs something else for AR consumers
      // (the Thinker's FIX16 hidden rows) -- the reference has one pack per
      // model and fails branching graphs with BadDtype.
      plan.tokens_i32 = plan_.graph.find_node(e.to)->kind == StageKind::DIFFUSION;
      f->stage_plans[e.from].push_back(std::move(plan));
      StreamReceiver recv = conn.subscribe(rid);
      const bool to_ar = plan_.graph.find_node(e.to)->kind == StageKind::AR;
      if (mode == EdgeMode::STREAMING && to_ar) f->pending_receivers.emplace(e.key(), std::move(recv));
      else f->held_receivers.emplace(e.key(), std::move(recv));
      if (mode == EdgeMode::STREAMING) fire.push_back(&e);
    }
    for (const TransferEdge* e : fire) apply_transfer(*f, *e, std::nullopt);
    ArAdmission adm;
    adm.sub.request_id = rid;
    adm.sub.prompt = f->req.prompt_tokens;
    adm.sub.seed = f->req.seed;
    adm.ctx = f->ctx;
    adm.emits = std::move(f->stage_plans[plan_.graph.entry]);
    ar_for(plan_.graph.entry, rid).admit(std::move(adm));
  } catch (const OmniError& e) {
    fail_request(rid, plan_.graph.entry, e.what());
  }
}

void Orchestrator::apply_transfer(InFlight& f, const TransferEdge& e, std::optional<Payload> upstream_final) {
  int& count = f.transfer_count[e.key()];
  if (count != 0) throw TransferFnError("transfer on " + e.key() + " fired twice");
  ++count;
  const uint64_t rid = f.req.request_id;
  TransferEnv env{*f.ctx, e, f.req, std::move(upstream_final), nullptr, nullptr};
  env.submit_ar = [this, &f, &e, rid](ArSubmission sub) {
    ArAdmission adm;
    sub.request_id = rid;
    adm.sub = std::move(sub);
    adm.ctx = f.ctx;
    if (auto pr = f.pending_receivers.find(e.key()); pr != f.pending_receivers.end()) {
      adm.upstream = std::move(pr->second);
      f.pending_receivers.erase(pr);
    }
    adm.emits = std::move(f.stage_plans[e.to]);
    ar_for(e.to, rid).admit(std::move(adm));
  };
  env.wire_diffusion = [this, &f, &e, rid](DiffusionWiring w) {
    f.diff_wirings.push_back({w, e.to, e.key(), false, 0});
    diff_active_.insert(rid);
  };
  try {
    registry_->transfer(e.transfer_ref)(env);
  } catch (const OmniError& err) {
    throw TransferFnError("transfer " + e.transfer_ref + " on " + e.key() + ": " + err.what());
  }
}

// Same submission order as the reference's full scan of inflight_ in request
// id order (orchestrator.hpp:549-578), restricted to requests that still have
// an open diffusion wiring.
void Orchestrator::pump_diffusion_inflows() {
  std::vector<uint64_t> rids(diff_active_.begin(), diff_active_.end());
  for (uint64_t rid : rids) {
    InFlight* f = find_inflight(rid);
    if (!f) {
      diff_active_.erase(rid);
      continue;
    }
    bool open = false;
    for (auto& w : f->diff_wirings) {
      if (w.eos_seen) continue;
      auto it = f->held_receivers.find(w.edge_key);
      if (it != f->held_receivers.end()) {
        while (auto c = it->second.try_recv()) {
          DiffusionJob job;
          job.request_id = rid;
          job.chunk_seq = c->seq;
          job.input = std::move(c->payload);
          job.steps = w.params.steps;
          job.samples_per_token = w.params.samples_per_token;
          job.eos = c->eos;
          job.token_offset = w.tokens_seen;
          w.tokens_seen += static_cast<uint32_t>(job.input.element_count() * (job.input.shape.empty() ? 0 : 1));
          diff_for(w.to_stage, rid).submit(std::move(job));
          if (c->eos) {
            w.eos_seen = true;
            break;
          }
        }
      }
      open = open || !w.eos_seen;
    }
    if (!open) diff_active_.erase(rid);
  }
}

void Orchestrator::handle_ar_report(const StageId& stage, ArEngine& eng, const StepReport& rep, uint64_t now) {
  for (const auto& [rid, why] : rep.failed) fail_request(rid, stage, why);
  for (uint64_t rid : rep.finished) {
    InFlight* f = find_inflight(rid);
    if (!f) {
      eng.drop_finished(rid);
      continue;
    }
    if (const SeqState* s = eng.finished_seq(rid)) f->stage_tokens[stage] = s->emitted;
    eng.drop_finished(rid);
    try {
      for (const TransferEdge* e : plan_.graph.edges_from(stage)) {
        const EdgeMode mode =
            (f->req.stream && e->mode == EdgeMode::STREAMING) ? EdgeMode::STREAMING : EdgeMode::FULL;
        if (mode != EdgeMode::FULL) continue;
        // The FULL plan just published its single eos chunk. An AR consumer
        // gets it through the transfer; a diffusion consumer's chunk stays in
        // the receiver for the inflow pump.
        std::optional<Payload> fin;
        if (plan_.graph.find_node(e->to)->kind == StageKind::AR) {
          if (auto hr = f->held_receivers.find(e->key()); hr != f->held_receivers.end())
            if (auto c = hr->second.try_recv()) fin = std::move(c->payload);
        }
        apply_transfer(*f, *e, std::move(fin));
      }
    } catch (const OmniError& e) {
      fail_request(rid, stage, e.what());
      continue;
    }
    if (is_exit(stage)) {
      f->exits_done.insert(stage);
      maybe_finalize(rid, now);
    }
  }
}

void Orchestrator::on_diffusion_output(const StageId& stage, const DiffusionOutput& out, uint64_t now) {
  InFlight* f = find_inflight(out.request_id);
  if (!f) return;
  ExitWave& w = f->waves[stage];
  w.parts[out.chunk_seq] = out.waveform;
  if (out.eos) w.expected = out.chunk_seq + 1;
  if (is_exit(stage)) {
    if (out.waveform.element_count() > 0 || out.eos) metrics_.on_final_chunk(out.request_id, now);
    if (f->req.stream) {
      if (!f->streaming_status) {
        f->streaming_status = true;
        f->ctx->set_status(RequestStatus::STREAMING);
      }
      f->handle->push_chunk({out.chunk_seq, out.waveform, out.eos});
    }
  }
  if (w.expected && w.parts.size() == *w.expected) {
    f->exits_done.insert(stage);
    maybe_finalize(out.request_id, now);
  }
}

bool Orchestrator::is_exit(const StageId& s) const {
  return std::find(plan_.graph.exits.begin(), plan_.graph.exits.end(), s) != plan_.graph.exits.end();
}

Orchestrator::InFlight* Orchestrator::find_inflight(uint64_t rid) {
  std::lock_guard lk(state_mu_);
  auto it = inflight_.find(rid);
  return it == inflight_.end() ? nullptr : &it->second;
}

void Orchestrator::maybe_finalize(uint64_t rid, uint64_t now) {
  InFlight* f = find_inflight(rid);
  if (!f) return;
  for (const auto& x : plan_.graph.exits)
    if (!f->exits_done.count(x)) return;
  FinalOutput out;
  if (!text_stage_.empty()) out.text_tokens = f->stage_tokens[text_stage_];
  if (!codec_stage_.empty()) out.codec_tokens = f->stage_tokens[codec_stage_];
  for (const auto& [stage, w] : f->waves) {
    auto& dst = out.exit_waveforms[stage];
    for (const auto& [seq, p] : w.parts) {
      const auto s = p.as_i32();
      dst.insert(dst.end(), s.begin(), s.end());
    }
  }
  if (!wave_stage_.empty()) out.waveform = out.exit_waveforms[wave_stage_];
  metrics_.set_counts(rid, out.text_tokens.size(), out.codec_tokens.size(), out.waveform.size());
  metrics_.on_done(rid, now, "DONE");
  out.metrics = metrics_.record(rid);
  out.status = "DONE";
  f->ctx->set_status(RequestStatus::DONE);
  auto handle = f->handle;
  cleanup_request(rid);
  {
    std::lock_guard lk(state_mu_);
    inflight_.erase(rid);
    ++completed_;
  }
  diff_active_.erase(rid);
  handle->finish(std::move(out));
  if (on_done_) on_done_(rid, now);
  drained_cv_.notify_all();
}

void Orchestrator::fail_request(uint64_t rid, const StageId& stage, const std::string& why) {
  InFlight* f = find_inflight(rid);
  if (!f) return;
  metrics_.on_done(rid, clock_->now_us(), "FAILED");
  FinalOutput out;
  out.status = "FAILED";
  out.error = "stage " + stage + ": " + why;
  out.metrics = metrics_.record(rid);
  if (f->ctx->status() == RequestStatus::RUNNING || f->ctx->status() == RequestStatus::STREAMING)
    f->ctx->set_status(RequestStatus::FAILED);
  auto handle = f->handle;
  cleanup_request(rid);
  {
    std::lock_guard lk(state_mu_);
    inflight_.erase(rid);
  }
  diff_active_.erase(rid);
  handle->finish(std::move(out));
  if (on_done_) on_done_(rid, clock_->now_us());
  drained_cv_.notify_all();
}

void Orchestrator::fail_all_locked(const std::string& why) {
  std::vector<uint64_t> rids;
  for (const auto& kv : inflight_) rids.push_back(kv.first);
  for (auto& s : submissions_) {
    FinalOutput out;
    out.status = "FAILED";
    out.error = why;
    s.handle->finish(std::move(out));
  }
  submissions_.clear();
  state_mu_.unlock();
  for (uint64_t rid : rids) fail_request(rid, "orchestrator", why);
  state_mu_.lock();
}

void Orchestrator::cleanup_request(uint64_t rid) {
  for (auto& [_, c] : connectors_) c->cleanup(rid);
  for (auto& m : models_)
    if (m.cleanup) m.cleanup(rid);
}

}  // namespace omni
