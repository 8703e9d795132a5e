#include "omni/ar_engine.hpp"

#include <algorithm>

namespace omni {

ArEngine::ArEngine(StageId stage, EngineConfig cfg, StageModel model, PreprocessFn preprocess,
                   MetricsCollector* metrics)
    : stage_(std::move(stage)),
      cfg_(std::move(cfg)),
      model_(std::move(model)),
      preprocess_(std::move(preprocess)),
      metrics_(metrics) {
  cfg_.check();
}

void ArEngine::admit(ArAdmission a) {
  if (!a.sub.prompt_streams && a.sub.prompt.size() > cfg_.kv_budget_tokens)
    throw RejectedTooLarge("prompt of " + std::to_string(a.sub.prompt.size()) +
                           " tokens exceeds kv budget " + std::to_string(cfg_.kv_budget_tokens) +
                           " on stage " + stage_);
  waiting_.push_back(std::move(a));
}

uint64_t ArEngine::resident_tokens() const {
  uint64_t n = 0;
  for (const auto& r : residents_) n += r.seq.prompt.size() + r.seq.emitted.size();
  return n;
}

ArEngine::Resident* ArEngine::find(uint64_t rid) {
  for (auto& r : residents_)
    if (r.seq.request_id == rid) return &r;
  return nullptr;
}

const SeqState* ArEngine::finished_seq(uint64_t rid) const {
  auto it = finished_.find(rid);
  return it == finished_.end() ? nullptr : &it->second;
}

bool ArEngine::ready() const {
  if (!computing_) return true;
  if (slots_.empty() || !model_.batch_ready) return true;
  return model_.batch_ready();
}

// ---- iteration ---------------------------------------------------------------
bool ArEngine::begin_iteration(uint64_t now) {
  if (computing_) throw OmniError("begin_iteration while computing");
  admit_waiting();
  run_preprocess();
  pending_ = StepReport{};
  pending_.batch = schedule_iteration();
  // Recompute preemption when decoders are blocked purely by the kv budget
  // (ar_engine.hpp:97-104): evict the youngest fixed-prompt resident.
  while (pending_.batch.entries.empty() && decode_blocked_by_budget() && preempt_youngest()) {
    admit_waiting();
    pending_.batch = schedule_iteration();
  }
  if (pending_.batch.entries.empty() && failures_.empty()) return false;
  if (metrics_)
    for (const auto& e : pending_.batch.entries) metrics_->on_stage_scheduled(e.request_id, stage_, now);
  if (model_.batched()) run_entries_batched();
  else run_entries_host();
  const uint64_t tokens = pending_.batch.total_tokens();
  pending_.cost_us = tokens > 0 ? iteration_cost_us(tokens, cfg_) : 0;
  computing_ = true;
  end_time_ = now + pending_.cost_us;
  ++iterations_;
  return true;
}

StepReport ArEngine::complete_iteration(uint64_t now) {
  if (!computing_) throw OmniError("complete_iteration while idle");
  computing_ = false;
  if (!slots_.empty()) collect_batched();
  for (const auto& e : pending_.batch.entries) {
    Resident* r = find(e.request_id);
    if (!r) continue;  // failed while running
    if (metrics_ && e.phase == Phase::DECODE) metrics_->on_stage_tokens(e.request_id, stage_, e.token_span, now);
    pending_.chunks_emitted += emit_output(*r);
  }
  if (model_.flush) model_.flush();
  // evict finished residents (their budget is released with them)
  std::vector<Resident> keep;
  keep.reserve(residents_.size());
  for (auto& r : residents_) {
    if (r.seq.phase != Phase::FINISHED) {
      keep.push_back(std::move(r));
      continue;
    }
    const uint64_t rid = r.seq.request_id;
    if (metrics_) metrics_->on_stage_finished(rid, stage_, now);
    if (model_.release) model_.release(rid);
    pending_.finished.push_back(rid);
    finished_.emplace(rid, std::move(r.seq));
  }
  residents_ = std::move(keep);
  for (auto& f : failures_) pending_.failed.push_back(std::move(f));
  failures_.clear();
  return std::move(pending_);
}

// Decoders first (request id ascending, span 1), then prefills in admission
// order capped by prefill_chunk / remaining prompt / batch budget; a sole
// resident (or an all-streamed resident set) may overrun the kv budget
// (ar_engine.hpp:149-192).
IterationBatch ArEngine::schedule_iteration() const {
  IterationBatch batch;
  uint64_t budget = cfg_.max_batch_tokens;
  const uint64_t used = resident_tokens();
  uint64_t headroom = cfg_.kv_budget_tokens > used ? cfg_.kv_budget_tokens - used : 0;

  std::vector<const Resident*> dec;
  for (const auto& r : residents_)
    if (r.seq.phase == Phase::DECODE && !r.stalled) dec.push_back(&r);
  std::sort(dec.begin(), dec.end(),
            [](const Resident* a, const Resident* b) { return a->seq.request_id < b->seq.request_id; });
  const bool several = residents_.size() > 1;
  const bool any_recomputable =
      several && std::any_of(residents_.begin(), residents_.end(),
                             [](const Resident& r) { return !r.prompt_streams; });
  for (const Resident* r : dec) {
    if (budget == 0) break;
    if (headroom == 0 && several && (any_recomputable || !batch.entries.empty())) break;
    batch.entries.push_back({r->seq.request_id, Phase::DECODE, 1});
    --budget;
    if (headroom > 0) --headroom;
  }
  for (const auto& r : residents_) {
    if (r.seq.phase != Phase::PREFILL || r.stalled) continue;
    if (budget == 0) break;
    const uint64_t remaining = r.seq.prompt.size() - r.seq.consumed_prompt;
    const uint64_t span = std::min({cfg_.prefill_chunk, remaining, budget});
    if (span == 0) continue;
    batch.entries.push_back({r.seq.request_id, Phase::PREFILL, static_cast<uint32_t>(span)});
    budget -= span;
  }
  return batch;
}

void ArEngine::admit_waiting() {
  // strict FIFO; the watermark keeps a decode reserve once anyone is resident
  while (!waiting_.empty() && residents_.size() < cfg_.max_resident_requests) {
    ArAdmission& a = waiting_.front();
    const uint64_t watermark = residents_.empty() ? 0 : cfg_.kv_budget_tokens / 16 + 1;
    if (resident_tokens() + a.sub.prompt.size() + watermark > cfg_.kv_budget_tokens) break;
    Resident r;
    r.seq.request_id = a.sub.request_id;
    r.seq.prompt = std::move(a.sub.prompt);
    r.seq.prompt_rows = std::move(a.sub.prompt_rows);
    r.seq.prompt_complete = !a.sub.prompt_streams;
    r.seq.rng_state = a.sub.seed;
    r.seed = a.sub.seed;
    r.prompt_streams = a.sub.prompt_streams;
    r.ctx = std::move(a.ctx);
    r.upstream = std::move(a.upstream);
    r.emits = std::move(a.emits);
    residents_.push_back(std::move(r));
    waiting_.pop_front();
  }
}

void ArEngine::run_preprocess() {
  for (auto& r : residents_) {
    r.stalled = false;
    if (!preprocess_) continue;
    try {
      r.stalled = preprocess_(*r.ctx, r.seq, r.upstream ? &*r.upstream : nullptr) == PreprocessStatus::STALL;
    } catch (const OmniError& e) {
      fail(r.seq.request_id, e.what());
    }
  }
  prune_failed();
}

bool ArEngine::decode_blocked_by_budget() const {
  if (resident_tokens() < cfg_.kv_budget_tokens) return false;
  return std::any_of(residents_.begin(), residents_.end(),
                     [](const Resident& r) { return r.seq.phase == Phase::DECODE && !r.stalled; });
}

bool ArEngine::preempt_youngest() {
  for (size_t i = residents_.size(); i-- > 0;) {
    if (residents_[i].prompt_streams) continue;
    if (residents_.size() <= 1) return false;
    Resident r = std::move(residents_[i]);
    residents_.erase(residents_.begin() + static_cast<std::ptrdiff_t>(i));
    if (model_.release) model_.release(r.seq.request_id);
    ArAdmission a;
    a.sub.request_id = r.seq.request_id;
    a.sub.prompt = std::move(r.seq.prompt);
    a.sub.prompt_rows = std::move(r.seq.prompt_rows);
    a.sub.prompt_streams = false;
    a.sub.seed = r.seed;
    a.ctx = std::move(r.ctx);
    a.upstream = std::move(r.upstream);
    a.emits = std::move(r.emits);  // keep sent_tokens: replay does not resend chunks
    waiting_.push_front(std::move(a));
    ++preemptions_;
    return true;
  }
  return false;
}

// Reference per-entry hook loop (ar_engine.hpp:308-337).
void ArEngine::run_entries_host() {
  for (const auto& e : pending_.batch.entries) {
    Resident* r = find(e.request_id);
    if (!r) continue;
    try {
      SeqState& s = r->seq;
      if (e.phase == Phase::PREFILL) {
        std::span<const uint8_t> span(s.prompt.data() + s.consumed_prompt, e.token_span);
        if (model_.prefill) model_.prefill(*r->ctx, s, span);
        s.consumed_prompt += e.token_span;
        if (s.prompt_complete && s.consumed_prompt == s.prompt.size()) {
          model_.on_prompt_consumed(*r->ctx, s);
          if (s.target_len < 1) throw ForwardError("model set target_len < 1");
          s.phase = Phase::DECODE;
        }
      } else {
        DecodeStep step = model_.decode(*r->ctx, s);
        s.emitted.push_back(step.token);
        if (step.has_hidden) s.hidden.push_back(step.hidden);
        if (s.emitted.size() == s.target_len) s.phase = Phase::FINISHED;
      }
    } catch (const OmniError& err) {
      fail(e.request_id, err.what());
    }
  }
  prune_failed();
}

// Batched device path: identical bookkeeping, token values filled at completion.
void ArEngine::run_entries_batched() {
  struct Pending {
    uint64_t rid;
    Phase phase;
    uint32_t span;
    size_t pos0;
    int32_t out_index;
  };
  std::vector<Pending> todo;
  todo.reserve(pending_.batch.entries.size());
  for (const auto& e : pending_.batch.entries) {
    Resident* r = find(e.request_id);
    if (!r) continue;
    try {
      SeqState& s = r->seq;
      if (e.phase == Phase::PREFILL) {
        const size_t pos0 = s.consumed_prompt;
        std::span<const uint8_t> span(s.prompt.data() + s.consumed_prompt, e.token_span);
        if (model_.prefill) model_.prefill(*r->ctx, s, span);
        s.consumed_prompt += e.token_span;
        if (s.prompt_complete && s.consumed_prompt == s.prompt.size()) {
          model_.on_prompt_consumed(*r->ctx, s);
          if (s.target_len < 1) throw ForwardError("model set target_len < 1");
          s.phase = Phase::DECODE;
        }
        todo.push_back({e.request_id, Phase::PREFILL, e.token_span, pos0, -1});
      } else {
        const size_t k = s.emitted.size();
        todo.push_back({e.request_id, Phase::DECODE, 1, s.prompt.size() + k, static_cast<int32_t>(k)});
        s.emitted.push_back(-1);  // placeholder, filled by collect_batched()
        if (s.emitted.size() == s.target_len) s.phase = Phase::FINISHED;
      }
    } catch (const OmniError& err) {
      fail(e.request_id, err.what());
    }
  }
  // device admission per entry: one sequence that cannot get KV pages fails
  // alone, before anything is launched
  if (model_.reserve) {
    for (const auto& t : todo) {
      Resident* r = find(t.rid);
      if (!r) continue;
      BatchSlot b;
      b.request_id = t.rid;
      b.phase = t.phase;
      b.span = t.span;
      b.pos0 = t.pos0;
      b.out_index = t.out_index;
      b.seq = &r->seq;
      b.ctx = r->ctx.get();
      try {
        model_.reserve(b);
      } catch (const OmniError& err) {
        fail(t.rid, err.what());
      }
    }
  }
  prune_failed();
  slots_.clear();
  for (const auto& t : todo) {
    Resident* r = find(t.rid);
    if (!r) continue;
    BatchSlot b;
    b.request_id = t.rid;
    b.phase = t.phase;
    b.span = t.span;
    b.pos0 = t.pos0;
    b.out_index = t.out_index;
    b.seq = &r->seq;
    b.ctx = r->ctx.get();
    slots_.push_back(b);
  }
  if (slots_.empty()) return;
  try {
    model_.launch_batch(slots_);
  } catch (const OmniError& err) {
    for (const auto& b : slots_) fail(b.request_id, err.what());
    slots_.clear();
    prune_failed();
  }
}

void ArEngine::collect_batched() {
  std::vector<int32_t> tokens(slots_.size(), -1);
  try {
    model_.collect_batch(slots_, tokens);
  } catch (const OmniError& err) {
    for (const auto& b : slots_) fail(b.request_id, err.what());
    slots_.clear();
    prune_failed();
    return;
  }
  for (size_t i = 0; i < slots_.size(); ++i) {
    const BatchSlot& b = slots_[i];
    if (b.phase != Phase::DECODE) continue;
    Resident* r = find(b.request_id);
    if (r) r->seq.emitted[static_cast<size_t>(b.out_index)] = tokens[i];
  }
  slots_.clear();
}

// STREAMING plans cut a chunk at every multiple of chunk_size, then the
// remainder and an empty eos chunk at finish; FULL plans send one eos chunk
// with everything at finish (ar_engine.hpp:339-365).
size_t ArEngine::emit_output(Resident& r) {
  size_t n = 0;
  const SeqState& s = r.seq;
  for (auto& plan : r.emits) {
    if (!plan.sender.valid()) continue;
    const bool done = s.phase == Phase::FINISHED;
    if (plan.mode == EdgeMode::STREAMING) {
      for (; s.emitted.size() >= plan.sent_tokens + plan.chunk_size; plan.sent_tokens += plan.chunk_size, ++n)
        send_chunk(r, plan, plan.sent_tokens, plan.sent_tokens + plan.chunk_size, false);
      if (!done) continue;
      if (plan.sent_tokens < s.emitted.size()) {
        send_chunk(r, plan, plan.sent_tokens, s.emitted.size(), false);
        plan.sent_tokens = s.emitted.size();
        ++n;
      }
      send_chunk(r, plan, plan.sent_tokens, plan.sent_tokens, true);
      ++n;
    } else if (done) {
      send_chunk(r, plan, 0, s.emitted.size(), true);
      ++n;
    }
  }
  return n;
}

void ArEngine::send_chunk(Resident& r, EmitPlan& plan, size_t b, size_t e, bool eos) {
  StreamChunk c;
  c.request_id = r.seq.request_id;
  c.seq = plan.next_seq++;
  c.eos = eos;
  c.payload = model_.pack_chunk(r.seq, b, e);
  if (plan.tokens_i32 && (c.payload.dtype != Dtype::I32 || c.payload.is_device()))
    c.payload = Payload::from_i32(std::span<const int32_t>(r.seq.emitted.data() + b, e - b));
  plan.sender.send(c);
}

void ArEngine::prune_failed() {
  if (failures_.empty()) return;
  for (const auto& [rid, why] : failures_) {
    auto it = std::find_if(residents_.begin(), residents_.end(),
                           [r = rid](const Resident& x) { return x.seq.request_id == r; });
    if (it == residents_.end()) continue;
    if (model_.release) model_.release(rid);
    residents_.erase(it);
  }
}

std::vector<uint64_t> ArEngine::abort_all() {
  std::vector<uint64_t> ids;
  for (auto& r : residents_) {
    ids.push_back(r.seq.request_id);
    if (model_.release) model_.release(r.seq.request_id);
  }
  for (auto& w : waiting_) ids.push_back(w.sub.request_id);
  residents_.clear();
  waiting_.clear();
  return ids;
}

}  // namespace omni
