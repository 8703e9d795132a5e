// B200 stage plugins over the libomni_dev C ABI (include/omni_dev.h).
//
//   thinker_forward  StageModel: host keeps the reference's length semantics
//                    (fold_prompt / target_length, reference_pipeline.hpp:24-32,
//                    98-103); every iteration is ONE omni_ar_step; chunks are
//                    FIX16 {n, 1+d} payloads packed on device (omni_pack_hidden)
//                    into the consumer's arena — one pack launch per iteration.
//   talker_forward   StageModel: target_len = 4 x |prompt| (:133-135); prefill
//                    rows read the thinker hidden rows straight from the arena.
//   ar_forward       thinker model whose chunks are plain I32 tokens (:227-234).
//   process_input    Talker preprocess over device chunks (:159-190 semantics).
//   Thinker2Talker / Talker2Vocoder   transfers (:192-223).
//   denoise          DiffusionModel: ONE omni_dit_step per diffusion iteration.
#include "omni/b200_pipeline.hpp"

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <optional>
#include <unordered_map>

#include "omni/errors.hpp"
#include "omni/stage_worker.hpp"

namespace omni {

namespace {

void dev_ok(omni_status s, const char* what) {
  if (s != OMNI_OK) throw DeviceError(std::string(what) + ": " + omni_last_error());
}

uint32_t mix(uint32_t h, uint32_t t) { return h * 1000003u + t + 1u; }  // reference_pipeline.hpp:20-22

// First-fit allocator over a device arena; blocks are owned per request and
// released when the request leaves the pipeline (connector cleanup).
class Arena {
 public:
  Arena(int dev, uint64_t bytes) : dev_(dev), bytes_(bytes) {
    dev_ok(omni_arena_create(dev, bytes, &arena_), "omni_arena_create");
    dev_ok(omni_arena_base(arena_, &base_, nullptr), "omni_arena_base");
    remote_base_ = base_;
    free_[0] = bytes;
  }
  // An arena a stage worker allocated and exported (CUDA IPC), mapped here:
  // producers in this process pack into it; addresses handed to the worker
  // are rebased onto its own mapping.
  Arena(WorkerClient& w, int dev, uint64_t bytes) : dev_(dev), bytes_(bytes) {
    omni_ipc_handle h{};
    w.create_arena(dev, bytes, &h, &remote_base_);
    dev_ok(omni_arena_import(&h, &arena_), "omni_arena_import");
    dev_ok(omni_arena_base(arena_, &base_, nullptr), "omni_arena_base");
    free_[0] = bytes;
  }
  ~Arena() { omni_arena_destroy(arena_); }
  uint64_t base() const { return base_; }
  int device() const { return dev_; }
  // a local address inside the arena -> the same byte in the worker's mapping
  uint64_t rebase(uint64_t addr) const { return addr ? addr - base_ + remote_base_ : 0; }
  uint64_t alloc(uint64_t rid, uint64_t n) {
    n = (n + 255) & ~uint64_t(255);
    for (auto it = free_.begin(); it != free_.end(); ++it) {
      if (it->second < n) continue;
      const uint64_t off = it->first, rest = it->second - n;
      free_.erase(it);
      if (rest) free_[off + n] = rest;
      owned_[rid].push_back({off, n});
      return off;
    }
    throw RegionFull("hidden-state arena exhausted (" + std::to_string(bytes_) + " bytes)");
  }
  void release(uint64_t rid) {
    auto it = owned_.find(rid);
    if (it == owned_.end()) return;
    for (auto [off, n] : it->second) {
      auto nx = free_.emplace(off, n).first;
      if (auto after = std::next(nx); after != free_.end() && nx->first + nx->second == after->first) {
        nx->second += after->second;
        free_.erase(after);
      }
      if (nx != free_.begin()) {
        auto before = std::prev(nx);
        if (before->first + before->second == nx->first) {
          before->second += nx->second;
          free_.erase(nx);
        }
      }
    }
    owned_.erase(it);
  }

 private:
  omni_arena* arena_ = nullptr;
  int dev_ = 0;
  uint64_t base_ = 0, bytes_ = 0, remote_base_ = 0;
  std::map<uint64_t, uint64_t> free_;
  std::unordered_map<uint64_t, std::vector<std::pair<uint64_t, uint64_t>>> owned_;
};

// Host-side cost of driving a stage: wall time inside launch() (descriptor
// build + C-ABI step call) and the gap from "previous step's results
// collected" to "next step launched" (control-plane latency on the chain).
struct HostTimer {
  using clk = std::chrono::steady_clock;
  double host_ms = 0, gap_ms = 0;
  uint64_t gaps = 0;
  clk::time_point t_ready{};
  bool have_ready = false;
  struct Scope {
    HostTimer& h;
    clk::time_point t0;
    explicit Scope(HostTimer& x) : h(x), t0(clk::now()) {
      if (h.have_ready) {
        h.gap_ms += std::chrono::duration<double, std::milli>(t0 - h.t_ready).count();
        ++h.gaps;
        h.have_ready = false;
      }
    }
    ~Scope() { h.host_ms += std::chrono::duration<double, std::milli>(clk::now() - t0).count(); }
  };
  void ready() {
    t_ready = clk::now();
    have_ready = true;
  }
  void reset() { host_ms = gap_ms = 0, gaps = 0, have_ready = false; }
};

struct ArStage {
  std::string name;  // forward name (trace lines); the registry key adds "#r" for replicas
  int kind = OMNI_MODEL_THINKER;
  int dev = 0;
  omni_model_desc model{};
  omni_stage* st = nullptr;
  bool pack_hidden = false;  // thinker_forward: FIX16 device chunks
  // thinker: the connector arena of each consumer (talker) replica, indexed
  // by replica_for(rid, n) -- the same router the orchestrator admits with,
  // so a request's rows land on the GPU of the talker replica that reads them
  std::vector<Arena*> dst_arenas;
  std::vector<ArStage*> upstreams;  // talker: every thinker replica that packs into its arena
  Tracer* tracer = nullptr;
  // parity capture (tests): thinker hidden rows per request, [index][d] bf16 bits
  std::map<uint64_t, std::vector<uint16_t>>* capture = nullptr;
  // stage hosted by a worker process (omni_stage calls become requests)
  WorkerClient* remote = nullptr;
  uint64_t remote_id = 0, remote_weight_bytes = 0;
  Arena* own_arena = nullptr;             // remote talker: its connector arena (rebase)
  std::vector<uint64_t> wait_events;      // remote talker: upstream pack events (worker ids)
  omni_ipc_event* pack_event = nullptr;   // thinker packing into a worker's arena
  bool pack_remote = false;
  std::optional<WorkerClient::StepReply> reply;
  // step arrays (kept alive until the step completes)
  std::vector<uint64_t> seq_id, cond_src;
  std::vector<int32_t> phase, span, pos0, out_index, tokens, cond_row, tok_out;
  std::vector<float> margin_out;
  bool in_flight = false;
  double dev_ms = 0;
  uint64_t steps = 0;
  HostTimer ht;
  // deferred packs of the current iteration
  struct Pack {
    uint64_t rid;
    int32_t begin, end;
    uint64_t offset;  // absolute device address of the blob
  };
  std::vector<Pack> packs;
  std::vector<int32_t> pack_tokens;

  ~ArStage() {
    if (st) omni_stage_destroy(st);
    if (remote && remote_id) remote->destroy_stage(remote_id);
    if (pack_event) omni_ipc_event_destroy(pack_event);
  }

  void launch(std::vector<BatchSlot>& slots) {
    HostTimer::Scope hs(ht);
    const size_t n = slots.size();
    seq_id.resize(n);
    phase.resize(n);
    span.resize(n);
    pos0.resize(n);
    out_index.resize(n);
    tok_out.assign(n, -1);
    margin_out.assign(n, 0.f);
    tokens.clear();
    cond_src.clear();
    cond_row.clear();
    const bool talker = kind == OMNI_MODEL_TALKER;
    bool reads_rows = false;
    for (size_t i = 0; i < n; ++i) {
      const BatchSlot& b = slots[i];
      const SeqState& s = *b.seq;
      seq_id[i] = b.request_id;
      phase[i] = b.phase == Phase::DECODE ? OMNI_PHASE_DECODE : OMNI_PHASE_PREFILL;
      span[i] = static_cast<int32_t>(b.span);
      pos0[i] = static_cast<int32_t>(b.pos0);
      out_index[i] = b.out_index;
      if (b.phase == Phase::PREFILL) {
        for (uint32_t t = 0; t < b.span; ++t) {
          const size_t j = b.pos0 + t;
          tokens.push_back(s.prompt[j]);
          if (talker) {
            if (j >= s.prompt_rows.size()) throw ForwardError("talker prompt row without a hidden row");
            cond_src.push_back(s.prompt_rows[j]);
            cond_row.push_back(static_cast<int32_t>(j));
            reads_rows = true;
          }
        }
      } else {
        const int32_t k = b.out_index;
        tokens.push_back(k == 0 ? -1 : s.emitted[static_cast<size_t>(k - 1)]);
        if (talker) {
          cond_src.push_back(0);
          cond_row.push_back(k / 4);  // row j = m / 4 (reference_pipeline.hpp:137-139)
        }
      }
      if (tracer && b.phase == Phase::DECODE)
        tracer->out += "D " + name + " " + std::to_string(tracer->now()) + " " + std::to_string(b.request_id) +
                       " " + std::to_string(b.out_index) + "\n";
    }
    // order this step after the packs that wrote its rows (possibly on other
    // GPUs) -- only the packs, not the producers' later steps
    if (reads_rows && !remote)
      for (ArStage* up : upstreams) dev_ok(omni_stage_after_pack(st, up->st), "omni_stage_after_pack");
    omni_ar_batch batch{};
    batch.n_entries = static_cast<int32_t>(n);
    batch.seq_id = seq_id.data();
    batch.phase = phase.data();
    batch.span = span.data();
    batch.pos0 = pos0.data();
    batch.out_index = out_index.data();
    batch.tokens = tokens.data();
    if (talker) {
      batch.cond_src = cond_src.data();
      batch.cond_row = cond_row.data();
    }
    in_flight = true;
    if (remote) {
      if (talker)  // hidden-row addresses in the worker's mapping of its arena
        for (auto& a : cond_src) a = own_arena->rebase(a);
      static const std::vector<uint64_t> none;
      reply.reset();
      remote->ar_step(remote_id, reads_rows ? wait_events : none, batch, static_cast<int>(tokens.size()));
      return;
    }
    dev_ok(omni_ar_step(st, &batch, tok_out.data(), margin_out.data()), "omni_ar_step");
  }

  bool ready() {
    if (remote) {
      if (!reply) reply = remote->poll(remote_id);
      return reply.has_value();
    }
    const omni_status s = omni_stage_query(st);
    if (s == OMNI_EAGAIN) return false;
    dev_ok(s, "omni_stage_query");
    return true;
  }

  void collect(std::vector<BatchSlot>& slots, std::vector<int32_t>& out) {
    float us = 0;
    if (remote) {
      if (!reply) reply = remote->wait(remote_id);
      if (reply->status != OMNI_OK) throw DeviceError("remote omni_ar_step: " + reply->error);
      std::copy(reply->tokens.begin(), reply->tokens.end(), tok_out.begin());
      std::copy(reply->margins.begin(), reply->margins.end(), margin_out.begin());
      us = reply->step_us;
      reply.reset();
    } else {
      dev_ok(omni_stage_wait(st), "omni_stage_wait");
      omni_stage_last_step_us(st, &us);
    }
    ht.ready();
    in_flight = false;
    dev_ms += us / 1e3;
    ++steps;
    for (size_t i = 0; i < slots.size(); ++i) {
      out[i] = tok_out[i];
      if (slots[i].phase == Phase::DECODE && tok_out[i] < 0) throw ForwardError("device step returned no token");
    }
    if (capture && kind == OMNI_MODEL_THINKER) capture_rows(slots);
  }

  // Copies the hidden-ring rows the step just wrote to the host (parity tests only).
  void capture_rows(const std::vector<BatchSlot>& slots) {
    const size_t d = static_cast<size_t>(model.d_model);
    for (const BatchSlot& b : slots) {
      if (b.phase != Phase::DECODE) continue;
      uint64_t row = 0;
      dev_ok(omni_seq_hidden_row(st, b.request_id, b.out_index, &row), "omni_seq_hidden_row");
      auto& v = (*capture)[b.request_id];
      if (v.size() < (static_cast<size_t>(b.out_index) + 1) * d) v.resize((static_cast<size_t>(b.out_index) + 1) * d);
      dev_ok(omni_mem_d2h(v.data() + static_cast<size_t>(b.out_index) * d, row, d * 2), "omni_mem_d2h");
    }
  }

  Payload pack_chunk(const SeqState& s, size_t b, size_t e) {
    if (tracer)
      tracer->out += "K " + name + " " + std::to_string(tracer->now()) + " " + std::to_string(s.request_id) +
                     " " + std::to_string(b) + " " + std::to_string(e) + "\n";
    if (!pack_hidden) return Payload::from_i32(std::span<const int32_t>(s.emitted.data() + b, e - b));
    const int32_t rows = static_cast<int32_t>(e - b);
    const uint64_t nbytes = omni_pack_bytes(rows, model.d_model);
    Arena* arena = dst_arenas.at(replica_for(s.request_id, dst_arenas.size()));
    const uint64_t addr = arena->base() + arena->alloc(s.request_id, nbytes);
    packs.push_back({s.request_id, static_cast<int32_t>(b), static_cast<int32_t>(e), addr});
    Payload p;
    p.dtype = Dtype::FIX16;
    p.shape = {static_cast<uint32_t>(rows), static_cast<uint32_t>(model.d_model + 1)};
    p.dev.device = arena->device();
    p.dev.blob = addr;
    p.dev.nbytes = nbytes;
    p.host_tokens.assign(s.emitted.begin() + static_cast<std::ptrdiff_t>(b),
                         s.emitted.begin() + static_cast<std::ptrdiff_t>(e));
    pack_tokens.insert(pack_tokens.end(), p.host_tokens.begin(), p.host_tokens.end());
    return p;
  }

  void flush() {
    if (packs.empty()) return;
    std::vector<uint64_t> sid, off;
    std::vector<int32_t> b, e;
    for (const auto& p : packs) {
      sid.push_back(p.rid);
      b.push_back(p.begin);
      e.push_back(p.end);
      off.push_back(p.offset);
    }
    // absolute destinations (dst_base 0): one launch may write several
    // consumer GPUs' arenas (remote stores over NVLink)
    dev_ok(omni_pack_hidden(st, static_cast<int32_t>(packs.size()), sid.data(), b.data(), e.data(),
                            pack_tokens.data(), 0, off.data()),
           "omni_pack_hidden");
    // consumers in worker processes wait on this interprocess event
    if (pack_remote) dev_ok(omni_stage_record_pack(st, pack_event), "omni_stage_record_pack");
    packs.clear();
    pack_tokens.clear();
  }
};

// The DiT plugin: one diffusion iteration's jobs (diffusion_engine.hpp:84-112)
// become ONE batched omni_dit_step. The DiT is token-local and batch-
// invariant, so samples are bit-identical for any batching / chunking
// (test_dit_parity_and_chunking).
struct DitStage {
  std::string name;
  int dev = 0;
  omni_model_desc model{};
  omni_stage* st = nullptr;
  Tracer* tracer = nullptr;
  std::vector<uint64_t> rid;
  std::vector<int32_t> off, ntok, tokens, samples;
  double dev_ms = 0;
  uint64_t steps = 0;
  HostTimer ht;
  WorkerClient* remote = nullptr;
  uint64_t remote_id = 0, remote_weight_bytes = 0;
  std::optional<WorkerClient::StepReply> reply;
  ~DitStage() {
    if (st) omni_stage_destroy(st);
    if (remote && remote_id) remote->destroy_stage(remote_id);
  }
  void launch(const std::vector<DiffusionJob>& jobs) {
    HostTimer::Scope hs(ht);
    rid.clear(), off.clear(), ntok.clear(), tokens.clear();
    for (const auto& j : jobs) {
      if (j.input.dtype != Dtype::I32 || j.input.is_device())
        throw BadDtype("diffusion input must be I32 codec tokens");
      const auto t = j.input.as_i32();
      rid.push_back(j.request_id);
      off.push_back(static_cast<int32_t>(j.token_offset));
      ntok.push_back(static_cast<int32_t>(t.size()));
      tokens.insert(tokens.end(), t.begin(), t.end());
    }
    samples.assign(tokens.size() * static_cast<size_t>(model.dit_samples), 0);
    omni_dit_batch b{};
    b.n_jobs = static_cast<int32_t>(jobs.size());
    b.request_id = rid.data();
    b.token_offset = off.data();
    b.n_tokens = ntok.data();
    b.tokens = tokens.data();
    if (remote) {
      reply.reset();
      remote->dit_step(remote_id, b);
      return;
    }
    dev_ok(omni_dit_step(st, &b, samples.data()), "omni_dit_step");
  }
  bool ready() {
    if (remote) {
      if (!reply) reply = remote->poll(remote_id);
      return reply.has_value();
    }
    const omni_status s = omni_stage_query(st);
    if (s == OMNI_EAGAIN) return false;
    dev_ok(s, "omni_stage_query");
    return true;
  }
  std::vector<Payload> collect() {
    float us = 0;
    if (remote) {
      if (!reply) reply = remote->wait(remote_id);
      if (reply->status != OMNI_OK) throw DeviceError("remote omni_dit_step: " + reply->error);
      if (reply->tokens.size() != samples.size()) throw ProtocolViolation("remote DiT returned a wrong sample count");
      samples = std::move(reply->tokens);
      us = reply->step_us;
      reply.reset();
    } else {
      dev_ok(omni_stage_wait(st), "omni_stage_wait");
      omni_stage_last_step_us(st, &us);
    }
    ht.ready();
    dev_ms += us / 1e3;
    ++steps;
    std::vector<Payload> out(ntok.size());
    size_t at = 0;
    for (size_t k = 0; k < ntok.size(); ++k) {
      const size_t m = static_cast<size_t>(ntok[k]) * model.dit_samples;
      out[k] = Payload::from_i32(std::span<const int32_t>(samples.data() + at, m));
      at += m;
    }
    return out;
  }
};

omni_model_desc model_for(int kind, bool small) {
  omni_model_desc m{};
  dev_ok(omni_model_default(kind, &m), "omni_model_default");
  if (small) {
    if (kind == OMNI_MODEL_DIT) {
      m.d_model = 256;
      m.n_layers = 2;
      m.n_heads = 2;
      m.n_kv_heads = 2;
      m.d_ff = 512;
    } else {
      m.d_model = 512;
      m.n_layers = 2;
      m.n_heads = 4;
      m.n_kv_heads = 2;
      m.d_ff = 1024;
      if (kind == OMNI_MODEL_TALKER) m.cond_dim = 512;
    }
  }
  return m;
}

}  // namespace

struct B200Pipeline::Impl {
  B200Options opt;
  // declared first: destroyed last, after every stage / arena that uses them
  std::map<std::string, std::unique_ptr<WorkerClient>> clients;  // by worker socket
  std::vector<std::unique_ptr<Arena>> remote_arenas;             // exported by workers, mapped here
  std::map<uint64_t, std::vector<uint16_t>> captured;
  // keyed by registry name: the forward name for replica 0, "name#r" after
  std::map<std::string, std::unique_ptr<ArStage>> ar;
  std::map<std::string, std::unique_ptr<DitStage>> dit;
  std::map<int, std::unique_ptr<Arena>> arenas;  // connector arena per consumer GPU
  Tracer* tracer = nullptr;

  std::vector<int> devices_of(const std::string& name) const {
    auto it = opt.devices.find(name);
    return it == opt.devices.end() || it->second.empty() ? std::vector<int>{0} : it->second;
  }
  EngineConfig engine_of(const std::string& name) const {
    auto it = opt.engines.find(name);
    return it == opt.engines.end() ? EngineConfig{} : it->second;
  }
  Arena& arena_on(int dev) {
    auto& a = arenas[dev];
    if (!a) a = std::make_unique<Arena>(dev, opt.arena_bytes);
    return *a;
  }
  // the worker hosting stage `name`'s replica on `dev`: by stage, else by
  // device ("cuda:N" keys) -- the Thinker always stays here (it packs)
  WorkerClient* worker_for(const std::string& name, int dev) {
    auto it = opt.workers.find(name);
    if (it == opt.workers.end() && name != "thinker_forward") it = opt.workers.find("cuda:" + std::to_string(dev));
    if (it == opt.workers.end()) return nullptr;
    auto& c = clients[it->second];
    if (!c) c = std::make_unique<WorkerClient>(IpcChannel::connect(it->second, 60000));
    return c.get();
  }

  std::vector<ArStage*> make_ar(const std::string& name, int kind, uint64_t seed_salt) {
    std::vector<ArStage*> out;
    const std::vector<int> devs = devices_of(name);
    const EngineConfig ec = engine_of(name);
    for (size_t r = 0; r < devs.size(); ++r) {
      auto s = std::make_unique<ArStage>();
      s->name = name;
      s->kind = kind;
      s->dev = devs[r];
      s->model = model_for(kind, opt.small_models);
      omni_stage_limits lim{};
      lim.max_batch_tokens = static_cast<int32_t>(std::max<uint64_t>(ec.max_batch_tokens, 16));
      lim.max_resident = static_cast<int32_t>(ec.max_resident_requests);
      if (kind == OMNI_MODEL_TALKER) {
        // prompt = the Thinker's text (<= 64 rows) + 4 codec tokens per row
        lim.max_seq_len = 64 + 256 + 16;
      } else {
        // any prompt the engine admits (<= kv_budget_tokens, ar_engine.hpp:66-70)
        // plus up to 64 generated tokens (target_length, reference_pipeline.hpp:
        // 30-32); the page pool holds the kv budget plus the decode overrun the
        // schedule allows (a sole resident, one token per decoder per step)
        lim.max_seq_len = static_cast<int32_t>(ec.kv_budget_tokens + 64);
        const uint64_t tokens = ec.kv_budget_tokens + 64 + 2 * ec.max_resident_requests;
        lim.kv_pages = static_cast<int32_t>((tokens + 15) / 16 + ec.max_resident_requests);
      }
      // identical weights on every replica (same seed)
      if ((s->remote = worker_for(name, s->dev)))
        s->remote_id = s->remote->create_stage(s->model, lim, s->dev, opt.weight_seed + seed_salt,
                                               &s->remote_weight_bytes);
      else
        dev_ok(omni_stage_create(&s->model, &lim, s->dev, opt.weight_seed + seed_salt, &s->st),
               "omni_stage_create");
      out.push_back(s.get());
      ar[replica_name(name, r)] = std::move(s);
    }
    return out;
  }
};

// SMs of the persistent DiT iteration when it shares its GPU with AR stages.
// 48 leaves 100 SMs: a Thinker QKV grid (192 CTAs, two per SM) still fits in
// one wave beside it. Pipeline req/s by share (profiles/r02_dit_sm_share.txt):
// 32: 173, 40: 204, 44: 212, 48: 214-218, 52: 205-212, 56: 197-205, 64: 193-200.
constexpr int32_t kDitSharedSms = 48;

B200Pipeline::B200Pipeline(B200Options opt) : impl_(std::make_unique<Impl>()) {
  impl_->opt = std::move(opt);
  int32_t n = 0;
  if (omni_device_count(&n) != OMNI_OK || n == 0)
    throw DeviceError("no CUDA device: the B200 pipeline has no CPU fallback");
  std::vector<int32_t> devs;
  for (const auto& [_, v] : impl_->opt.devices) devs.insert(devs.end(), v.begin(), v.end());
  if (devs.empty()) devs.push_back(0);
  std::sort(devs.begin(), devs.end());
  devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
  for (int d : devs)
    if (d < 0 || d >= n)
      throw ConfigInvalid("placement names cuda:" + std::to_string(d) + " but " + std::to_string(n) +
                          " device(s) are visible");
  dev_ok(omni_init(static_cast<int32_t>(devs.size()), devs.data()), "omni_init");
  auto& I = *impl_;
  if (I.opt.workers.count("thinker_forward"))
    throw ConfigInvalid("the Thinker packs the connector and stays in the orchestrator process; "
                        "place its consumers in workers instead");
  auto want = [&I](const std::string& n) { return I.opt.needed.empty() || I.opt.needed.count(n) != 0; };
  // weight seeds: thinker / ar share the thinker model family, talker and DiT own seeds
  std::vector<ArStage*> thinkers, talkers;
  if (want("thinker_forward") || want("talker_forward")) {
    thinkers = I.make_ar("thinker_forward", OMNI_MODEL_THINKER, 0);
    for (ArStage* t : thinkers) t->pack_hidden = true;
  }
  if (want("talker_forward")) {
    talkers = I.make_ar("talker_forward", OMNI_MODEL_TALKER, 1);
    for (ArStage* t : talkers) t->upstreams = thinkers;
  }
  // connector arenas live on the consumer's GPU; with no talker in the graph
  // the thinker's chunks stay on its own GPU
  std::vector<Arena*> dst;
  for (ArStage* t : talkers) {
    if (t->remote) {  // the arena belongs to the worker; producers here map it (CUDA IPC)
      I.remote_arenas.push_back(std::make_unique<Arena>(*t->remote, t->dev, I.opt.arena_bytes));
      t->own_arena = I.remote_arenas.back().get();
    } else {
      t->own_arena = &I.arena_on(t->dev);
    }
    dst.push_back(t->own_arena);
  }
  // a worker's talker waits for the packs through one interprocess event per thinker
  for (ArStage* th : thinkers) {
    bool any = false;
    for (ArStage* t : talkers) any = any || t->remote;
    if (!any) continue;
    omni_ipc_event_handle h{};
    dev_ok(omni_ipc_event_create(th->dev, &th->pack_event, &h), "omni_ipc_event_create");
    th->pack_remote = true;
    for (ArStage* t : talkers)
      if (t->remote) t->wait_events.push_back(t->remote->open_event(t->dev, h));
  }
  for (ArStage* t : thinkers) t->dst_arenas = dst.empty() ? std::vector<Arena*>{&I.arena_on(t->dev)} : dst;
  if (want("ar_forward")) I.make_ar("ar_forward", OMNI_MODEL_THINKER, 0);
  for (const char* dn : {"denoise", "dit_image"}) {
    if (!want(dn)) continue;
    const std::vector<int> ddevs = I.devices_of(dn);
    const EngineConfig ec = I.engine_of(dn);
    for (size_t r = 0; r < ddevs.size(); ++r) {
      auto d = std::make_unique<DitStage>();
      d->name = dn;
      d->dev = ddevs[r];
      d->model = model_for(OMNI_MODEL_DIT, I.opt.small_models);
      omni_stage_limits lim{};
      lim.max_resident = static_cast<int32_t>(ec.max_resident_requests);
      lim.dit_max_tokens = 512;
      const uint64_t seed = I.opt.weight_seed + (std::string(dn) == "denoise" ? 2 : 3);
      if ((d->remote = I.worker_for(dn, d->dev)))
        d->remote_id = d->remote->create_stage(d->model, lim, d->dev, seed, &d->remote_weight_bytes);
      else
        dev_ok(omni_stage_create(&d->model, &lim, d->dev, seed, &d->st), "omni_stage_create(dit)");
      I.dit[replica_name(dn, r)] = std::move(d);
    }
  }
  // A DiT sharing its GPU with AR stages leaves them SMs: its iteration is one
  // persistent kernel holding whole SMs (measured, omni3 on one B200: all 148
  // SMs 52 req/s, 100 -> 122, 64 -> 202, 40 -> 194; per-op kernels 198).
  for (auto& [_, d] : I.dit) {
    bool shared = false;
    for (const auto& [__, a] : I.ar) shared = shared || a->dev == d->dev;
    if (d->remote)
      d->remote->set_sm_share(d->remote_id, shared ? kDitSharedSms : 0);
    else
      dev_ok(omni_stage_set_sm_share(d->st, shared ? kDitSharedSms : 0), "omni_stage_set_sm_share");
  }
}

B200Pipeline::~B200Pipeline() = default;

void B200Pipeline::set_capture(bool on) {
  impl_->captured.clear();
  for (auto& [_, s] : impl_->ar) s->capture = on ? &impl_->captured : nullptr;
}
const std::vector<uint16_t>* B200Pipeline::captured_hidden(uint64_t rid) const {
  auto it = impl_->captured.find(rid);
  return it == impl_->captured.end() ? nullptr : &it->second;
}

void B200Pipeline::set_tracer(Tracer* t) {
  impl_->tracer = t;
  for (auto& [_, s] : impl_->ar) s->tracer = t;
  for (auto& [_, s] : impl_->dit) s->tracer = t;
}

// Per forward name, summed over replicas (device busy time, steps); the
// host-gap figure is the mean over the replicas' steps.
std::map<std::string, double> B200Pipeline::device_ms() const {
  std::map<std::string, double> m;
  for (const auto& [_, s] : impl_->ar) m[s->name] += s->dev_ms;
  for (const auto& [_, s] : impl_->dit) m[s->name] += s->dev_ms;
  return m;
}
std::map<std::string, std::pair<double, double>> B200Pipeline::host_ms() const {
  std::map<std::string, std::pair<double, double>> m;
  std::map<std::string, std::pair<double, uint64_t>> gaps;
  auto add = [&](const std::string& n, const HostTimer& h) {
    m[n].first += h.host_ms;
    gaps[n].first += h.gap_ms;
    gaps[n].second += h.gaps;
  };
  for (const auto& [_, s] : impl_->ar) add(s->name, s->ht);
  for (const auto& [_, s] : impl_->dit) add(s->name, s->ht);
  for (auto& [n, v] : m) v.second = gaps[n].second ? gaps[n].first / gaps[n].second : 0.0;
  return m;
}
std::map<std::string, uint64_t> B200Pipeline::step_counts() const {
  std::map<std::string, uint64_t> m;
  for (const auto& [_, s] : impl_->ar) m[s->name] += s->steps;
  for (const auto& [_, s] : impl_->dit) m[s->name] += s->steps;
  return m;
}
uint64_t B200Pipeline::weight_bytes() const {
  uint64_t t = 0, b = 0;
  for (const auto& [_, s] : impl_->ar)
    if (s->remote) t += s->remote_weight_bytes;
    else if (omni_stage_weight_bytes(s->st, &b) == OMNI_OK) t += b;
  for (const auto& [_, s] : impl_->dit)
    if (s->remote) t += s->remote_weight_bytes;
    else if (omni_stage_weight_bytes(s->st, &b) == OMNI_OK) t += b;
  return t;
}
void B200Pipeline::reset_counters() {
  for (auto& [_, s] : impl_->ar) s->dev_ms = 0, s->steps = 0, s->ht.reset();
  for (auto& [_, s] : impl_->dit) s->dev_ms = 0, s->steps = 0, s->ht.reset();
}

void B200Pipeline::register_into(FunctionRegistry& reg) {
  auto& I = *impl_;
  auto trace_prefill = [&I](const std::string& name) {
    return [&I, name](RequestContext&, SeqState& s, std::span<const uint8_t> span) {
      if (I.tracer)
        I.tracer->out += "P " + name + " " + std::to_string(I.tracer->now()) + " " + std::to_string(s.request_id) +
                         " " + std::to_string(s.consumed_prompt) + " " + std::to_string(span.size()) + "\n";
      if (name != "talker_forward")  // thinker: lengths from the host fold (reference_pipeline.hpp:98-100)
        for (uint8_t t : span) s.rng_state = mix(s.rng_state, t);
    };
  };
  auto trace_consumed = [&I](const std::string& name, bool talker) {
    return [&I, name, talker](RequestContext&, SeqState& s) {
      s.target_len = talker ? 4 * s.prompt.size() : (s.rng_state % 64u) + 1u;
      if (I.tracer)
        I.tracer->out += "O " + name + " " + std::to_string(I.tracer->now()) + " " + std::to_string(s.request_id) +
                         " " + std::to_string(s.target_len) + "\n";
    };
  };
  for (auto& [key, sp] : I.ar) {
    ArStage* s = sp.get();
    StageModel m;
    m.prefill = trace_prefill(s->name);
    m.on_prompt_consumed = trace_consumed(s->name, s->kind == OMNI_MODEL_TALKER);
    if (!s->remote) m.reserve = [s](const BatchSlot& b) {
      if (s->kind == OMNI_MODEL_THINKER && b.phase == Phase::PREFILL && b.seq) {
        // prompt ids of the span: the prefix cache maps cached pages first
        std::vector<int32_t> ids(b.seq->prompt.begin() + b.pos0, b.seq->prompt.begin() + b.pos0 + b.span);
        dev_ok(omni_seq_reserve_prompt(s->st, b.request_id, static_cast<int32_t>(b.pos0),
                                       static_cast<int32_t>(b.span), ids.data()),
               "omni_seq_reserve_prompt");
        return;
      }
      dev_ok(omni_seq_reserve(s->st, b.request_id, static_cast<int32_t>(b.pos0 + b.span)), "omni_seq_reserve");
    };
    m.pack_chunk = [s](const SeqState& q, size_t b, size_t e) { return s->pack_chunk(q, b, e); };
    m.launch_batch = [s](std::vector<BatchSlot>& slots) { s->launch(slots); };
    m.batch_ready = [s] { return s->ready(); };
    m.collect_batch = [s](std::vector<BatchSlot>& slots, std::vector<int32_t>& out) { s->collect(slots, out); };
    m.release = [s](uint64_t rid) {
      if (s->remote) s->remote->release(s->remote_id, rid);
      else dev_ok(omni_seq_release(s->st, rid), "omni_seq_release");
    };
    m.flush = [s] { s->flush(); };
    m.cleanup = [s](uint64_t rid) {
      for (Arena* a : s->dst_arenas) a->release(rid);  // idempotent; arenas may be shared
    };
    reg.register_forward(key, std::move(m));
  }

  // Talker preprocess over device chunks: same READY/STALL rule as the
  // reference (reference_pipeline.hpp:159-190); rows stay in HBM, the host
  // keeps only token ids and row addresses.
  reg.register_preprocess("process_input", [](RequestContext&, SeqState& s, StreamReceiver* up) {
    if (up) {
      while (auto c = up->try_recv()) {
        const Payload& p = c->payload;
        if (p.is_device() && p.shape.size() == 2) {
          for (uint32_t r = 0; r < p.shape[0]; ++r) {
            s.prompt.push_back(static_cast<uint8_t>(p.host_tokens.at(r)));
            s.prompt_rows.push_back(p.device_elem(r, 1));
          }
        } else if (p.element_count() > 0 || p.shape.size() == 2) {
          if (!(p.shape.size() == 2 && p.shape[0] == 0)) throw BadDtype("talker expects device FIX16 rows");
        }
        if (c->eos) s.prompt_complete = true;
      }
    }
    if (s.phase == Phase::PREFILL) {
      if (s.consumed_prompt < s.prompt.size()) return PreprocessStatus::READY;
      return s.prompt_complete ? PreprocessStatus::READY : PreprocessStatus::STALL;
    }
    if (s.phase == Phase::DECODE)
      return s.emitted.size() / 4 < s.prompt_rows.size() ? PreprocessStatus::READY : PreprocessStatus::STALL;
    return PreprocessStatus::READY;
  });

  reg.register_transfer("Thinker2Talker", [](TransferEnv& env) {
    ArSubmission sub;
    sub.request_id = env.request.request_id;
    sub.seed = env.request.seed;
    if (env.upstream_final) {
      const Payload& p = *env.upstream_final;
      if (!p.is_device() || p.shape.size() != 2) throw TransferFnError("Thinker2Talker: unexpected payload");
      for (uint32_t r = 0; r < p.shape[0]; ++r) {
        sub.prompt.push_back(static_cast<uint8_t>(p.host_tokens.at(r)));
        sub.prompt_rows.push_back(p.device_elem(r, 1));
      }
      sub.prompt_streams = false;
    } else {
      sub.prompt_streams = true;
    }
    env.submit_ar(std::move(sub));
  });
  reg.register_transfer("Talker2Vocoder", [](TransferEnv& env) { env.wire_diffusion({4, 16}); });
  // branching graphs (BASELINE config 5): Thinker text ids -> image DiT
  reg.register_transfer("Thinker2Image", [](TransferEnv& env) { env.wire_diffusion({4, 16}); });

  for (auto& [key, dp] : I.dit) {
    DitStage* d = dp.get();
    DiffusionModel dm;
    dm.launch_batch = [d](const std::vector<DiffusionJob>& jobs) { d->launch(jobs); };
    dm.batch_ready = [d] { return d->ready(); };
    dm.collect_batch = [d] { return d->collect(); };
    reg.register_denoiser(key, std::move(dm));
  }
}

}  // namespace omni
