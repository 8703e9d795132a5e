// Stage worker processes: remote omni_stage execution over control frames
// (see omni/stage_worker.hpp).
#include "omni/stage_worker.hpp"

#include <cstring>

namespace omni {

namespace {

constexpr uint64_t kTimeoutMs = 600000;

struct W {  // little-endian body writer
  std::vector<uint8_t> b;
  W& u32(uint32_t v) {
    wire::put_u32(b, v);
    return *this;
  }
  W& u64(uint64_t v) {
    wire::put_u64(b, v);
    return *this;
  }
  W& i32(int32_t v) { return u32(static_cast<uint32_t>(v)); }
  W& f32(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    return u32(u);
  }
  W& raw(const void* p, size_t n) {
    const auto* c = static_cast<const uint8_t*>(p);
    b.insert(b.end(), c, c + n);
    return *this;
  }
  W& str(const std::string& s) {
    wire::put_str(b, s);
    return *this;
  }
  template <class T>
  W& arr32(const T* p, size_t n) {  // int32 / float arrays
    for (size_t i = 0; i < n; ++i) {
      uint32_t u;
      std::memcpy(&u, p + i, 4);
      u32(u);
    }
    return *this;
  }
  W& arr64(const uint64_t* p, size_t n) {
    for (size_t i = 0; i < n; ++i) u64(p[i]);
    return *this;
  }
};

struct R {  // body reader
  wire::Reader r;
  explicit R(const std::vector<uint8_t>& v) : r{std::span<const uint8_t>(v.data(), v.size())} {}
  uint32_t u32() { return r.u32(); }
  uint64_t u64() { return r.u64(); }
  int32_t i32() { return static_cast<int32_t>(r.u32()); }
  float f32() {
    const uint32_t u = r.u32();
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  }
  void raw(void* p, size_t n) {
    const auto v = r.raw(n);
    std::memcpy(p, v.data(), n);
  }
  std::string str() { return r.str(); }
  std::vector<int32_t> i32s(size_t n) {
    std::vector<int32_t> v(n);
    for (auto& x : v) x = i32();
    return v;
  }
  std::vector<float> f32s(size_t n) {
    std::vector<float> v(n);
    for (auto& x : v) x = f32();
    return v;
  }
  std::vector<uint64_t> u64s(size_t n) {
    std::vector<uint64_t> v(n);
    for (auto& x : v) x = u64();
    return v;
  }
};

ControlMessage frame(ControlMessage::Kind k, const std::string& op, uint64_t id, std::vector<uint8_t> body) {
  ControlMessage m;
  m.kind = k;
  m.key = op;
  m.request_id = id;
  m.locator.kind = Locator::Kind::INLINE;
  m.locator.inline_bytes = std::move(body);
  return m;
}

}  // namespace

// ---- worker side -------------------------------------------------------------

void run_stage_worker(IpcChannel& ch) {
  std::map<uint64_t, omni_stage*> stages;
  std::map<uint64_t, omni_arena*> arenas;
  std::map<uint64_t, omni_ipc_event*> events;
  uint64_t next = 1;
  auto reply = [&](const std::string& op, uint64_t id, W w) {
    ch.send(frame(ControlMessage::Kind::ACK, op, id, std::move(w.b)));
  };
  auto stage_of = [&](uint64_t id) {
    auto it = stages.find(id);
    if (it == stages.end()) throw ProtocolViolation("unknown remote stage " + std::to_string(id));
    return it->second;
  };
  for (;;) {
    ControlMessage m;
    try {
      m = ch.recv(365ull * 24 * 3600 * 1000);
    } catch (const TransportDown&) {
      break;  // orchestrator went away
    }
    if (m.kind != ControlMessage::Kind::PUT_NOTICE || m.locator.kind != Locator::Kind::INLINE)
      throw ProtocolViolation("worker: expected a request frame");
    R in(m.locator.inline_bytes);
    const std::string& op = m.key;
    if (op == "shutdown") break;
    if (op == "create") {
      omni_model_desc md{};
      omni_stage_limits lim{};
      in.raw(&md, sizeof md);
      in.raw(&lim, sizeof lim);
      const int32_t dev = in.i32();
      const uint64_t seed = in.u64();
      omni_stage* st = nullptr;
      W w;
      if (omni_stage_create(&md, &lim, dev, seed, &st) != OMNI_OK) {
        w.u64(0).u64(0).str(omni_last_error());
      } else {
        uint64_t wb = 0;
        omni_stage_weight_bytes(st, &wb);
        stages[next] = st;
        w.u64(next++).u64(wb).str("");
      }
      reply(op, m.request_id, std::move(w));
    } else if (op == "destroy") {
      if (auto it = stages.find(m.request_id); it != stages.end()) {
        omni_stage_destroy(it->second);
        stages.erase(it);
      }
    } else if (op == "sm_share") {
      const omni_status s = omni_stage_set_sm_share(stage_of(m.request_id), in.i32());
      W w;
      w.i32(s).str(s == OMNI_OK ? "" : omni_last_error());
      reply(op, m.request_id, std::move(w));
    } else if (op == "arena") {
      const int32_t dev = in.i32();
      const uint64_t bytes = in.u64();
      omni_arena* a = nullptr;
      omni_ipc_handle h{};
      uint64_t base = 0;
      W w;
      if (omni_arena_create(dev, bytes, &a) != OMNI_OK || omni_arena_export(a, &h) != OMNI_OK ||
          omni_arena_base(a, &base, nullptr) != OMNI_OK) {
        w.u64(0).raw(&h, sizeof h).u64(0).str(omni_last_error());
      } else {
        arenas[next] = a;
        w.u64(next++).raw(&h, sizeof h).u64(base).str("");
      }
      reply(op, m.request_id, std::move(w));
    } else if (op == "event") {
      const int32_t dev = in.i32();
      omni_ipc_event_handle h{};
      in.raw(&h, sizeof h);
      omni_ipc_event* e = nullptr;
      W w;
      if (omni_ipc_event_open(dev, &h, &e) != OMNI_OK) {
        w.u64(0).str(omni_last_error());
      } else {
        events[next] = e;
        w.u64(next++).str("");
      }
      reply(op, m.request_id, std::move(w));
    } else if (op == "ar_step") {
      omni_stage* st = stage_of(m.request_id);
      const auto ev = in.u64s(in.u32());
      const uint32_t n = in.u32();
      const auto seq = in.u64s(n);
      const auto phase = in.i32s(n), span = in.i32s(n), pos0 = in.i32s(n), outi = in.i32s(n);
      const uint32_t nt = in.u32();
      const auto tokens = in.i32s(nt);
      const bool cond = in.r.u8() != 0;
      std::vector<uint64_t> cs;
      std::vector<int32_t> cr;
      if (cond) {
        cs = in.u64s(nt);
        cr = in.i32s(nt);
      }
      omni_ar_batch b{static_cast<int32_t>(n), seq.data(), phase.data(), span.data(), pos0.data(), outi.data(),
                      tokens.data(), cond ? cs.data() : nullptr, cond ? cr.data() : nullptr};
      std::vector<int32_t> tok(n, -1);
      std::vector<float> mg(n, 0.f);
      omni_status s = OMNI_OK;
      for (uint64_t e : ev) {  // the producer's packs that wrote this step's rows
        auto it = events.find(e);
        if (it == events.end()) throw ProtocolViolation("unknown remote event");
        if (s == OMNI_OK) s = omni_stage_wait_event(st, it->second);
      }
      if (s == OMNI_OK) s = omni_ar_step(st, &b, tok.data(), mg.data());
      if (s == OMNI_OK) s = omni_stage_wait(st);
      float us = 0.f;
      omni_stage_last_step_us(st, &us);
      W w;
      w.i32(s).str(s == OMNI_OK ? "" : omni_last_error()).u32(n).arr32(tok.data(), n).u32(n).arr32(mg.data(), n);
      w.f32(us);
      reply(op, m.request_id, std::move(w));
    } else if (op == "dit_step") {
      omni_stage* st = stage_of(m.request_id);
      const uint32_t nj = in.u32();
      const auto rid = in.u64s(nj);
      const auto off = in.i32s(nj), ntok = in.i32s(nj);
      const uint32_t nt = in.u32();
      const auto tokens = in.i32s(nt);
      const uint32_t samples_per = in.u32();
      std::vector<int32_t> samples(static_cast<size_t>(nt) * samples_per, 0);
      omni_dit_batch b{static_cast<int32_t>(nj), rid.data(), off.data(), ntok.data(), tokens.data()};
      omni_status s = omni_dit_step(st, &b, samples.data());
      if (s == OMNI_OK) s = omni_stage_wait(st);
      float us = 0.f;
      omni_stage_last_step_us(st, &us);
      W w;
      w.i32(s).str(s == OMNI_OK ? "" : omni_last_error()).u32(static_cast<uint32_t>(samples.size()));
      w.arr32(samples.data(), samples.size()).u32(0).f32(us);
      reply(op, m.request_id, std::move(w));
    } else if (op == "release") {
      omni_seq_release(stage_of(m.request_id), in.u64());
    } else {
      throw ProtocolViolation("worker: unknown operation " + op);
    }
  }
  for (auto& [_, st] : stages) omni_stage_destroy(st);
  for (auto& [_, e] : events) omni_ipc_event_destroy(e);
  for (auto& [_, a] : arenas) omni_arena_destroy(a);
}

// ---- orchestrator side ---------------------------------------------------------

WorkerClient::~WorkerClient() {
  try {
    send("shutdown", 0, {});
  } catch (...) {
  }
}

void WorkerClient::send(const std::string& op, uint64_t id, std::vector<uint8_t> body) {
  ch_.send(frame(ControlMessage::Kind::PUT_NOTICE, op, id, std::move(body)));
}

void WorkerClient::pump(bool block) {
  for (;;) {
    std::optional<ControlMessage> m = block ? std::optional<ControlMessage>(ch_.recv(kTimeoutMs)) : ch_.try_recv();
    if (!m) return;
    if (m->kind != ControlMessage::Kind::ACK) throw ProtocolViolation("worker sent a non-reply frame");
    if (m->key == "ar_step" || m->key == "dit_step") {
      R in(m->locator.inline_bytes);
      StepReply r;
      r.status = in.i32();
      r.error = in.str();
      r.tokens = in.i32s(in.u32());
      r.margins = in.f32s(in.u32());
      r.step_us = in.f32();
      done_[m->request_id] = std::move(r);
    } else {
      sync_.push_back(std::move(*m));
    }
    if (block) return;
  }
}

ControlMessage WorkerClient::call(const std::string& op, uint64_t id, std::vector<uint8_t> body) {
  send(op, id, std::move(body));
  for (;;) {
    for (auto it = sync_.begin(); it != sync_.end(); ++it)
      if (it->key == op && it->request_id == id) {
        ControlMessage m = std::move(*it);
        sync_.erase(it);
        return m;
      }
    pump(true);
  }
}

uint64_t WorkerClient::create_stage(const omni_model_desc& m, const omni_stage_limits& lim, int dev, uint64_t seed,
                                    uint64_t* weight_bytes) {
  W w;
  w.raw(&m, sizeof m).raw(&lim, sizeof lim).i32(dev).u64(seed);
  const ControlMessage r = call("create", 0, std::move(w.b));
  R in(r.locator.inline_bytes);
  const uint64_t id = in.u64(), wb = in.u64();
  const std::string err = in.str();
  if (!id) throw DeviceError("remote omni_stage_create: " + err);
  if (weight_bytes) *weight_bytes = wb;
  return id;
}

void WorkerClient::destroy_stage(uint64_t stage) { send("destroy", stage, {}); }

void WorkerClient::set_sm_share(uint64_t stage, int sms) {
  W w;
  w.i32(sms);
  const ControlMessage r = call("sm_share", stage, std::move(w.b));
  R in(r.locator.inline_bytes);
  if (in.i32() != OMNI_OK) throw DeviceError("remote omni_stage_set_sm_share: " + in.str());
}

uint64_t WorkerClient::create_arena(int dev, uint64_t bytes, omni_ipc_handle* h, uint64_t* remote_base) {
  W w;
  w.i32(dev).u64(bytes);
  const ControlMessage r = call("arena", 0, std::move(w.b));
  R in(r.locator.inline_bytes);
  const uint64_t id = in.u64();
  in.raw(h, sizeof *h);
  *remote_base = in.u64();
  const std::string err = in.str();
  if (!id) throw DeviceError("remote omni_arena_create: " + err);
  return id;
}

uint64_t WorkerClient::open_event(int dev, const omni_ipc_event_handle& h) {
  W w;
  w.i32(dev).raw(&h, sizeof h);
  const ControlMessage r = call("event", 0, std::move(w.b));
  R in(r.locator.inline_bytes);
  const uint64_t id = in.u64();
  if (!id) throw DeviceError("remote omni_ipc_event_open: " + in.str());
  return id;
}

void WorkerClient::ar_step(uint64_t stage, const std::vector<uint64_t>& events, const omni_ar_batch& b,
                           int n_tokens) {
  const size_t n = static_cast<size_t>(b.n_entries), nt = static_cast<size_t>(n_tokens);
  W w;
  w.u32(static_cast<uint32_t>(events.size())).arr64(events.data(), events.size());
  w.u32(static_cast<uint32_t>(n)).arr64(b.seq_id, n).arr32(b.phase, n).arr32(b.span, n).arr32(b.pos0, n);
  w.arr32(b.out_index, n).u32(static_cast<uint32_t>(nt)).arr32(b.tokens, nt);
  w.b.push_back(b.cond_src ? 1 : 0);
  if (b.cond_src) w.arr64(b.cond_src, nt).arr32(b.cond_row, nt);
  done_.erase(stage);
  send("ar_step", stage, std::move(w.b));
}

void WorkerClient::dit_step(uint64_t stage, const omni_dit_batch& b) {
  const size_t nj = static_cast<size_t>(b.n_jobs);
  size_t nt = 0;
  for (size_t j = 0; j < nj; ++j) nt += static_cast<size_t>(b.n_tokens[j]);
  W w;
  w.u32(static_cast<uint32_t>(nj)).arr64(b.request_id, nj).arr32(b.token_offset, nj).arr32(b.n_tokens, nj);
  w.u32(static_cast<uint32_t>(nt)).arr32(b.tokens, nt).u32(16);
  done_.erase(stage);
  send("dit_step", stage, std::move(w.b));
}

void WorkerClient::release(uint64_t stage, uint64_t rid) {
  W w;
  w.u64(rid);
  send("release", stage, std::move(w.b));
}

std::optional<WorkerClient::StepReply> WorkerClient::poll(uint64_t stage) {
  pump(false);
  auto it = done_.find(stage);
  if (it == done_.end()) return std::nullopt;
  StepReply r = std::move(it->second);
  done_.erase(it);
  return r;
}

WorkerClient::StepReply WorkerClient::wait(uint64_t stage) {
  for (;;) {
    if (auto r = poll(stage)) return std::move(*r);
    pump(true);
  }
}

}  // namespace omni
