// ORACLE / TEST INFRASTRUCTURE — never linked into the product.
//
// The reference's integer mock pipeline (reference_pipeline.hpp:20-247 and
// the closed-form denoiser diffusion_engine.hpp:28-43), restated as plugins
// for the B200 build's C++ control plane (libomni_serve), plus a trace driver
// that prints the exact line format of oracle/ref_harness.cpp. Running the
// same workload through both and diffing the traces proves that routing,
// batch membership, chunk cuts, payload bytes and per-request metrics of the
// new control plane are bit-identical to the reference.
#include <cstdio>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>

#include "omni/bench.hpp"
#include "omni/config.hpp"
#include "omni/orchestrator.hpp"
#include "omni/http_service.hpp"

using namespace omni;

namespace {

uint32_t mix(uint32_t h, uint32_t t) { return h * 1000003u + t + 1u; }
uint32_t target_length(uint32_t h) { return (h % 64u) + 1u; }
int32_t token_of(uint32_t h) { return static_cast<int32_t>(h % 255u) + 1; }
HiddenState hidden_of(uint32_t h) {
  HiddenState s;
  for (int k = 0; k < 8; ++k) s.values[k] = (h >> (4 * k)) & 0xF;
  return s;
}
int32_t codec_token(int32_t t, int sum, int i) { return (t * 7 + sum + i) % 64; }
std::string hid_key(size_t j) { return "hid/" + std::to_string(j); }

Payload denoise_closed_form(const DiffusionJob& job) {
  if (job.input.dtype != Dtype::I32) throw BadDtype("diffusion input must be I32 codec tokens");
  if (job.steps < 1) throw OmniError("steps must be >= 1");
  std::vector<int32_t> out;
  for (int32_t c : job.input.as_i32())
    for (uint32_t s = 0; s < job.samples_per_token; ++s) {
      int64_t v = (static_cast<int64_t>(c) * (s + 1)) % 128;
      if (v < 0) v += 128;
      out.push_back(static_cast<int32_t>(v - 64));
    }
  return Payload::from_i32(out);
}

StageModel thinker() {
  StageModel m;
  m.prefill = [](RequestContext&, SeqState& s, std::span<const uint8_t> span) {
    for (uint8_t t : span) s.rng_state = mix(s.rng_state, t);
  };
  m.on_prompt_consumed = [](RequestContext&, SeqState& s) { s.target_len = target_length(s.rng_state); };
  m.decode = [](RequestContext&, SeqState& s) {
    s.rng_state = mix(s.rng_state, static_cast<uint32_t>(s.emitted.size()));
    DecodeStep d;
    d.token = token_of(s.rng_state);
    d.hidden = hidden_of(s.rng_state);
    d.has_hidden = true;
    return d;
  };
  m.pack_chunk = [](const SeqState& s, size_t b, size_t e) {
    Payload p;
    p.dtype = Dtype::U8;
    p.shape = {static_cast<uint32_t>(e - b), 9};
    for (size_t i = b; i < e; ++i) {
      p.bytes.push_back(static_cast<uint8_t>(s.emitted[i]));
      for (int k = 0; k < 8; ++k) p.bytes.push_back(s.hidden[i].values[k]);
    }
    return p;
  };
  return m;
}

StageModel talker() {
  StageModel m;
  m.prefill = [](RequestContext&, SeqState&, std::span<const uint8_t>) {};
  m.on_prompt_consumed = [](RequestContext&, SeqState& s) { s.target_len = 4 * s.prompt.size(); };
  m.decode = [](RequestContext& ctx, SeqState& s) {
    const size_t mi = s.emitted.size();
    const Payload& row = ctx.get(hid_key(mi / 4));
    if (row.bytes.size() != 9) throw ForwardError("bad hidden row");
    const int32_t t = row.bytes[0];
    if (t < 1) throw ForwardError("text token below alphabet floor");
    int sum = 0;
    for (int k = 0; k < 8; ++k) sum += row.bytes[1 + k];
    DecodeStep d;
    d.token = codec_token(t, sum, static_cast<int>(mi % 4));
    return d;
  };
  m.pack_chunk = [](const SeqState& s, size_t b, size_t e) {
    return Payload::from_i32(std::span<const int32_t>(s.emitted.data() + b, e - b));
  };
  return m;
}

void register_mock(FunctionRegistry& reg) {
  reg.register_forward("thinker_forward", thinker());
  reg.register_forward("talker_forward", talker());
  StageModel ar = thinker();
  ar.pack_chunk = [](const SeqState& s, size_t b, size_t e) {
    return Payload::from_i32(std::span<const int32_t>(s.emitted.data() + b, e - b));
  };
  reg.register_forward("ar_forward", ar);
  reg.register_preprocess("process_input", [](RequestContext& ctx, SeqState& s, StreamReceiver* up) {
    if (up) {
      while (auto c = up->try_recv()) {
        if (c->payload.shape.size() == 2 && c->payload.shape[1] == 9) {
          for (size_t r = 0; r < c->payload.shape[0]; ++r) {
            std::vector<uint8_t> row(c->payload.bytes.begin() + r * 9, c->payload.bytes.begin() + (r + 1) * 9);
            const uint8_t tok = row[0];
            ctx.put(hid_key(s.prompt.size()), Payload::from_u8(std::move(row)));
            s.prompt.push_back(tok);
          }
        }
        if (c->eos) s.prompt_complete = true;
      }
    }
    if (s.phase == Phase::PREFILL) {
      if (s.consumed_prompt < s.prompt.size()) return PreprocessStatus::READY;
      return s.prompt_complete ? PreprocessStatus::READY : PreprocessStatus::STALL;
    }
    if (s.phase == Phase::DECODE)
      return ctx.has(hid_key(s.emitted.size() / 4)) ? PreprocessStatus::READY : PreprocessStatus::STALL;
    return PreprocessStatus::READY;
  });
  reg.register_transfer("Thinker2Talker", [](TransferEnv& env) {
    ArSubmission sub;
    sub.request_id = env.request.request_id;
    sub.seed = env.request.seed;
    if (env.upstream_final) {
      const Payload& p = *env.upstream_final;
      if (p.shape.size() != 2 || p.shape[1] != 9) throw TransferFnError("Thinker2Talker: unexpected payload shape");
      for (size_t j = 0; j < p.shape[0]; ++j) {
        std::vector<uint8_t> row(p.bytes.begin() + j * 9, p.bytes.begin() + (j + 1) * 9);
        sub.prompt.push_back(row[0]);
        env.ctx.put(hid_key(j), Payload::from_u8(std::move(row)));
      }
    } else {
      sub.prompt_streams = true;
    }
    env.submit_ar(std::move(sub));
  });
  reg.register_transfer("Talker2Vocoder", [](TransferEnv& env) { env.wire_diffusion({4, 16}); });
  DiffusionModel dm;
  dm.denoise = denoise_closed_form;
  reg.register_denoiser("denoise", dm);
}

std::string hex64(uint64_t v) {
  char b[32];
  std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(v));
  return b;
}
uint64_t fnv_i32s(const std::vector<int32_t>& v, uint64_t h) {
  for (int32_t x : v) {
    uint8_t b[4];
    for (int i = 0; i < 4; ++i) b[i] = uint8_t(uint32_t(x) >> (8 * i));
    h = fnv1a64(std::span<const uint8_t>(b, 4), h);
  }
  return h;
}

struct Tr {
  const Clock* clock = nullptr;
  std::ostringstream out;
  StageModel wrap(const std::string& name, StageModel m) {
    StageModel w = m;
    w.prefill = [this, name, in = m.prefill](RequestContext& c, SeqState& s, std::span<const uint8_t> sp) {
      out << "P " << name << " " << clock->now_us() << " " << s.request_id << " " << s.consumed_prompt << " "
          << sp.size() << "\n";
      if (in) in(c, s, sp);
    };
    w.on_prompt_consumed = [this, name, in = m.on_prompt_consumed](RequestContext& c, SeqState& s) {
      in(c, s);
      out << "O " << name << " " << clock->now_us() << " " << s.request_id << " " << s.target_len << "\n";
    };
    w.decode = [this, name, in = m.decode](RequestContext& c, SeqState& s) {
      DecodeStep d = in(c, s);
      out << "D " << name << " " << clock->now_us() << " " << s.request_id << " " << s.emitted.size() << " "
          << d.token << "\n";
      return d;
    };
    w.pack_chunk = [this, name, in = m.pack_chunk](const SeqState& s, size_t b, size_t e) {
      Payload p = in(s, b, e);
      auto blob = encode_payload(p);
      out << "K " << name << " " << clock->now_us() << " " << s.request_id << " " << b << " " << e << " "
          << int(p.dtype);
      for (auto d : p.shape) out << " " << d;
      out << " " << hex64(fnv1a64(blob)) << "\n";
      return p;
    };
    return w;
  }
};

}  // namespace

// live HTTP serving over the mock hooks (tests/test_http_service.py)
struct MockServer {
  FunctionRegistry reg;
  std::unique_ptr<Orchestrator> orch;
  std::unique_ptr<HttpService> http;
};
MockServer* g_server = nullptr;

extern "C" {

// Starts the control plane (wall clock) + HTTP front end over the reference's
// mock hooks. Returns the bound port, or -1 (message in `err`).
int oracle_mock_serve_start(const char* config_json, const char* listen, char* err, size_t cap) {
  try {
    if (g_server) throw std::runtime_error("already serving");
    auto s = std::make_unique<MockServer>();
    DeploymentPlan plan = parse_plan_text(config_json);
    plan.clock_kind = "wall";
    register_mock(s->reg);
    s->orch = std::make_unique<Orchestrator>(plan, &s->reg);
    s->orch->start();
    s->orch->serve_async();
    s->http = std::make_unique<HttpService>(*s->orch);
    s->http->start(listen);
    const int port = s->http->port();
    g_server = s.release();
    return port;
  } catch (const std::exception& e) {
    std::snprintf(err, cap, "%s", e.what());
    return -1;
  }
}

void oracle_mock_serve_stop() {
  if (!g_server) return;
  g_server->http->stop();
  g_server->orch->shutdown(true);
  delete g_server;
  g_server = nullptr;
}

// Runs the workload through the new control plane with the mock hooks on a
// virtual clock and writes the trace (same format as ref_harness). Returns the
// trace length, or -1 on error (message in `out`).
long oracle_mock_trace(const char* config_json, uint64_t n, uint64_t seed, uint64_t conc, int stream,
                       int chunk0, int chunk1, char* out, size_t cap) {
  std::string text;
  try {
    DeploymentPlan plan = parse_plan_text(config_json);
    plan.clock_kind = "virtual";
    if (chunk0 > 0) plan.graph.edges.at(0).streaming_chunk_size = chunk0;
    if (chunk1 > 0 && plan.graph.edges.size() > 1) plan.graph.edges.at(1).streaming_chunk_size = chunk1;
    bench::WorkloadSpec spec;
    spec.n = n;
    spec.seed = seed;
    spec.stream = stream != 0;
    auto wl = bench::gen_workload(spec);
    plan.server.admission_cap = wl.size() + 1;
    Tr tr;
    FunctionRegistry base, reg;
    register_mock(base);
    register_mock(reg);
    for (const char* f : {"thinker_forward", "talker_forward", "ar_forward"})
      reg.register_forward(f, tr.wrap(f, base.forward(f)));
    // replicated AR stages: one traced model per replica ("name#r" in the
    // trace lines) so tests can see which replica served which request
    for (const auto& nd : plan.graph.nodes) {
      const size_t R = placement_devices(plan, nd.id).size();
      if (nd.kind != StageKind::AR || R < 2) continue;
      for (size_t r = 1; r < R; ++r)
        reg.register_forward(replica_name(nd.forward_ref, r),
                             tr.wrap(replica_name(nd.forward_ref, r), base.forward(nd.forward_ref)));
    }
    Orchestrator orch(plan, &reg);
    tr.clock = &orch.clock();
    orch.start();
    std::vector<std::shared_ptr<ResultHandle>> hs(wl.size());
    size_t next = 0;
    auto launch = [&](uint64_t at) {
      if (next >= wl.size()) return;
      const size_t i = next++;
      hs[i] = orch.submit_at(wl[i], at);
    };
    orch.set_on_done([&](uint64_t, uint64_t now) { launch(now); });
    for (size_t i = 0; i < std::min<size_t>(conc, wl.size()); ++i) launch(0);
    orch.run_until_drained();
    std::ostringstream rs;
    for (size_t i = 0; i < wl.size(); ++i) {
      const auto& o = hs[i]->wait();
      const auto& m = o.metrics;
      uint64_t od = 1469598103934665603ull;
      od = fnv_i32s(o.text_tokens, od);
      od = fnv_i32s(o.codec_tokens, od);
      od = fnv_i32s(o.waveform, od);
      rs << "R " << wl[i].request_id << " " << o.status << " " << m.submitted_at << " " << m.done_at << " "
         << (m.first_final_chunk_at == kTimeUnset ? -1LL : (long long)m.first_final_chunk_at) << " "
         << o.text_tokens.size() << " " << o.codec_tokens.size() << " " << o.waveform.size() << " " << hex64(od);
      for (const auto& [st, t] : m.stages)
        rs << " " << st << ":" << (long long)t.first_scheduled_at << ":" << (long long)t.first_token_at << ":"
           << (long long)t.finished_at << ":" << t.tokens;
      rs << "\n";
    }
    // replicated stages (placement lists several devices): iterations per replica
    for (const auto& nd : plan.graph.nodes) {
      const auto it = orch.replica_iterations(nd.id);
      if (it.size() < 2) continue;
      rs << "I " << nd.id;
      for (uint64_t x : it) rs << " " << x;
      rs << "\n";
    }
    orch.shutdown(true);
    text = tr.out.str() + rs.str();
  } catch (const std::exception& e) {
    std::snprintf(out, cap, "%s", e.what());
    return -1;
  }
  if (out && cap) {
    const size_t k = std::min(cap - 1, text.size());
    std::memcpy(out, text.data(), k);
    out[k] = 0;
  }
  return static_cast<long>(text.size());
}

// CSV v1 of the disaggregated bench on the new control plane with mock hooks
// (compared byte-for-byte with the reference's CSV digest).
long oracle_mock_csv(const char* config_json, uint64_t n, uint64_t seed, uint64_t conc, char* out, size_t cap) {
  std::string csv;
  try {
    DeploymentPlan plan = parse_plan_text(config_json);
    plan.clock_kind = "virtual";
    bench::WorkloadSpec spec;
    spec.n = n;
    spec.seed = seed;
    FunctionRegistry reg;
    register_mock(reg);
    bench::BenchOptions bo;
    bo.concurrency = conc;
    auto rep = bench::run_bench_disaggregated(plan, reg, bench::gen_workload(spec), spec, bo);
    csv = rep.csv;
  } catch (const std::exception& e) {
    std::snprintf(out, cap, "%s", e.what());
    return -1;
  }
  if (out && cap) {
    const size_t k = std::min(cap - 1, csv.size());
    std::memcpy(out, csv.data(), k);
    out[k] = 0;
  }
  return static_cast<long>(csv.size());
}

// FNV digest of gen_workload(n, seed) in the ref_harness layout.
uint64_t oracle_workload_digest(uint64_t n, uint64_t seed) {
  bench::WorkloadSpec spec;
  spec.n = n;
  spec.seed = seed;
  uint64_t h = 1469598103934665603ull;
  for (const auto& r : bench::gen_workload(spec)) {
    uint8_t b[8];
    for (int i = 0; i < 8; ++i) b[i] = uint8_t(r.request_id >> (8 * i));
    h = fnv1a64(std::span<const uint8_t>(b, 8), h);
    h = fnv1a64(r.prompt_tokens, h);
    for (int i = 0; i < 4; ++i) b[i] = uint8_t(r.seed >> (8 * i));
    h = fnv1a64(std::span<const uint8_t>(b, 4), h);
  }
  return h;
}

}  // extern "C"
