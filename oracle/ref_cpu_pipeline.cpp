// ORACLE / TEST INFRASTRUCTURE — the CPU baseline ("reference arm").
//
// The UNMODIFIED reference control plane (/root/reference/proj/include:
// Orchestrator, ArEngine, DiffusionEngine, Connector — compiled from its
// headers, prebuilt into oracle/_ref/) with its StageModel hooks backed by the
// fp32 CPU oracle of the same random-init Thinker / Talker / DiT
// (oracle/models_cpu.c, OpenMP over all host cores). Wall clock with
// step_latency_us = 0 so the cost model charges nothing and the measured time
// is the real CPU compute (SURVEY §8d "CPU baseline", BASELINE.md plan).
//
// The reference has no diffusion hook (denoise() is a built-in free function,
// diffusion_engine.hpp:28-43, called at :98). A better-matching overload
// (non-const DiffusionJob&) declared before the header is included routes
// that call to the CPU DiT; every other line of the reference is untouched.
//
// The reference's StageModel API is per sequence (ar_engine.hpp:308-337), so
// every decode step is one GEMV pass per sequence — "the reference CPU
// pipeline as designed"; the orchestrator runs all stages on one thread.
#include <omp.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "omniserve/payload.hpp"
#include "omniserve/registry.hpp"

extern "C" {
typedef struct {
  int kind, d, L, H, KVH, hd, ff, V, cond_dim, C, S, T;
} om_desc;
void* om_create(const om_desc*, uint64_t seed);
void om_destroy(void*);
void* om_seq_new(const void*, int cap);
void om_seq_free(void*);
int om_ar_feed(const void*, void*, int n, const int* tokens, const int* cond_rows, const uint16_t* hid_rows,
               int is_decode, float* logits_out, uint16_t* hidden_out, float* margin_out);
void om_dit_denoise(const void*, int n, const uint64_t* rid, const int* pos, const int* ids, int32_t* samples,
                    float* latents);
}

namespace omni {
struct DiffusionJob;
template <class J>
Payload denoise(J& job);  // preferred over denoise(const DiffusionJob&) for non-const lvalues
}  // namespace omni

#include "omniserve/bench.hpp"
#include "omniserve/config.hpp"
#include "omniserve/orchestrator.hpp"

using namespace omni;

namespace {

struct Models {
  void* thinker = nullptr;
  void* talker = nullptr;
  void* dit = nullptr;
  om_desc th{}, ta{}, dt{};
  uint32_t vocoder_chunk = 8;
};
Models g;

om_desc desc(int kind, bool small) {
  om_desc d{};
  d.kind = kind;
  d.hd = 128;
  if (kind == 2) {
    d.d = small ? 256 : 1024;
    d.L = small ? 2 : 4;
    d.H = small ? 2 : 8;
    d.KVH = d.H;
    d.ff = small ? 512 : 4096;
    d.V = 256;
    d.C = 64;
    d.S = 16;
    d.T = 4;
  } else {
    d.d = small ? 512 : 2048;
    d.L = kind == 0 ? (small ? 2 : 8) : (small ? 2 : 4);
    d.H = small ? 4 : 16;
    d.KVH = small ? 2 : 4;
    d.ff = small ? 1024 : 8192;
    d.V = kind == 0 ? 256 : 64;
    d.cond_dim = kind == 1 ? d.d : 0;
  }
  return d;
}

uint32_t mix(uint32_t h, uint32_t t) { return h * 1000003u + t + 1u; }

struct SeqBox {
  std::map<uint64_t, void*> seqs;
  void* model;
  int cap;
  void* get(uint64_t rid) {
    auto it = seqs.find(rid);
    if (it != seqs.end()) return it->second;
    return seqs[rid] = om_seq_new(model, cap);
  }
  void drop(uint64_t rid) {
    auto it = seqs.find(rid);
    if (it == seqs.end()) return;
    om_seq_free(it->second);
    seqs.erase(it);
  }
};
SeqBox g_th, g_ta;

std::string hid_key(size_t j) { return "hidrow/" + std::to_string(j); }

void register_cpu(FunctionRegistry& reg) {
  StageModel th;
  th.prefill = [](RequestContext&, SeqState& s, std::span<const uint8_t> span) {
    if (s.consumed_prompt == 0) g_th.drop(s.request_id);  // recompute-preemption replay
    std::vector<int> t(span.begin(), span.end());
    om_ar_feed(g.thinker, g_th.get(s.request_id), (int)t.size(), t.data(), nullptr, nullptr, 0, nullptr, nullptr,
               nullptr);
    for (uint8_t x : span) s.rng_state = mix(s.rng_state, x);
  };
  th.on_prompt_consumed = [](RequestContext&, SeqState& s) { s.target_len = (s.rng_state % 64u) + 1u; };
  th.decode = [](RequestContext& ctx, SeqState& s) {
    const int in = s.emitted.empty() ? -1 : s.emitted.back();
    std::vector<uint16_t> hid(g.th.d);
    std::vector<float> lg(g.th.V);
    float mg = 0;
    DecodeStep d;
    d.token = om_ar_feed(g.thinker, g_th.get(s.request_id), 1, &in, nullptr, nullptr, 1, lg.data(), hid.data(), &mg);
    // keep the full bf16 hidden row for the talker (FIX16 row = [token, h...])
    Payload row;
    row.dtype = Dtype::FIX16;
    row.shape = {static_cast<uint32_t>(g.th.d + 1)};
    row.bytes.resize(2 * (g.th.d + 1));
    row.bytes[0] = static_cast<uint8_t>(d.token);
    std::memcpy(row.bytes.data() + 2, hid.data(), 2 * g.th.d);
    ctx.put("th/" + std::to_string(s.emitted.size()), std::move(row));
    if (s.emitted.size() + 1 == s.target_len) g_th.drop(s.request_id);
    return d;
  };
  th.pack_chunk = [](const SeqState& s, size_t b, size_t e) {
    Payload p;
    p.dtype = Dtype::FIX16;
    p.shape = {static_cast<uint32_t>(e - b), 2};  // (token, emitted index): rows live in the context
    for (size_t i = b; i < e; ++i)
      for (uint32_t v : {static_cast<uint32_t>(s.emitted[i]), static_cast<uint32_t>(i)}) {
        p.bytes.push_back(static_cast<uint8_t>(v));
        p.bytes.push_back(static_cast<uint8_t>(v >> 8));
      }
    return p;
  };
  reg.register_forward("thinker_forward", th);

  StageModel ta;
  ta.prefill = [](RequestContext& ctx, SeqState& s, std::span<const uint8_t> span) {
    if (s.consumed_prompt == 0) g_ta.drop(s.request_id);
    const int n = static_cast<int>(span.size());
    std::vector<int> toks(span.begin(), span.end()), rows(n);
    std::vector<uint16_t> hid(static_cast<size_t>(n) * g.ta.cond_dim);
    for (int i = 0; i < n; ++i) {
      const size_t j = s.consumed_prompt + i;
      rows[i] = static_cast<int>(j);
      const Payload& r = ctx.get(hid_key(j));
      std::memcpy(hid.data() + static_cast<size_t>(i) * g.ta.cond_dim, r.bytes.data() + 2, 2 * g.ta.cond_dim);
    }
    om_ar_feed(g.talker, g_ta.get(s.request_id), n, toks.data(), rows.data(), hid.data(), 0, nullptr, nullptr,
               nullptr);
  };
  ta.on_prompt_consumed = [](RequestContext&, SeqState& s) { s.target_len = 4 * s.prompt.size(); };
  ta.decode = [](RequestContext&, SeqState& s) {
    const int in = s.emitted.empty() ? -1 : s.emitted.back();
    const int row = static_cast<int>(s.emitted.size() / 4);
    std::vector<float> lg(g.ta.V);
    DecodeStep d;
    d.token = om_ar_feed(g.talker, g_ta.get(s.request_id), 1, &in, &row, nullptr, 1, lg.data(), nullptr, nullptr);
    if (s.emitted.size() + 1 == s.target_len) g_ta.drop(s.request_id);
    return d;
  };
  ta.pack_chunk = [](const SeqState& s, size_t b, size_t e) {
    return Payload::from_i32(std::span<const int32_t>(s.emitted.data() + b, e - b));
  };
  reg.register_forward("talker_forward", ta);

  reg.register_preprocess("process_input", [](RequestContext& ctx, SeqState& s, StreamReceiver* up) {
    if (up) {
      while (auto c = up->try_recv()) {
        const Payload& p = c->payload;
        if (p.shape.size() == 2 && p.shape[1] == 2)
          for (uint32_t r = 0; r < p.shape[0]; ++r) {
            const uint32_t idx = p.bytes[4 * r + 2] | (p.bytes[4 * r + 3] << 8);
            ctx.put(hid_key(s.prompt.size()), ctx.get("th/" + std::to_string(idx)));
            s.prompt.push_back(p.bytes[4 * r]);
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
    sub.prompt_streams = !env.upstream_final.has_value();
    if (env.upstream_final) {
      const Payload& p = *env.upstream_final;
      for (uint32_t r = 0; r < p.shape[0]; ++r) {
        const uint32_t idx = p.bytes[4 * r + 2] | (p.bytes[4 * r + 3] << 8);
        env.ctx.put(hid_key(r), env.ctx.get("th/" + std::to_string(idx)));
        sub.prompt.push_back(p.bytes[4 * r]);
      }
    }
    env.submit_ar(std::move(sub));
  });
  reg.register_transfer("Talker2Vocoder", [](TransferEnv& env) { env.wire_diffusion({4, 16}); });
}

}  // namespace

namespace omni {
template <class J>
Payload denoise(J& job) {
  const auto codec = job.input.as_i32();
  std::vector<int32_t> out(codec.size() * 16);
  if (!codec.empty()) {
    std::vector<uint64_t> rid(codec.size(), job.request_id);
    std::vector<int> pos(codec.size()), ids(codec.begin(), codec.end());
    for (size_t i = 0; i < codec.size(); ++i) pos[i] = static_cast<int>(job.chunk_seq * g.vocoder_chunk + i);
    om_dit_denoise(g.dit, static_cast<int>(codec.size()), rid.data(), pos.data(), ids.data(), out.data(), nullptr);
  }
  return Payload::from_i32(out);
}
}  // namespace omni

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "ref_cpu_pipeline <config.json> <n> <seed> <conc> <small 0|1> [weight_seed]\n");
    return 2;
  }
  try {
    auto plan = load_plan(argv[1]);
    const uint64_t n = std::stoull(argv[2]), seed = std::stoull(argv[3]), conc = std::stoull(argv[4]);
    const bool small = std::stoi(argv[5]) != 0;
    const uint64_t wseed = argc > 6 ? std::stoull(argv[6]) : 1234;
    plan.clock_kind = "wall";
    plan.server_id = "cpu_baseline";
    for (auto& [_, e] : plan.engines) e.step_latency_us = 0;  // real compute only
    if (plan.graph.edges.size() > 1) g.vocoder_chunk = plan.graph.edges[1].streaming_chunk_size;
    g.th = desc(0, small);
    g.ta = desc(1, small);
    g.dt = desc(2, small);
    auto t_load = std::chrono::steady_clock::now();
    g.thinker = om_create(&g.th, wseed + 0);
    g.talker = om_create(&g.ta, wseed + 1);
    g.dit = om_create(&g.dt, wseed + 2);
    g_th.model = g.thinker;
    g_th.cap = 512 + 64;
    g_ta.model = g.talker;
    g_ta.cap = 64 + 256 + 16;
    const double load_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_load).count();
    FunctionRegistry reg;
    register_cpu(reg);
    bench::WorkloadSpec spec;
    spec.n = n;
    spec.seed = seed;
    auto wl = bench::gen_workload(spec);
    plan.server.admission_cap = wl.size() + 1;
    Orchestrator orch(plan, &reg);
    orch.start();
    std::vector<std::shared_ptr<ResultHandle>> hs(wl.size());
    size_t next = 0;
    auto launch = [&](uint64_t at) {
      if (next >= wl.size()) return;
      const size_t i = next++;
      hs[i] = orch.submit_at(wl[i], at);
    };
    orch.set_on_done([&](uint64_t, uint64_t now) { launch(now); });
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t c0 = orch.clock().now_us();
    for (size_t i = 0; i < std::min<size_t>(conc, wl.size()); ++i) launch(c0);
    orch.run_until_drained();
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<double> jct;
    uint64_t done = 0, text = 0, codec = 0, wave = 0;
    for (auto& h : hs) {
      const auto& o = h->wait();
      if (o.status != "DONE") continue;
      ++done;
      jct.push_back(double(jct_us(o.metrics)));
      text += o.text_tokens.size();
      codec += o.codec_tokens.size();
      wave += o.waveform.size();
    }
    orch.shutdown(true);
    double mean = 0;
    for (double x : jct) mean += x;
    mean = jct.empty() ? 0 : mean / jct.size();
    std::printf(
        "{\"completed\": %llu, \"wall_s\": %.6f, \"requests_per_s\": %.6f, \"mean_jct_us\": %.1f, "
        "\"p99_jct_us\": %.1f, \"text_tokens\": %llu, \"codec_tokens\": %llu, \"wave_samples\": %llu, "
        "\"threads\": %d, \"weight_init_s\": %.3f}\n",
        (unsigned long long)done, wall, done / wall, mean, bench::detail::nearest_rank(jct, 0.99),
        (unsigned long long)text, (unsigned long long)codec, (unsigned long long)wave, omp_get_max_threads(),
        load_s);
    om_destroy(g.thinker);
    om_destroy(g.talker);
    om_destroy(g.dit);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_cpu_pipeline: %s\n", e.what());
    return 1;
  }
  return 0;
}
