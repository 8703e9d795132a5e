// ORACLE / TEST INFRASTRUCTURE — never linked into the product.
//
// Driver that compiles the UNMODIFIED reference headers (/root/reference/proj/
// include, read-only) and dumps golden vectors for the B200 build's parity
// tests:
//   digests                       — gen_workload / monolithic oracle / CSV
//                                   digests (bench.hpp:31-56, 225-303;
//                                   reference_pipeline.hpp:260-312)
//   trace <cfg.json> <n> <seed> <conc> <stream> [chunk0 chunk1]
//                                 — per-iteration batch trace of the
//                                   reference control plane driven by its own
//                                   mock hooks (ar_engine.hpp:149-337), the
//                                   packed chunk layout (ar_engine.hpp:339-374)
//                                   and per-request outputs/metrics.
// Output goes to stdout; oracle/make_golden.sh commits it under tests/golden.
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>

#include "omniserve/bench.hpp"
#include "omniserve/config.hpp"
#include "omniserve/orchestrator.hpp"
#include "omniserve/reference_pipeline.hpp"

using namespace omni;

namespace {

uint64_t fnv(const uint8_t* p, size_t n, uint64_t h = 1469598103934665603ull) {
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}
uint64_t fnv_u64(uint64_t v, uint64_t h) {
  uint8_t b[8];
  for (int i = 0; i < 8; ++i) b[i] = uint8_t(v >> (8 * i));
  return fnv(b, 8, h);
}
uint64_t fnv_i32s(const std::vector<int32_t>& v, uint64_t h) {
  for (int32_t x : v) {
    uint8_t b[4];
    for (int i = 0; i < 4; ++i) b[i] = uint8_t(uint32_t(x) >> (8 * i));
    h = fnv(b, 4, h);
  }
  return h;
}

std::string hex64(uint64_t v) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)v);
  return buf;
}

int cmd_digests() {
  bench::WorkloadSpec spec;
  spec.n = 100;
  spec.seed = 7;
  auto wl = bench::gen_workload(spec);
  uint64_t wd = 1469598103934665603ull;
  for (const auto& r : wl) {
    wd = fnv_u64(r.request_id, wd);
    wd = fnv(r.prompt_tokens.data(), r.prompt_tokens.size(), wd);
    uint8_t s[4];
    for (int i = 0; i < 4; ++i) s[i] = uint8_t(r.seed >> (8 * i));
    wd = fnv(s, 4, wd);
  }
  auto plan = load_plan(std::string(OMNI_CONFIG_DIR) + "/reference.json");
  uint64_t od = 1469598103934665603ull;
  size_t nt = 0, nc = 0, nw = 0;
  for (const auto& r : wl) {
    VirtualClock clk;
    auto out = ref::monolithic_oracle(r, plan.engines, clk);
    od = fnv_i32s(out.text_tokens, od);
    od = fnv_i32s(out.codec_tokens, od);
    od = fnv_i32s(out.waveform, od);
    nt += out.text_tokens.size();
    nc += out.codec_tokens.size();
    nw += out.waveform.size();
  }
  FunctionRegistry reg;
  ref::register_reference_pipeline(reg);
  plan.server_id = "golden_dig";
  auto dis = bench::run_bench(plan, reg, wl, spec, "disaggregated");
  auto mono = bench::run_bench(plan, reg, wl, spec, "monolithic");
  double red = 100.0 * (mono.mean.jct_us - dis.mean.jct_us) / mono.mean.jct_us;
  std::printf("{\"workload_n\": 100, \"workload_seed\": 7,\n");
  std::printf(" \"workload_digest\": \"%s\",\n", hex64(wd).c_str());
  std::printf(" \"first_request\": {\"id\": %llu, \"len\": %zu, \"seed\": %u},\n",
              (unsigned long long)wl[0].request_id, wl[0].prompt_tokens.size(),
              wl[0].seed);
  std::printf(" \"mono_output_digest\": \"%s\", \"text_total\": %zu, "
              "\"codec_total\": %zu, \"wave_total\": %zu,\n",
              hex64(od).c_str(), nt, nc, nw);
  std::printf(" \"disagg_csv_digest\": \"%s\", \"disagg_csv_len\": %zu,\n",
              hex64(fnv((const uint8_t*)dis.csv.data(), dis.csv.size())).c_str(),
              dis.csv.size());
  std::printf(" \"mono_csv_digest\": \"%s\", \"mono_csv_len\": %zu,\n",
              hex64(fnv((const uint8_t*)mono.csv.data(), mono.csv.size())).c_str(),
              mono.csv.size());
  std::printf(" \"disagg_mean_jct_us\": %.6f, \"mono_mean_jct_us\": %.6f, "
              "\"reduction_pct\": %.6f}\n",
              dis.mean.jct_us, mono.mean.jct_us, red);
  return 0;
}

// Wraps every registered forward so each hook call is logged with the
// virtual-clock instant it ran at.
struct Tracer {
  const Clock* clock = nullptr;
  std::ostringstream out;

  StageModel wrap(const std::string& name, StageModel m) {
    StageModel w;
    w.prefill = [this, name, inner = m.prefill](RequestContext& ctx, SeqState& seq,
                                                std::span<const uint8_t> span) {
      out << "P " << name << " " << clock->now_us() << " " << seq.request_id << " "
          << seq.consumed_prompt << " " << span.size() << "\n";
      if (inner) inner(ctx, seq, span);
    };
    w.on_prompt_consumed = [this, name, inner = m.on_prompt_consumed](
                               RequestContext& ctx, SeqState& seq) {
      inner(ctx, seq);
      out << "O " << name << " " << clock->now_us() << " " << seq.request_id << " "
          << seq.target_len << "\n";
    };
    w.decode = [this, name, inner = m.decode](RequestContext& ctx, SeqState& seq) {
      DecodeStep s = inner(ctx, seq);
      out << "D " << name << " " << clock->now_us() << " " << seq.request_id << " "
          << seq.emitted.size() << " " << s.token << "\n";
      return s;
    };
    w.pack_chunk = [this, name, inner = m.pack_chunk](const SeqState& seq, size_t b,
                                                      size_t e) {
      Payload p = inner(seq, b, e);
      auto blob = encode_payload(p);
      out << "K " << name << " " << clock->now_us() << " " << seq.request_id << " "
          << b << " " << e << " " << int(p.dtype);
      for (auto d : p.shape) out << " " << d;
      out << " " << hex64(fnv(blob.data(), blob.size())) << "\n";
      return p;
    };
    return w;
  }
};

int cmd_trace(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "trace <cfg> <n> <seed> <conc> <stream> [chunk0 chunk1]\n");
    return 2;
  }
  auto plan = load_plan(argv[2]);
  plan.server_id = "golden_trace";
  plan.clock_kind = "virtual";
  bench::WorkloadSpec spec;
  spec.n = std::stoull(argv[3]);
  spec.seed = std::stoull(argv[4]);
  size_t conc = std::stoull(argv[5]);
  spec.stream = std::stoi(argv[6]) != 0;
  if (argc >= 9) {
    plan.graph.edges.at(0).streaming_chunk_size = std::stoul(argv[7]);
    if (plan.graph.edges.size() > 1)
      plan.graph.edges.at(1).streaming_chunk_size = std::stoul(argv[8]);
  }
  auto wl = bench::gen_workload(spec);
  plan.server.admission_cap = wl.size() + 1;

  Tracer tr;
  FunctionRegistry base;
  ref::register_reference_pipeline(base);
  FunctionRegistry reg;
  ref::register_reference_pipeline(reg);
  for (const char* f : {"thinker_forward", "talker_forward", "ar_forward"})
    reg.register_forward(f, tr.wrap(f, base.forward(f)));

  auto clk = std::make_unique<VirtualClock>();
  tr.clock = clk.get();
  Orchestrator orch(plan, &reg, std::move(clk));
  orch.start();
  std::vector<std::shared_ptr<ResultHandle>> handles(wl.size());
  size_t next = 0;
  auto launch = [&](uint64_t at) {
    if (next >= wl.size()) return;
    size_t i = next++;
    handles[i] = orch.submit_at(wl[i], at);
  };
  orch.set_on_done([&](uint64_t, uint64_t now) { launch(now); });
  for (size_t i = 0; i < std::min(conc, wl.size()); ++i) launch(0);
  orch.run_until_drained();

  std::cout << tr.out.str();
  for (size_t i = 0; i < wl.size(); ++i) {
    const auto& o = handles[i]->wait();
    const auto& m = o.metrics;
    uint64_t od = 1469598103934665603ull;
    od = fnv_i32s(o.text_tokens, od);
    od = fnv_i32s(o.codec_tokens, od);
    od = fnv_i32s(o.waveform, od);
    std::cout << "R " << wl[i].request_id << " " << o.status << " " << m.submitted_at
              << " " << m.done_at << " "
              << (m.first_final_chunk_at == kTimeUnset ? -1
                                                        : (long long)m.first_final_chunk_at)
              << " " << o.text_tokens.size() << " " << o.codec_tokens.size() << " "
              << o.waveform.size() << " " << hex64(od);
    for (const auto& [st, tim] : m.stages)
      std::cout << " " << st << ":" << (long long)tim.first_scheduled_at << ":"
                << (long long)tim.first_token_at << ":" << (long long)tim.finished_at
                << ":" << tim.tokens;
    std::cout << "\n";
  }
  orch.shutdown(true);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_harness digests | trace ...\n");
    return 2;
  }
  std::string cmd = argv[1];
  try {
    if (cmd == "digests") return cmd_digests();
    if (cmd == "trace") return cmd_trace(argc, argv);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_harness: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
  return 2;
}
