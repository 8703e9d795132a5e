// C ABI of libomni_serve (include/omni_serve.h).
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <vector>
#include <set>
#include <string>

#include "omni/b200_pipeline.hpp"
#include "omni/bench.hpp"
#include "omni/config.hpp"
#include "omni/http_service.hpp"
#include "omni/stage_worker.hpp"
#include "omni_serve.h"

namespace {
thread_local std::string g_err;

template <typename F>
omni_status guard(F&& f) {
  try {
    f();
    return OMNI_OK;
  } catch (const omni::DeviceError& e) {
    g_err = e.what();
    return OMNI_E_CUDA;
  } catch (const omni::RegionFull& e) {
    g_err = e.what();
    return OMNI_E_OOM;
  } catch (const omni::ForwardError& e) {
    g_err = e.what();
    return OMNI_E_FORWARD;
  } catch (const std::exception& e) {
    g_err = e.what();
    return OMNI_E_BADARG;
  }
}

uint64_t fnv_i32(const std::vector<int32_t>& v, uint64_t h) {
  for (int32_t x : v)
    for (int i = 0; i < 4; ++i) {
      h ^= static_cast<uint8_t>(static_cast<uint32_t>(x) >> (8 * i));
      h *= 1099511628211ull;
    }
  return h;
}

std::string hex64(uint64_t v) {
  char b[32];
  std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(v));
  return b;
}
}  // namespace

struct omni_pipeline {
  omni::DeploymentPlan plan;
  std::unique_ptr<omni::B200Pipeline> dev;
  omni::FunctionRegistry reg;
  std::string csv, trace;
  struct Captured {
    std::vector<uint8_t> prompt;
    std::vector<int32_t> text, codec, wave;
  };
  std::map<uint64_t, Captured> outputs;  // spec->capture: per-request outputs of the last bench
  // live serving (omni_pipeline_serve_start): orchestrator loop + HTTP front end
  std::unique_ptr<omni::Orchestrator> orch;
  std::unique_ptr<omni::HttpService> http;
  ~omni_pipeline() {
    if (http) http->stop();
    if (orch) orch->shutdown(false);
  }
};

extern "C" {

const char* omni_serve_last_error(void) { return g_err.c_str(); }

omni_status omni_pipeline_create(const char* config_json, const omni_pipeline_opts* opts, omni_pipeline** out) {
  return guard([&] {
    auto p = std::make_unique<omni_pipeline>();
    p->plan = omni::parse_plan_text(config_json);
    omni::B200Options o;
    if (opts) {
      o.weight_seed = opts->weight_seed;
      o.small_models = opts->small_models != 0;
    }
    const int dev = opts ? opts->device : 0;
    for (const auto& [id, w] : p->plan.workers) {
      if (id.rfind("cuda:", 0) == 0) {  // device-keyed: every stage replica there but the Thinker
        o.workers[id] = w;
        continue;
      }
      bool known = false;
      for (const auto& n : p->plan.graph.nodes) known = known || n.id == id;
      if (!known) throw omni::ConfigInvalid("workers names unknown stage '" + id + "'");
    }
    for (const auto& n : p->plan.graph.nodes) {
      const std::string fn = n.kind == omni::StageKind::AR ? n.forward_ref
                                                           : (n.forward_ref.empty() ? "denoise" : n.forward_ref);
      // the plan's placement (stage -> "cuda:N[,cuda:M...]"), else opts->device
      o.devices[fn] = omni::placement_devices(p->plan, n.id, dev);
      if (auto w = p->plan.workers.find(n.id); w != p->plan.workers.end()) o.workers[fn] = w->second;
      o.engines[fn] = p->plan.engines.at(n.id);
      o.needed.insert(fn);
    }
    p->dev = std::make_unique<omni::B200Pipeline>(std::move(o));
    p->dev->register_into(p->reg);
    *out = p.release();
  });
}

omni_status omni_pipeline_serve_start(omni_pipeline* p, const char* listen, int32_t* port) {
  return guard([&] {
    if (p->http) throw omni::AlreadyOpen("pipeline is already serving");
    omni::DeploymentPlan plan = p->plan;
    plan.clock_kind = "device";
    p->orch = std::make_unique<omni::Orchestrator>(plan, &p->reg);
    p->orch->start();
    p->orch->serve_async();
    p->http = std::make_unique<omni::HttpService>(*p->orch);
    p->http->start(listen && *listen ? listen : "127.0.0.1:0");
    if (port) *port = p->http->port();
  });
}

omni_status omni_pipeline_serve_stop(omni_pipeline* p) {
  return guard([&] {
    if (p->http) p->http->stop();
    if (p->orch) p->orch->shutdown(true);
    p->http.reset();
    p->orch.reset();
  });
}

omni_status omni_worker_serve(const char* socket_path, int32_t accept_timeout_ms) {
  return guard([&] {
    omni::IpcChannel ch = omni::IpcChannel::listen_accept(socket_path, static_cast<uint64_t>(accept_timeout_ms));
    omni::run_stage_worker(ch);
  });
}

omni_status omni_pipeline_destroy(omni_pipeline* p) {
  return guard([&] { delete p; });
}

omni_status omni_pipeline_bench(omni_pipeline* p, const omni_bench_spec* s, omni_bench_result* r) {
  return guard([&] {
    omni::DeploymentPlan plan = p->plan;
    plan.clock_kind = s->clock ? s->clock : "device";
    // chunk overrides by edge role (transfer function), not edge position
    for (auto& e : plan.graph.edges) {
      if (s->talker_chunk > 0 && e.transfer_ref == "Thinker2Talker")
        e.streaming_chunk_size = static_cast<uint32_t>(s->talker_chunk);
      if (s->vocoder_chunk > 0 && e.transfer_ref == "Talker2Vocoder")
        e.streaming_chunk_size = static_cast<uint32_t>(s->vocoder_chunk);
    }
    omni::bench::WorkloadSpec spec;
    spec.n = s->n;
    spec.seed = s->seed;
    spec.stream = s->stream != 0;
    spec.arrival = s->poisson ? "poisson" : "closed-loop";
    spec.rate = s->rate > 0 ? s->rate : 1.0;
    if (s->prompt_min) spec.prompt_min = s->prompt_min;
    if (s->prompt_max) spec.prompt_max = s->prompt_max;
    auto workload = omni::bench::gen_workload(spec);
    omni::bench::BenchOptions bo;
    bo.concurrency = s->concurrency ? s->concurrency : 16;
    const std::string th = plan.graph.entry;
    bo.thinker_stage = th;
    bo.talker_stage = "talker";
    for (const auto& n : plan.graph.nodes)
      if (n.kind == omni::StageKind::AR && n.forward_ref == "talker_forward") bo.talker_stage = n.id;
    p->outputs.clear();
    p->dev->set_capture(s->capture != 0);
    omni::Tracer tracer;
    p->dev->set_tracer(s->trace ? &tracer : nullptr);
    p->dev->reset_counters();
    // The orchestrator owns its clock; trace timestamps read it through the tracer.
    auto clock = std::unique_ptr<omni::Clock>();
    const auto t0 = std::chrono::steady_clock::now();
    omni::bench::BenchReport rep;
    {
      if (plan.server.admission_cap < workload.size() + 1) plan.server.admission_cap = workload.size() + 1;
      omni::Orchestrator orch(plan, &p->reg);
      tracer.clock = &orch.clock();
      orch.start();
      std::vector<std::shared_ptr<omni::ResultHandle>> handles(workload.size());
      size_t next = 0;
      auto launch = [&](uint64_t at) {
        if (next >= workload.size()) return;
        const size_t i = next++;
        handles[i] = orch.submit_at(workload[i], at);
      };
      if (s->poisson) {
        const uint64_t base = orch.clock().now_us();
        for (size_t i = 0; i < workload.size(); ++i)
          handles[i] = orch.submit_at(workload[i], base + workload[i].submitted_at_us);
        next = workload.size();
      } else {
        orch.set_on_done([&](uint64_t, uint64_t now) { launch(now); });
        const uint64_t start = orch.clock().now_us();
        for (size_t i = 0; i < std::min<size_t>(bo.concurrency, workload.size()); ++i) launch(start);
      }
      orch.run_until_drained();
      rep.mode = "disaggregated";
      std::vector<omni::MetricsRecord> recs;
      uint64_t digest = 1469598103934665603ull, first = omni::kTimeUnset, last = 0;
      for (size_t i = 0; i < workload.size(); ++i) {
        const auto& out = handles[i]->wait();
        recs.push_back(out.metrics);
        auto row = omni::bench::row_from_record(out.metrics, bo.thinker_stage, bo.talker_stage);
        row.request_id = workload[i].request_id;
        if (out.status != "DONE") row.status = out.status;
        rep.rows.push_back(row);
        uint64_t od = 1469598103934665603ull;
        od = fnv_i32(out.text_tokens, od);
        od = fnv_i32(out.codec_tokens, od);
        od = fnv_i32(out.waveform, od);
        digest = fnv_i32(out.text_tokens, digest);
        digest = fnv_i32(out.codec_tokens, digest);
        digest = fnv_i32(out.waveform, digest);
        if (out.status == "DONE") ++rep.completed;
        if (s->capture) {
          auto& c = p->outputs[workload[i].request_id];
          c.prompt = workload[i].prompt_tokens;
          c.text = out.text_tokens;
          c.codec = out.codec_tokens;
          c.wave = out.waveform;
        }
        const auto& m = out.metrics;
        if (m.submitted_at != omni::kTimeUnset) first = std::min(first, m.submitted_at);
        if (m.done_at != omni::kTimeUnset) last = std::max(last, m.done_at);
        if (s->trace) {
          tracer.out += "R " + std::to_string(workload[i].request_id) + " " + out.status + " " +
                        std::to_string(m.submitted_at) + " " + std::to_string(m.done_at) + " " +
                        std::to_string(m.first_final_chunk_at == omni::kTimeUnset ? -1LL
                                                                                 : (long long)m.first_final_chunk_at) +
                        " " + std::to_string(out.text_tokens.size()) + " " + std::to_string(out.codec_tokens.size()) +
                        " " + std::to_string(out.waveform.size()) + " " + hex64(od);
          for (const auto& [st, tim] : m.stages)
            tracer.out += " " + st + ":" + std::to_string((long long)tim.first_scheduled_at) + ":" +
                          std::to_string((long long)tim.first_token_at) + ":" +
                          std::to_string((long long)tim.finished_at) + ":" + std::to_string(tim.tokens);
          tracer.out += "\n";
        }
      }
      r->preemptions = 0;
      for (const auto& n : plan.graph.nodes) r->preemptions += orch.preemptions(n.id);
      orch.shutdown(true);
      omni::bench::finish_report(rep, recs, spec);
      rep.makespan_us = (first == omni::kTimeUnset || last < first) ? 0 : last - first;
      rep.requests_per_s = rep.makespan_us ? rep.completed / (rep.makespan_us / 1e6) : 0;
      r->output_digest = digest;
    }
    p->dev->set_tracer(nullptr);
    r->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    r->completed = rep.completed;
    r->failed = workload.size() - rep.completed;
    r->makespan_us = static_cast<double>(rep.makespan_us);
    r->requests_per_s = rep.requests_per_s;
    r->mean_jct_us = rep.mean.jct_us;
    r->p50_jct_us = rep.p50.jct_us;
    r->p95_jct_us = rep.p95.jct_us;
    r->p99_jct_us = rep.p99.jct_us;
    r->mean_ttft_us = rep.mean.ttft_us;
    r->p99_ttft_us = rep.p99.ttft_us;
    r->mean_rtf = rep.mean.rtf;
    r->text_tokens = r->codec_tokens = r->wave_samples = 0;
    for (const auto& row : rep.rows) {
      r->text_tokens += row.text_tokens;
      r->codec_tokens += row.codec_tokens;
      r->wave_samples += row.waveform_samples;
    }
    const auto ms = p->dev->device_ms();
    const auto st = p->dev->step_counts();
    auto get = [](const auto& m, const char* k) { auto it = m.find(k); return it == m.end() ? decltype(it->second){} : it->second; };
    r->dev_ms_thinker = get(ms, "thinker_forward") + get(ms, "ar_forward");
    r->dev_ms_talker = get(ms, "talker_forward");
    r->dev_ms_dit = get(ms, "denoise") + get(ms, "dit_image");
    r->steps_thinker = get(st, "thinker_forward") + get(st, "ar_forward");
    r->steps_talker = get(st, "talker_forward");
    r->steps_dit = get(st, "denoise") + get(st, "dit_image");
    const auto hm = p->dev->host_ms();
    auto hget = [&](const char* k) { auto it = hm.find(k); return it == hm.end() ? std::pair<double, double>{0, 0} : it->second; };
    r->host_ms_thinker = hget("thinker_forward").first + hget("ar_forward").first;
    r->host_ms_talker = hget("talker_forward").first;
    r->host_ms_dit = hget("denoise").first + hget("dit_image").first;
    r->gap_us_thinker = 1e3 * std::max(hget("thinker_forward").second, hget("ar_forward").second);
    r->gap_us_talker = 1e3 * hget("talker_forward").second;
    r->gap_us_dit = 1e3 * std::max(hget("denoise").second, hget("dit_image").second);
    p->csv = rep.csv;
    p->trace = std::move(tracer.out);
  });
}

size_t omni_pipeline_output(omni_pipeline* p, uint64_t request_id, int32_t what, void* buf, size_t cap) {
  auto it = p->outputs.find(request_id);
  if (it == p->outputs.end()) return 0;
  const auto& c = it->second;
  const void* src = nullptr;
  size_t n = 0;
  switch (what) {
    case OMNI_OUT_PROMPT: src = c.prompt.data(), n = c.prompt.size(); break;
    case OMNI_OUT_TEXT: src = c.text.data(), n = c.text.size() * 4; break;
    case OMNI_OUT_CODEC: src = c.codec.data(), n = c.codec.size() * 4; break;
    case OMNI_OUT_WAVE: src = c.wave.data(), n = c.wave.size() * 4; break;
    case OMNI_OUT_HIDDEN: {
      const auto* h = p->dev->captured_hidden(request_id);
      if (h) src = h->data(), n = h->size() * 2;
      break;
    }
    default: return 0;
  }
  if (buf && src) std::memcpy(buf, src, std::min(cap, n));
  return n;
}

size_t omni_pipeline_text(omni_pipeline* p, int32_t what, char* buf, size_t cap) {
  const std::string& s = what == 0 ? p->csv : p->trace;
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return s.size();
}

}  // extern "C"
