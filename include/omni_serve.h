/*
 * omni_serve.h — C ABI of the stage-graph serving runtime (libomni_serve.so).
 *
 * The reference's public surface for this path is C++: Orchestrator
 * (orchestrator.hpp:107-284) driven by bench::run_bench (bench.hpp:225-312)
 * over a DeploymentPlan loaded from JSON (config.hpp:73-171). libomni_serve
 * keeps that C++ API (namespace omni, headers under csrc/serve/omni/) and
 * adds this C entry point so non-C++ hosts (the Python bench/tests here, a
 * cgo/ctypes binding elsewhere) can build a B200 pipeline from the same
 * config file and run the reference's benchmark workload on it.
 */
#ifndef OMNI_SERVE_H
#define OMNI_SERVE_H

#include <stddef.h>
#include <stdint.h>

#include "omni_dev.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct omni_pipeline omni_pipeline;

typedef struct omni_pipeline_opts {
  uint64_t weight_seed;   /* random-init weights (counter stream) */
  int32_t small_models;   /* 1 = reduced dims (tests) */
  int32_t device;         /* CUDA ordinal for every stage (single-GPU placement) */
} omni_pipeline_opts;

/* Builds every stage the plan's graph names (weights materialised on device). */
omni_status omni_pipeline_create(const char* config_json, const omni_pipeline_opts* opts,
                                 omni_pipeline** out);
omni_status omni_pipeline_destroy(omni_pipeline* p);

typedef struct omni_bench_spec {
  uint64_t n;            /* requests (bench.hpp:23-31 WorkloadSpec) */
  uint64_t seed;
  uint64_t concurrency;  /* closed-loop window (bench.hpp:217) */
  int32_t stream;        /* request.stream */
  int32_t poisson;       /* 0 closed loop, 1 poisson arrivals */
  double rate;
  uint32_t prompt_min, prompt_max;
  const char* clock;     /* "virtual" (parity), "device" (performance), "wall" */
  int32_t trace;         /* 1 = record the reference-harness trace */
  int32_t talker_chunk;  /* >0 overrides the Thinker2Talker edge chunk size */
  int32_t vocoder_chunk; /* >0 overrides the Talker2Vocoder edge chunk size */
  int32_t capture;       /* 1 = keep per-request outputs + thinker hidden rows (parity tests) */
} omni_bench_spec;

typedef struct omni_bench_result {
  uint64_t completed, failed;
  double makespan_us, requests_per_s;
  double mean_jct_us, p50_jct_us, p95_jct_us, p99_jct_us;
  double mean_ttft_us, p99_ttft_us, mean_rtf;
  uint64_t text_tokens, codec_tokens, wave_samples;
  double dev_ms_thinker, dev_ms_talker, dev_ms_dit; /* summed CUDA-event step times */
  uint64_t steps_thinker, steps_talker, steps_dit;
  uint64_t output_digest; /* FNV-1a over every request's (text, codec, waveform) */
  uint64_t preemptions;
  double wall_s;
  /* host cost of driving each stage: ms spent inside the step launches, and
     the mean gap (us) from collecting a step's results to launching the next */
  double host_ms_thinker, host_ms_talker, host_ms_dit;
  double gap_us_thinker, gap_us_talker, gap_us_dit;
} omni_bench_result;

/* Runs one full workload through a fresh Orchestrator on the pipeline. */
omni_status omni_pipeline_bench(omni_pipeline* p, const omni_bench_spec* spec, omni_bench_result* out);
/* Text of the last bench: what 0 = CSV v1, 1 = trace. Returns the full length. */
size_t omni_pipeline_text(omni_pipeline* p, int32_t what, char* buf, size_t cap);

/* Per-request outputs of the last bench run with spec->capture = 1 (parity
 * tests replay them teacher-forced through the CPU oracle). Copies up to
 * `cap` bytes into buf (may be NULL) and returns the full byte length; 0 for
 * an unknown request. */
enum {
  OMNI_OUT_PROMPT = 0, /* u8 prompt tokens                         */
  OMNI_OUT_TEXT = 1,   /* i32 thinker tokens                        */
  OMNI_OUT_CODEC = 2,  /* i32 talker codec tokens                   */
  OMNI_OUT_WAVE = 3,   /* i32 waveform samples (first diffusion exit) */
  OMNI_OUT_HIDDEN = 4  /* u16 bf16 bits of the thinker hidden rows, [text index][d] */
};
size_t omni_pipeline_output(omni_pipeline* p, uint64_t request_id, int32_t what, void* buf, size_t cap);

/* Live serving (reference http_service.hpp:88-212): starts an
 * Orchestrator loop on the device clock plus the HTTP/1.1 front end on
 * `listen` ("host:port", port 0 = any free port; the bound port is returned).
 * Routes: POST /v1/generate (JSON, or NDJSON waveform chunks when "stream"),
 * GET /v1/health, GET /v1/metrics -- the reference's bodies and status codes. */
omni_status omni_pipeline_serve_start(omni_pipeline* p, const char* listen, int32_t* port);
/* Stops accepting, drains in-flight requests, stops the loop. */
omni_status omni_pipeline_serve_stop(omni_pipeline* p);

/* Stage worker process: listens on the AF_UNIX `socket_path`,
 * accepts one orchestrator and runs the stages it creates there (steps,
 * connector arenas exported with CUDA IPC, interprocess events) until it is
 * told to shut down. A deployment plan places a stage in a worker with
 * "workers": {"<stage id>": "<socket path>"} (omni_stage_worker.hpp). */
omni_status omni_worker_serve(const char* socket_path, int32_t accept_timeout_ms);

const char* omni_serve_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* OMNI_SERVE_H */
