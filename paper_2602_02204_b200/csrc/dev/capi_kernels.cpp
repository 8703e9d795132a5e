// C-ABI: process-level entry points and kernel-level test/bench hooks.
#include <cuda_runtime.h>

#include <mutex>
#include <string>
#include <vector>

#include "common.h"
#include "gemm.h"
#include "kernels.h"
#include "omni_dev.h"

namespace omni_dev {
cudaError_t gemm_marks_set(void* p);
cudaError_t attn_trace_set(void* p);

namespace {
thread_local std::string g_last_error;

void require_gpu() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw DevError(OMNI_E_NOGPU, "no CUDA device visible (libomni_dev has no CPU fallback)");
  int dev = 0, major = 0;
  OMNI_CUDA(cudaGetDevice(&dev));
  OMNI_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) throw DevError(OMNI_E_NOGPU, "libomni_dev is built for sm_100a only");
}

void run_test_gemm(uint64_t W, int N, int K, uint64_t X, int M, int epi, uint64_t out, int ldo,
                   uint64_t gate, int ldg, int gate_off, int rpg, int* splits_out, int iters,
                   float* ms, int max_splits = 8) {
  require_gpu();
  OMNI_REQUIRE(N > 0 && K > 0 && M > 0, OMNI_E_BADARG, "gemm: empty shape");
  const int N_pad = (N + 127) / 128 * 128;
  GemmWeight w;
  GemmInput x;
  OMNI_REQUIRE(gemm_make_weight(w, reinterpret_cast<const __nv_bfloat16*>(W), N, N_pad, K, max_splits),
               OMNI_E_BADARG, "gemm: weight tensor map (N, K multiples of 128 / 64?)");
  OMNI_REQUIRE(gemm_make_input(x, reinterpret_cast<const __nv_bfloat16*>(X), M, K), OMNI_E_BADARG,
               "gemm: input tensor map");
  GemmEpilogue e;
  e.out = reinterpret_cast<void*>(out);
  e.ldo = ldo;
  e.gate = reinterpret_cast<const float*>(gate);
  e.ldg = ldg;
  e.gate_off = gate_off;
  e.rows_per_group = rpg;
  if (splits_out) *splits_out = w.splits;
  if (iters <= 0) {
    OMNI_CUDA(gemm_run(w, x, M, epi, e, 0));
    OMNI_CUDA(cudaDeviceSynchronize());
    return;
  }
  // Time a CUDA graph of `iters` launches so host launch cost is excluded.
  cudaStream_t cs;
  OMNI_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  OMNI_CUDA(gemm_run(w, x, M, epi, e, cs));  // warm-up (also sets smem attributes)
  OMNI_CUDA(cudaStreamSynchronize(cs));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  OMNI_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < iters; ++i) OMNI_CUDA(gemm_run(w, x, M, epi, e, cs));
  OMNI_CUDA(cudaStreamEndCapture(cs, &g));
  OMNI_CUDA(cudaGraphInstantiate(&ge, g, 0));
  OMNI_CUDA(cudaGraphLaunch(ge, cs));
  OMNI_CUDA(cudaStreamSynchronize(cs));
  cudaEvent_t a, b;
  OMNI_CUDA(cudaEventCreate(&a));
  OMNI_CUDA(cudaEventCreate(&b));
  OMNI_CUDA(cudaEventRecord(a, cs));
  OMNI_CUDA(cudaGraphLaunch(ge, cs));
  OMNI_CUDA(cudaEventRecord(b, cs));
  OMNI_CUDA(cudaEventSynchronize(b));
  float t = 0;
  OMNI_CUDA(cudaEventElapsedTime(&t, a, b));
  *ms = t / iters;
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(cs);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
}

}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

DevCounters& counters() {
  static DevCounters c;
  return c;
}

}  // namespace omni_dev

using namespace omni_dev;

extern "C" {

int omni_abi_version(void) { return OMNI_ABI_VERSION; }
const char* omni_last_error(void) { return g_last_error.c_str(); }

omni_status omni_device_count(int32_t* n) {
  return guarded([&] {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
    *n = c;
  });
}

omni_status omni_dev_graph_counters(uint64_t* captures, uint64_t* replays) {
  return guarded([&] {
    if (captures) *captures = counters().graph_captures;
    if (replays) *replays = counters().graph_replays;
  });
}

omni_status omni_dev_counters(uint64_t* launches, uint64_t* h2d_bytes, uint64_t* d2h_bytes) {
  return guarded([&] {
    const auto& c = counters();
    if (launches) *launches = c.launches;
    if (h2d_bytes) *h2d_bytes = c.h2d_bytes;
    if (d2h_bytes) *d2h_bytes = c.d2h_bytes;
  });
}

omni_status omni_mem_alloc(int32_t dev, uint64_t bytes, uint64_t* dev_ptr) {
  return guarded([&] {
    require_gpu();
    OMNI_CUDA(cudaSetDevice(dev));
    void* p = nullptr;
    OMNI_CUDA(cudaMalloc(&p, bytes ? bytes : 1));
    *dev_ptr = reinterpret_cast<uint64_t>(p);
  });
}
omni_status omni_mem_free(uint64_t dev_ptr) {
  return guarded([&] { OMNI_CUDA(cudaFree(reinterpret_cast<void*>(dev_ptr))); });
}
omni_status omni_mem_h2d(uint64_t dst, const void* src, uint64_t bytes) {
  return guarded([&] {
    OMNI_CUDA(cudaMemcpy(reinterpret_cast<void*>(dst), src, bytes, cudaMemcpyHostToDevice));
  });
}
omni_status omni_mem_d2h(void* dst, uint64_t src, uint64_t bytes) {
  return guarded([&] {
    OMNI_CUDA(cudaMemcpy(dst, reinterpret_cast<const void*>(src), bytes, cudaMemcpyDeviceToHost));
  });
}
omni_status omni_mem_set(uint64_t dst, int32_t byte, uint64_t bytes) {
  return guarded([&] { OMNI_CUDA(cudaMemset(reinterpret_cast<void*>(dst), byte, bytes)); });
}
omni_status omni_device_sync(void) {
  return guarded([&] { OMNI_CUDA(cudaDeviceSynchronize()); });
}

omni_status omni_k_gemm(uint64_t W, int32_t N, int32_t K, uint64_t X, int32_t M, int32_t epi,
                        uint64_t out, int32_t ldo, uint64_t gate, int32_t ldg, int32_t gate_off,
                        int32_t rows_per_group, int32_t max_splits, int32_t* splits) {
  return guarded([&] {
    run_test_gemm(W, N, K, X, M, epi, out, ldo, gate, ldg, gate_off, rows_per_group, splits, 0,
                  nullptr, max_splits);
  });
}

omni_status omni_k_gemm_time(uint64_t W, int32_t N, int32_t K, uint64_t X, int32_t M, int32_t epi,
                             uint64_t out, int32_t ldo, int32_t max_splits, int32_t iters,
                             float* ms) {
  return guarded([&] {
    run_test_gemm(W, N, K, X, M, epi, out, ldo, 0, 0, 0, 1, nullptr, iters, ms, max_splits);
  });
}

omni_status omni_k_gemm_time_multi(const uint64_t* Ws, int32_t n_w, int32_t N, int32_t K, uint64_t X,
                                   int32_t M, int32_t epi, uint64_t out, int32_t ldo, int32_t max_splits,
                                   int32_t iters, float* ms) {
  return guarded([&] {
    require_gpu();
    OMNI_REQUIRE(n_w > 0 && iters > 0, OMNI_E_BADARG, "gemm_time_multi: empty");
    const int N_pad = (N + 127) / 128 * 128;
    std::vector<GemmWeight> ws(n_w);
    // max_splits < 0: a compute-bound (DiT-style) weight, split cap -max_splits,
    // token tile chosen by the fill-the-SMs cost model (gemm_tc.cu bn_for)
    const bool fill = max_splits < 0;
    const int cap = fill ? -max_splits : max_splits;
    for (int i = 0; i < n_w; ++i) {
      OMNI_REQUIRE(gemm_make_weight(ws[i], reinterpret_cast<const __nv_bfloat16*>(Ws[i]), N, N_pad, K, cap,
                                    fill ? 64 : 192),
                   OMNI_E_BADARG, "weight tensor map");
      ws[i].fill_sms = fill;
    }
    GemmInput x;
    OMNI_REQUIRE(gemm_make_input(x, reinterpret_cast<const __nv_bfloat16*>(X), M, K), OMNI_E_BADARG, "input map");
    GemmEpilogue e;
    e.out = reinterpret_cast<void*>(out);
    e.ldo = ldo;
    cudaStream_t cs;
    OMNI_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    // decode weights as the stages store them (pre-tiled when gemm_decode_weights_blocked)
    std::vector<void*> blks;
    if (!fill && gemm_decode_weights_blocked())
      for (auto& w : ws) {
        void* p = nullptr;
        OMNI_CUDA(cudaMalloc(&p, (size_t)N_pad * K * 2));
        blks.push_back(p);
        OMNI_CUDA(gemm_block_weight(w.ptr, N_pad, K, static_cast<uint8_t*>(p), cs));
        w.blk = static_cast<const uint8_t*>(p);
      }
    for (int i = 0; i < n_w; ++i) OMNI_CUDA(gemm_run(ws[i], x, M, epi, e, cs));
    OMNI_CUDA(cudaStreamSynchronize(cs));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    OMNI_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < iters; ++i) OMNI_CUDA(gemm_run(ws[i % n_w], x, M, epi, e, cs));
    OMNI_CUDA(cudaStreamEndCapture(cs, &g));
    OMNI_CUDA(cudaGraphInstantiate(&ge, g, 0));
    OMNI_CUDA(cudaGraphLaunch(ge, cs));
    OMNI_CUDA(cudaStreamSynchronize(cs));
    cudaEvent_t a, b;
    OMNI_CUDA(cudaEventCreate(&a));
    OMNI_CUDA(cudaEventCreate(&b));
    OMNI_CUDA(cudaEventRecord(a, cs));
    OMNI_CUDA(cudaGraphLaunch(ge, cs));
    OMNI_CUDA(cudaEventRecord(b, cs));
    OMNI_CUDA(cudaEventSynchronize(b));
    float t = 0;
    OMNI_CUDA(cudaEventElapsedTime(&t, a, b));
    *ms = t / iters;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(cs);
    for (void* p : blks) cudaFree(p);
  });
}

omni_status omni_k_gemm_trace(const uint64_t* Ws, int32_t n_w, int32_t N, int32_t K, uint64_t X, int32_t M,
                              int32_t epi, uint64_t out, int32_t ldo, int32_t max_splits, uint64_t trace_dev,
                              int32_t* grid_ctas) {
  return guarded([&] {
    require_gpu();
    OMNI_REQUIRE(n_w > 0, OMNI_E_BADARG, "gemm_trace: empty");
    const int N_pad = (N + 127) / 128 * 128;
    std::vector<GemmWeight> ws(n_w);
    for (int i = 0; i < n_w; ++i)
      OMNI_REQUIRE(gemm_make_weight(ws[i], reinterpret_cast<const __nv_bfloat16*>(Ws[i]), N, N_pad, K, max_splits),
                   OMNI_E_BADARG, "weight tensor map");
    GemmInput x;
    OMNI_REQUIRE(gemm_make_input(x, reinterpret_cast<const __nv_bfloat16*>(X), M, K), OMNI_E_BADARG, "input map");
    GemmEpilogue e;
    e.out = reinterpret_cast<void*>(out);
    e.ldo = ldo;
    cudaStream_t cs;
    OMNI_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (int i = 0; i < n_w; ++i) OMNI_CUDA(gemm_run(ws[i], x, M, epi, e, cs));  // warm-up chain
    OMNI_CUDA(cudaStreamSynchronize(cs));
    // a PDL chain of n_w launches; the last one is traced
    for (int i = 0; i < n_w; ++i) {
      if (i == n_w - 1) e.trace = reinterpret_cast<unsigned long long*>(trace_dev);
      OMNI_CUDA(gemm_run(ws[i], x, M, epi, e, cs));
    }
    OMNI_CUDA(cudaStreamSynchronize(cs));
    cudaStreamDestroy(cs);
    if (grid_ctas) *grid_ctas = (N_pad / 128) * ((M + gemm_block_n(M) - 1) / gemm_block_n(M)) * ws[0].splits;
  });
}

omni_status omni_k_debug_traces(uint64_t attn_trace, uint64_t gemm_marks) {
  return guarded([&] {
    OMNI_CUDA(attn_trace_set(reinterpret_cast<void*>(attn_trace)));
    OMNI_CUDA(gemm_marks_set(reinterpret_cast<void*>(gemm_marks)));
  });
}

omni_status omni_k_fill_weights(uint64_t dst, int64_t n, uint64_t seed, uint32_t tensor_id,
                                float scale) {
  return guarded([&] {
    require_gpu();
    OMNI_CUDA(fill_weights(reinterpret_cast<__nv_bfloat16*>(dst), n, n, 1, seed, tensor_id, scale, 0));
    OMNI_CUDA(cudaDeviceSynchronize());
  });
}

}  // extern "C"
