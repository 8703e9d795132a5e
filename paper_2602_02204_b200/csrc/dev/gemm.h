// Host-side interface of the tcgen05 GEMM (K1). Internal to libomni_dev.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace omni_dev {

enum GemmEpi : int {
  EPI_BF16 = 0,         // Y_bf16[tok, n] = acc
  EPI_F32 = 1,          // Y_f32[tok, n] = acc
  EPI_RESID = 2,        // R_f32[tok, n] += acc                  (residual stream)
  EPI_GATED_RESID = 3,  // R_f32[tok, n] += gate[tok/G, off+n] * acc   (DiT adaLN gate)
  EPI_SWIGLU = 4,       // act_bf16[tok, f] = silu(acc[gate f]) * acc[up f]  (tile-interleaved)
  EPI_GELU = 5,         // Y_bf16[tok, n] = gelu_tanh(acc)
};

// A weight matrix W[N_pad, K] bf16 row-major resident in HBM, plus its TMA
// descriptor. Rows >= N are zero padding (N_pad multiple of 128). `splits`
// is the split-K factor, a function of (N, K) only (batch invariance).
struct GemmWeight {
  const __nv_bfloat16* ptr = nullptr;
  int N = 0, N_pad = 0, K = 0;
  int splits = 1;
  CUtensorMap tmap;
};

// An activation buffer X[rows_cap, K] bf16 row-major; one TMA descriptor per
// token-tile height (16, 32, 64, 128, 256).
struct GemmInput {
  const __nv_bfloat16* ptr = nullptr;
  int rows_cap = 0, K = 0;
  CUtensorMap tmaps[5];
  const CUtensorMap& tmap_for(int bn) const {
    return tmaps[bn <= 16 ? 0 : bn <= 32 ? 1 : bn <= 64 ? 2 : bn <= 128 ? 3 : 4];
  }
};

struct GemmEpilogue {
  void* out = nullptr;  // bf16 / f32 output or f32 residual (per epilogue)
  int ldo = 0;
  const float* gate = nullptr;
  int ldg = 0, gate_off = 0, rows_per_group = 1;
};

// Kernel-side argument block.
struct GemmArgs {
  int M, N, K, n_valid, splits;
  void* out;
  int ldo;
  const float* gate;
  int ldg, gate_off, rows_per_group;
};

int gemm_block_n(int M);
int gemm_choose_splits(int N_pad, int K, int max_splits);
// max_splits: 8 for decode-path (weight-streaming) matrices, 1 for the
// compute-bound DiT matrices. The choice is frozen into the weight.
bool gemm_make_weight(GemmWeight& w, const __nv_bfloat16* ptr, int N, int N_pad, int K,
                      int max_splits);
bool gemm_make_input(GemmInput& x, const __nv_bfloat16* ptr, int rows_cap, int K);
cudaError_t gemm_run(const GemmWeight& w, const GemmInput& x, int M, int epi,
                     const GemmEpilogue& e, cudaStream_t st);

}  // namespace omni_dev
