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
  EPI_RESID_NORM = 6,   // R_f32[tok, n] += acc; Xb_bf16[tok, n] = bf16(R); ss_out[tok, tile] = sum R^2
  EPI_ROPE_KV = 7,      // one tile = one 128-dim head of QKV: RoPE(q,k), q -> q_out rows, k/v -> paged KV
  EPI_EULER = 8,        // DiT Euler update: x_f32[tok, n] += dt * acc; xb = bf16(x); last step: int32 sample of ch 0
};

// Fused RoPE + paged-KV append (EPI_ROPE_KV): the QKV GEMM tile n is head n
// (q heads, then k heads, then v heads), so the rotate-half pairs (i, i+64)
// live in one tile. `rows` are the step's ArRowDesc (ar_kernels.h).
struct RopeKvArgs {
  const void* rows = nullptr;
  const int32_t* page_table = nullptr;
  int max_pages = 0;
  const float2* table = nullptr;  // [pos][64] (cos, sin)
  __nv_bfloat16* q_out = nullptr;
  __nv_bfloat16* kv = nullptr;
  int n_heads = 0, n_kv = 0, layer = 0, n_layers = 0;
};

// A weight matrix W[N_pad, K] bf16 row-major resident in HBM, plus its TMA
// descriptor. Rows >= N are zero padding (N_pad multiple of 128). `splits`
// is the split-K factor, a function of (N, K) only (batch invariance).
struct GemmWeight {
  const __nv_bfloat16* ptr = nullptr;
  int N = 0, N_pad = 0, K = 0;
  int splits = 1;
  bool fill_sms = false;  // compute-bound (DiT): pick the token tile to fill 148 SMs
  CUtensorMap tmap;
  // optional pre-tiled copy: [N_pad/128][K/64] blocks of 16 KB, each the
  // SWIZZLE_128B shared-memory image of its 128 x 64 tile (gemm_block_weight);
  // loaded with 1-D bulk copies instead of strided 2-D TMA boxes
  const uint8_t* blk = nullptr;
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
  // EPI_GATED_RESID: gate row of group g = gate_index ? gate_index[g * gate_index_stride] : g
  // (DiT: the adaLN table row of the token's conditioning id)
  const int32_t* gate_index = nullptr;
  int gate_index_stride = 1;
  // Fused RMSNorm of the GEMM input X (un-normalised bf16 rows): every output
  // column (token) is scaled by rsqrt(sum_{j<ss_n} ss_in[tok*ss_ld+j] / norm_d + eps),
  // the per-128-feature partial sums of squares written by the producer
  // (EPI_RESID_NORM / the embed kernel), summed in fixed j order.
  const float* ss_in = nullptr;
  int ss_ld = 0, ss_n = 0;
  float norm_d = 0.f, norm_eps = 0.f;
  // EPI_RESID_NORM outputs (ld of xb = ldo, of ss_out = ss_ld)
  __nv_bfloat16* xb = nullptr;
  float* ss_out = nullptr;
  RopeKvArgs rope;
  // L2 prefetch of a later kernel's weights (see ptx.cuh prefetch_l2_share)
  const void* pf_ptr = nullptr;
  uint64_t pf_bytes = 0;
  // EPI_F32 only: out[tok, n] = acc + row_bias[tok % bias_period, n] (bf16 rows of width N)
  const __nv_bfloat16* row_bias = nullptr;
  int bias_period = 1;
  // EPI_EULER: step size, and on the final step the int32 sample output
  // (rint(sample_scale * x[tok, 0]) clamped to [-64, 63]; nullptr otherwise)
  float dt = 0.f, sample_scale = 0.f;
  int32_t* samples = nullptr;
  // phase trace (tools only): per CTA 8 u64 = globaltimer at entry / exit and
  // clock64 deltas of setup, producer-wait, last-load, mainloop-done, drain, end
  unsigned long long* trace = nullptr;
};

// Kernel-side argument block.
struct GemmArgs {
  int M, N, K, n_valid, splits;
  void* out;
  int ldo;
  const float* gate;
  int ldg, gate_off, rows_per_group;
  const int32_t* gate_index;
  int gate_index_stride;
  const float* ss_in;
  int ss_ld, ss_n;
  float norm_d, norm_eps;
  __nv_bfloat16* xb;
  float* ss_out;
  RopeKvArgs rope;
  const void* pf_ptr;
  uint64_t pf_bytes;
  const __nv_bfloat16* row_bias;
  int bias_period;
  unsigned long long* trace;
  float dt, sample_scale;
  int32_t* samples;
  const uint8_t* w_blk;  // GemmWeight::blk (nullptr: 2-D TMA of the row-major weight)
};

int gemm_block_n(int M);
// The AR stages' streaming weights (gate-up, down) and the DiT's GEMM weights
// are stored pre-tiled (default; OMNI_WBLOCK=0 keeps them row-major).
bool gemm_decode_weights_blocked();
// Writes the pre-tiled copy of a row-major weight [N_pad, K] (GemmWeight::blk).
cudaError_t gemm_block_weight(const __nv_bfloat16* w, int N_pad, int K, uint8_t* blk, cudaStream_t st);
// Split-K reduction by st.async push (decode tiles BN <= 32, 2- or 8-way
// splits); OMNI_SPLITK_PUSH=0 selects the cluster-barrier pull variant.
bool gemm_push_enabled();
int gemm_choose_splits(int N_pad, int K, int max_splits, int target_ctas = 192);
// max_splits / target_ctas: 8 / 192 for decode-path (weight-streaming)
// matrices (measured in-chain optimum: qkv 24x8, wo 16x8, down 16x8,
// gate-up 128x1 CTAs), 1 for the compute-bound DiT matrices. The choice is
// frozen into the weight (batch invariance).
bool gemm_make_weight(GemmWeight& w, const __nv_bfloat16* ptr, int N, int N_pad, int K,
                      int max_splits, int target_ctas = 192);
bool gemm_make_input(GemmInput& x, const __nv_bfloat16* ptr, int rows_cap, int K);
// bf16 K-major [rows, K] map, box [box_rows, 64], 128-B swizzle (an MMA operand).
bool gemm_encode_kmajor(CUtensorMap& m, const void* ptr, uint64_t rows, uint64_t K, uint32_t box_rows);
// Plain (unswizzled) 2-D tile map of a row-major [rows, cols] fp32 / bf16
// matrix with box [box_rows, box_cols] (TMA stores / reduce-adds of epilogue tiles).
bool encode_tile_map(CUtensorMap& m, const void* ptr, bool f32, uint64_t rows, uint64_t cols, uint32_t box_cols,
                     uint32_t box_rows);
cudaError_t gemm_run(const GemmWeight& w, const GemmInput& x, int M, int epi,
                     const GemmEpilogue& e, cudaStream_t st);
// Validates (w, x, M, epi, e) and fills the kernel argument block (the step
// chain, chain.cu, launches GEMM tiles itself).
cudaError_t gemm_make_args(const GemmWeight& w, const GemmInput& x, int M, int epi, const GemmEpilogue& e,
                           GemmArgs& a);

}  // namespace omni_dev
