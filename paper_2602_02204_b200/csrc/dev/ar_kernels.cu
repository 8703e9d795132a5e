// K2-K4: the non-GEMM kernels of one batched AR step (Thinker / Talker).
//
//   embed            token (+ talker conditioning) -> fp32 residual rows,
//                    bf16 copy + sums of squares for the fused RMSNorm
//   (RMSNorm and RoPE + paged-KV append are fused into the GEMM epilogues,
//    gemm_tc.cu EPI_RESID_NORM / EPI_ROPE_KV / GemmEpilogue::ss_in)
//   attention        paged-KV causal attention for mixed decode / chunked-
//                    prefill entries (GQA), pages staged by 1-D TMA bulk copies
//   final_gather     final RMSNorm of DECODE rows -> hidden rows (bf16),
//                    also written to the sequence's hidden ring (Thinker)
//   argmax           greedy id + top-2 margin over the valid vocabulary
//
// All per-row work depends only on that row's own inputs (batch invariance,
// SURVEY §0.7a). Replaces StageModel::prefill/decode (registry.hpp:79-89;
// mock semantics reference_pipeline.hpp:96-154).
#include <algorithm>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ar_dev.cuh"
#include "ar_kernels.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace omni_dev {

__global__ void embed_kernel(const ArStepDev s, const __nv_bfloat16* __restrict__ emb,
                             const __nv_bfloat16* __restrict__ emb2, const float* __restrict__ hproj,
                             float* __restrict__ cond_table, int cond_rows, int d, int start_id,
                             float* __restrict__ x, __nv_bfloat16* __restrict__ xb,
                             float* __restrict__ ss_out, int ss_ld, const void* pf_ptr,
                             uint64_t pf_bytes) {
  prefetch_l2_share(pf_ptr, pf_bytes, blockIdx.x, gridDim.x, threadIdx.x, blockDim.x);
  embed_row(blockIdx.x, s, emb, emb2, hproj, cond_table, cond_rows, d, start_id, x, xb, ss_out, ss_ld, PdlDep{});
}

// Step descriptor blob pinned host -> device by the step's first kernel
// (UVA load of the pinned staging buffer) instead of a copy-engine H2D.
__global__ void desc_copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, int n16,
                                 const PageDeltaHeader* __restrict__ dsrc, int32_t* __restrict__ pt) {
  pdl_wait();  // the previous step's kernels may still read the blob / page table
  pdl_trigger();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) dst[i] = src[i];
  if (dsrc && pt) {
    const int n = dsrc->n;
    const PageDelta* dl = reinterpret_cast<const PageDelta*>(dsrc + 1);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      const PageDelta dd = dl[i];
      pt[dd.index] = dd.page;
    }
  }
}

cudaError_t launch_desc_copy(void* dst, const void* src, size_t bytes, const void* delta_src, int32_t* page_table,
                             cudaStream_t st) {
  const int n16 = (int)((bytes + 15) / 16);
  const int blocks = std::max(1, std::min(16, (n16 + 255) / 256));
  return launch_k(desc_copy_kernel, dim3(blocks), dim3(256), 0, st, 1, static_cast<uint4*>(dst),
                  static_cast<const uint4*>(src), n16, static_cast<const PageDeltaHeader*>(delta_src), page_table);
}

__global__ void gather_cond_kernel(const ArStepDev s, int d, __nv_bfloat16* __restrict__ out) {
  gather_cond_row(blockIdx.x, s, d, out, PdlDep{});
}

// Debug phase trace of the attention CTAs (omni_k_attn_trace; null = off):
// 8 globaltimer stamps per CTA of the LAST attention launch.
__device__ unsigned long long* g_attn_trace = nullptr;
cudaError_t attn_trace_set(void* p) { return cudaMemcpyToSymbol(g_attn_trace, &p, sizeof(p)); }

constexpr int kAttnWarps = 8;
constexpr int kAttnChunk = 128;
using AttnSmemK = AttnSmem<kAttnWarps, kAttnChunk>;

__global__ void __launch_bounds__(kAttnWarps * 32)
    attention_kernel(const ArStepDev s, const __nv_bfloat16* __restrict__ q, int n_heads, int n_kv,
                     int layer, int n_layers, const __nv_bfloat16* __restrict__ kv,
                     __nv_bfloat16* __restrict__ out, float scale, const void* pf_ptr,
                     uint64_t pf_bytes) {
  extern __shared__ __align__(128) uint8_t attn_smem_raw[];
  // static weights of a later GEMM (OMNI_PF_MB, default off)
  prefetch_l2_share(pf_ptr, pf_bytes, blockIdx.y * gridDim.x + blockIdx.x, gridDim.x * gridDim.y,
                    threadIdx.x, blockDim.x);
  unsigned long long* tr = g_attn_trace;
  if (tr) tr += 8ull * ((layer * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
  const AttnBlockDesc blk = s.attn_blocks[blockIdx.x];
  if (blk.ntok * (n_heads / n_kv) <= 16)
    attention_block_mma<kAttnWarps, kAttnChunk>(blockIdx.x, blockIdx.y, s, q, n_heads, n_kv, layer, n_layers, kv,
                                                out, scale, *reinterpret_cast<AttnSmemK*>(attn_smem_raw), PdlDep{},
                                                tr);
  else
    attention_block<kAttnWarps, kAttnChunk>(blockIdx.x, blockIdx.y, s, q, n_heads, n_kv, layer, n_layers, kv, out,
                                            scale, *reinterpret_cast<AttnSmemK*>(attn_smem_raw), PdlDep{}, tr);
}

__global__ void final_gather_kernel(const ArStepDev s, const float* __restrict__ x, int d, float eps,
                                    __nv_bfloat16* __restrict__ hout, __nv_bfloat16* __restrict__ ring,
                                    int ring_rows) {
  __shared__ float red[32];
  final_gather_row(blockIdx.x, s, x, d, eps, hout, ring, ring_rows, red, PdlDep{});
}

__global__ void sample_kernel(const ArStepDev s, const float* __restrict__ logits, int ld, int lo, int hi,
                              int top_k, uint64_t seed, int* __restrict__ tok_out, float* __restrict__ margin_out) {
  sample_row(blockIdx.x, s, logits, ld, lo, hi, top_k, seed, tok_out, margin_out, PdlDep{});
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_embed(const ArStepDev& s, int n_rows, const __nv_bfloat16* emb,
                         const __nv_bfloat16* emb2, const float* hproj, float* cond_table,
                         int cond_rows, int d, int start_id, float* x, __nv_bfloat16* xb, float* ss,
                         int ss_ld, const void* pf_ptr, uint64_t pf_bytes, cudaStream_t st) {
  if (d % 128 != 0) return cudaErrorInvalidValue;
  return launch_k(embed_kernel, dim3(n_rows), dim3(256), 0, st, 1, s, emb, emb2, hproj, cond_table,
                  cond_rows, d, start_id, x, xb, ss, ss_ld, pf_ptr, pf_bytes & ~uint64_t(15));
}
cudaError_t launch_gather_cond(const ArStepDev& s, int n_rows, int d, __nv_bfloat16* out,
                               cudaStream_t st) {
  return launch_k(gather_cond_kernel, dim3(n_rows), dim3(256), 0, st, 1, s, d, out);
}
cudaError_t launch_attention(const ArStepDev& s, int n_blocks, const __nv_bfloat16* q,
                             int n_heads, int n_kv, int layer, int n_layers,
                             const __nv_bfloat16* kv, __nv_bfloat16* out, const void* pf_ptr,
                             uint64_t pf_bytes, cudaStream_t st) {
  if (n_heads / n_kv > 8) return cudaErrorInvalidValue;
  static std::atomic<uint64_t> configured{0};
  const size_t smem = sizeof(AttnSmemK);
  if (cudaError_t e = smem_attr_once(attention_kernel, smem, configured); e != cudaSuccess) return e;
  return launch_k(attention_kernel, dim3(n_blocks, n_kv), dim3(kAttnWarps * 32), smem, st, 1, s, q, n_heads,
                  n_kv, layer, n_layers, kv, out, 1.0f / sqrtf((float)kHeadDim), pf_ptr,
                  pf_bytes & ~uint64_t(15));
}
cudaError_t launch_final_gather(const ArStepDev& s, int n_dec, const float* x, int d, float eps,
                                __nv_bfloat16* hout, __nv_bfloat16* ring, int ring_rows,
                                cudaStream_t st) {
  return launch_k(final_gather_kernel, dim3(n_dec), dim3(256), 0, st, 1, s, x, d, eps, hout, ring,
                  ring_rows);
}
cudaError_t launch_sample(const ArStepDev& s, const float* logits, int ld, int n, int lo, int hi, int top_k,
                          uint64_t seed, int* tok, float* margin, cudaStream_t st) {
  if (hi - lo > 32 * kSamplePerLane) return cudaErrorInvalidValue;
  return launch_k(sample_kernel, dim3(n), dim3(32), 0, st, 1, s, logits, ld, lo, hi, top_k, seed, tok, margin);
}

}  // namespace omni_dev
