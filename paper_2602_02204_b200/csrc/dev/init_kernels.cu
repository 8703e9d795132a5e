// Device-side weight materialisation: random-init bf16 tensors generated in
// place from the counter-based stream (rng.h), so a stage's weights never
// cross PCIe and match the CPU oracle bit for bit.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "rng.h"

namespace omni_dev {

__global__ void fill_weights_kernel(__nv_bfloat16* __restrict__ dst, int64_t n, uint64_t seed,
                                    uint32_t tensor_id, float mult, int64_t rows_valid,
                                    int64_t cols, int64_t row_stride_elems) {
  // Logical tensor [rows_valid, cols]; physical rows padded to row_stride.
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = i / row_stride_elems, c = i % row_stride_elems;
  float v = 0.f;
  if (r < rows_valid && c < cols) v = static_cast<float>(irwin4(weight_hash(seed, tensor_id, r * cols + c))) * mult;
  dst[i] = __float2bfloat16_rn(v);
}

// Gate/up weights of a SwiGLU MLP, interleaved per 128-row GEMM tile:
// physical row p of tile t = p / 128 holds gate feature t*64 + r (r < 64) or
// up feature t*64 + r - 64, so EPI_SWIGLU finds both halves in one tile.
__global__ void fill_swiglu_kernel(__nv_bfloat16* __restrict__ dst, int64_t n, int64_t cols,
                                   uint64_t seed, uint32_t tid_gate, uint32_t tid_up, float mult) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t p = i / cols, c = i % cols;
  const int64_t t = p / 128, r = p % 128;
  const bool gate = r < 64;
  const int64_t f = t * 64 + (gate ? r : r - 64);
  const float v = static_cast<float>(irwin4(weight_hash(seed, gate ? tid_gate : tid_up, f * cols + c))) * mult;
  dst[i] = __float2bfloat16_rn(v);
}

cudaError_t fill_swiglu(__nv_bfloat16* dst, int64_t ff, int64_t cols, uint64_t seed,
                        uint32_t tid_gate, uint32_t tid_up, float scale, cudaStream_t st) {
  const int64_t n = 2 * ff * cols;
  const int threads = 256;
  fill_swiglu_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, st>>>(
      dst, n, cols, seed, tid_gate, tid_up, weight_mult(scale));
  return cudaGetLastError();
}

cudaError_t fill_weights(__nv_bfloat16* dst, int64_t rows_pad, int64_t rows_valid, int64_t cols,
                         uint64_t seed, uint32_t tensor_id, float scale, cudaStream_t st) {
  const int64_t n = rows_pad * cols;
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  fill_weights_kernel<<<(unsigned)blocks, threads, 0, st>>>(dst, n, seed, tensor_id,
                                                           weight_mult(scale), rows_valid, cols, cols);
  return cudaGetLastError();
}

}  // namespace omni_dev
