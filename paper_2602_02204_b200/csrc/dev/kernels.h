// Launchers of the non-GEMM kernels (K2-K6). Internal to libomni_dev.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace omni_dev {

cudaError_t fill_weights(__nv_bfloat16* dst, int64_t rows_pad, int64_t rows_valid, int64_t cols,
                         uint64_t seed, uint32_t tensor_id, float scale, cudaStream_t st);

cudaError_t fill_swiglu(__nv_bfloat16* dst, int64_t ff, int64_t cols, uint64_t seed,
                        uint32_t tid_gate, uint32_t tid_up, float scale, cudaStream_t st);

}  // namespace omni_dev
