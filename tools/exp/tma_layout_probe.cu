// Weight-streaming layout probe: 128 CTAs stream a 67 MB bf16 matrix [16384, 2048]
// into a 6-stage shared-memory ring, (a) as 2-D TMA boxes of 128 rows x 64 cols
// (SWIZZLE_128B, the gate-up GEMM's A operand: 128 strided 128-B segments per
// box) or (b) as 1-D bulk copies of 16 KB contiguous blocks (the same bytes
// pre-tiled). No MMA: pure operand ingress. Prints us per pass (CUDA events,
// median of 20) and GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda tma_layout_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { auto e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int N = 16384, K = 2048, ROWS = 128, KB = 64, STAGES = 6;
constexpr int BOX = ROWS * KB * 2;  // 16 KB
constexpr int NKB = K / KB;         // 32 boxes per CTA

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ uint64_t evict_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }

template <bool BULK>
__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* blocked, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES];
  const int tile = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float acc = 0.f;
  const uint64_t pol = evict_first();
  for (int i = 0; i < NKB + STAGES; ++i) {
    if (i >= STAGES) {  // consume box i - STAGES
      const int s = (i - STAGES) % STAGES;
      wait(&full[s], ((i - STAGES) / STAGES) & 1);
      acc += ((const float*)(ring + s * BOX))[threadIdx.x];
      __syncthreads();
    }
    if (i < NKB && threadIdx.x == 0) {
      const int s = i % STAGES;
      expect_tx(&full[s], BOX);
      if constexpr (BULK) {
        const uint8_t* src = blocked + ((size_t)tile * NKB + i) * BOX;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(sa(ring + s * BOX)), "l"(src), "r"(BOX), "r"(sa(&full[s])), "l"(pol) : "memory");
      } else {
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;"
                     ::"r"(sa(ring + s * BOX)), "l"(&tm), "r"(sa(&full[s])), "r"(i * KB), "r"(tile * ROWS), "l"(pol) : "memory");
      }
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const size_t bytes = (size_t)N * K * 2;
  const int copies = 4;  // rotate copies: 268 MB > L2
  std::vector<uint8_t*> W(copies), B(copies);
  for (int c = 0; c < copies; ++c) {
    CK(cudaMalloc(&W[c], bytes)); CK(cudaMemset(W[c], 1, bytes));
    CK(cudaMalloc(&B[c], bytes)); CK(cudaMemset(B[c], 1, bytes));
  }
  float* sink; CK(cudaMalloc(&sink, 4));
  CUtensorMap tm[copies];
  for (int c = 0; c < copies; ++c) {
    cuuint64_t dims[2] = {K, N}, strides[1] = {K * 2};
    cuuint32_t box[2] = {KB, ROWS}, es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm[c], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W[c], dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  }
  const size_t smem = STAGES * BOX + 1024;
  CK(cudaFuncSetAttribute(stream_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(stream_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    for (int grid : {128}) {
      std::vector<float> ts;
      for (int it = 0; it < 12; ++it) {  // 16 back-to-back launches per sample (launch overhead amortised)
        cudaEventRecord(a);
        for (int r = 0; r < 16; ++r) {
          const int c = r % copies;
          if (mode == 0) stream_kernel<false><<<grid, 128, smem>>>(tm[c], B[c], sink);
          else stream_kernel<true><<<grid, 128, smem>>>(tm[c], B[c], sink);
        }
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (it >= 2) ts.push_back(ms * 1e3f / 16);
      }
      std::sort(ts.begin(), ts.end());
      const float us = ts[ts.size() / 2];
      printf("%s grid %d: %.2f us (min %.2f) = %.0f GB/s\n", mode ? "bulk 16KB contiguous" : "tma 2d 128x64 sw128", grid, us, ts[0], bytes / us / 1e3);
    }
  }
  return 0;
}
