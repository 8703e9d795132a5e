// Host helpers for K1: TMA descriptor encoding and the (N, K) -> split-K rule.
#include <cudaTypedefs.h>

#include <mutex>

#include "gemm.h"

namespace omni_dev {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 K-major tensor [rows, K] with box [box_rows, 64] and 128-B swizzle.
bool encode_2d(CUtensorMap& m, const void* ptr, uint64_t rows, uint64_t K, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {K, rows};
  cuuint64_t strides[1] = {K * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

bool gemm_encode_kmajor(CUtensorMap& m, const void* ptr, uint64_t rows, uint64_t K, uint32_t box_rows) {
  return encode_2d(m, ptr, rows, K, box_rows);
}

bool encode_tile_map(CUtensorMap& m, const void* ptr, bool f32, uint64_t rows, uint64_t cols, uint32_t box_cols,
                     uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const uint64_t es = f32 ? 4 : 2;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * es};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int gemm_choose_splits(int N_pad, int K, int max_splits, int target_ctas) {
  // Fill up to `target_ctas` CTAs (decode weights: 192 — the in-chain optimum
  // measured by tools/gemm_sweep.py) with at least two 64-wide K blocks per
  // split; one cluster (<= 8 CTAs) per output tile.
  // Depends on the weight shape only — never on the batch.
  const int tiles = N_pad / 128;
  const int kb = K / 64;
  int s = 1;
  while (s * 2 <= max_splits && tiles * s * 2 <= target_ctas && (kb % (s * 2)) == 0 && kb / (s * 2) >= 2)
    s *= 2;
  return s;
}

bool gemm_make_weight(GemmWeight& w, const __nv_bfloat16* ptr, int N, int N_pad, int K,
                      int max_splits, int target_ctas) {
  if (N_pad % 128 != 0 || K % 64 != 0 || N > N_pad) return false;
  w.ptr = ptr;
  w.N = N;
  w.N_pad = N_pad;
  w.K = K;
  w.splits = gemm_choose_splits(N_pad, K, max_splits < 1 ? 1 : (max_splits > 16 ? 16 : max_splits), target_ctas);
  return encode_2d(w.tmap, ptr, N_pad, K, 128);
}

bool gemm_make_input(GemmInput& x, const __nv_bfloat16* ptr, int rows_cap, int K) {
  if (K % 64 != 0) return false;
  x.ptr = ptr;
  x.rows_cap = rows_cap;
  x.K = K;
  const uint32_t boxes[5] = {16, 32, 64, 128, 256};
  for (int i = 0; i < 5; ++i)
    if (!encode_2d(x.tmaps[i], ptr, rows_cap, K, boxes[i])) return false;
  return true;
}

}  // namespace omni_dev
