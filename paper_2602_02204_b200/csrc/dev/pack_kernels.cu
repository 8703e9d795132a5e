// K5: connector gather/pack of thinker hidden rows into the reference wire
// layout (payload.hpp:142-166) — one launch packs every chunk an iteration
// emits, straight into the consumer's device arena (local or NVLink peer).
//
// Blob of a chunk with n rows:  [u8 dtype=2 FIX16][u8 rank=2][u32 n][u32 1+d]
// then n x (1+d) little-endian u16: col 0 = token id, cols 1..d = bf16 bits
// of hidden row (begin + r). Replaces the per-row byte loop of the thinker's
// pack_chunk (reference_pipeline.hpp:113-123) + encode_payload + stash
// (connector.hpp:214-236).
//
// The chunk descriptor and the chunk's token ids live in pinned host memory
// and are read over UVA (no H2D copy ahead of the pack on the Thinker
// stream): small reads over PCIe are throughput-limited, so each block reads
// them ONCE into shared memory and the grid has only a few blocks per chunk
// (each thread loops over its words). The row of a blob word comes from a
// float reciprocal with an exact integer correction (no 64-bit division per
// thread). At 16.8 MB (64 chunks x 64 rows x d 2048) the first version took
// 52.6 us (0.10 of HBM) with per-thread UVA reads (profiles/r02_pack_large.txt).
//
// Large packs (descriptors and token ids copied to device memory first):
// every thread reads its chunk descriptor directly (one broadcast load, no
// barrier) and produces one aligned 16-byte word of the blob. Interior words
// (8 hidden elements of one row) are assembled from two 128-bit loads of the
// 16-B aligned hidden ring with a funnel shift — the row start moves by one
// u16 per row because of the token column — so both sides of the copy are
// 128-bit vector accesses; header / token-column / row-crossing words take a
// scalar path.
#include <algorithm>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "launch.cuh"
#include "pack_kernels.h"
#include "ptx.cuh"

namespace omni_dev {

namespace {

// row of hidden element e (= u16 slot - 5) in a blob of rows of w = d + 1 u16:
// e / w from a float reciprocal (exact after one correction step: e < 2^24)
__device__ __forceinline__ uint32_t row_of(uint32_t e, uint32_t w, float inv_w) {
  uint32_t r = __float2uint_rz((float)e * inv_w);
  if (r * w > e) --r;
  else if ((r + 1) * w <= e) ++r;
  return r;
}

__device__ __forceinline__ uint32_t u16_at(const PackChunkDesc& c, const int32_t* tok, const __nv_bfloat16* ring,
                                           int d, int ring_rows, int64_t u) {
  // u = u16 slot index within the blob; slots 0..4 are the 10-byte header.
  if (u < 5) {
    const uint32_t n = (uint32_t)(c.end - c.begin), w = (uint32_t)(d + 1);
    switch (u) {
      case 0: return 2u | (2u << 8);  // dtype FIX16, rank 2
      case 1: return n & 0xFFFFu;
      case 2: return n >> 16;
      case 3: return w & 0xFFFFu;
      default: return w >> 16;
    }
  }
  const uint32_t e = (uint32_t)(u - 5), w = (uint32_t)d + 1;
  const uint32_t r = row_of(e, w, 1.f / (float)w), col = e - r * w;
  if (col == 0) return (uint32_t)tok[r] & 0xFFFFu;
  const unsigned short* row =
      reinterpret_cast<const unsigned short*>(ring + ((size_t)c.slot * ring_rows + c.begin + r) * d);
  return row[col - 1];
}

// kDevDesc: the chunk descriptors and token ids are in device memory (large
// packs): every thread reads its chunk's descriptor directly (one broadcast
// load) and a token id only for a token-column word, so a block's prologue is
// one dependent load and no barrier. Otherwise (pinned host memory over UVA)
// one thread per block reads the descriptor and the block stages the token
// ids in shared memory: small reads over PCIe are throughput-limited.
template <bool kDevDesc>
__global__ void pack_hidden_kernel(const PackChunkDesc* __restrict__ chunks,
                                   const __nv_bfloat16* __restrict__ ring, int d, int ring_rows,
                                   uint8_t* __restrict__ dst_base) {
  pdl_wait();
  pdl_trigger();
  __shared__ PackChunkDesc sc;
  __shared__ int32_t stok[kDevDesc ? 1 : kPackMaxRows];
  PackChunkDesc c;
  const int32_t* tok;
  if constexpr (kDevDesc) {
    c = chunks[blockIdx.y];
    tok = c.tokens_dev;
  } else {
    if (threadIdx.x == 0) sc = chunks[blockIdx.y];  // one UVA read per block
    __syncthreads();
    c = sc;
    for (int i = threadIdx.x; i < c.end - c.begin; i += blockDim.x) stok[i] = c.tokens_dev[i];
    __syncthreads();
    tok = stok;
  }
  const uint32_t wrow = (uint32_t)d + 1;
  const float inv_w = 1.f / (float)wrow;
  const int64_t rows = c.end - c.begin;
  const int64_t total_u16 = 5 + rows * (d + 1);
  const int64_t words = (total_u16 + 7) / 8;
  uint4* out = reinterpret_cast<uint4*>(dst_base + c.dst_offset);
  const __nv_bfloat16* rows_base = ring + ((size_t)c.slot * ring_rows + c.begin) * d;
  // kW words per thread (block-strided, coalesced per j; loads of all kW
  // words issued before the first store). Measured at 33.6 MB: kW = 1 with
  // one word per thread 14.7 us, kW = 2 / 4 (fewer blocks) 17.1 / 17.2 us --
  // occupancy, not per-thread ILP, keeps the loads in flight
  // (profiles/r02_pack_large.txt)
  constexpr int kW = 1;
  const int64_t tile = (int64_t)blockDim.x * kW;
  for (int64_t base = blockIdx.x * tile; base < words; base += (int64_t)gridDim.x * tile) {
    uint4 lo[kW], hi[kW];
    int sh[kW];
    bool fast[kW];
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      const int64_t k = base + j * (int64_t)blockDim.x + threadIdx.x;
      const int64_t u0 = 8 * k;
      fast[j] = false;
      sh[j] = 0;
      if (k < words && u0 >= 5 && u0 + 7 < total_u16) {
        const uint32_t e0 = (uint32_t)(u0 - 5);
        const uint32_t r = row_of(e0, wrow, inv_w), col0 = e0 - r * wrow;
        if (col0 >= 1 && col0 + 7 <= (uint32_t)d) {  // 8 hidden values of one row
          fast[j] = true;
          const int h0 = (int)col0 - 1;
          const uint4* src = reinterpret_cast<const uint4*>(rows_base + (size_t)r * d + (h0 & ~7));
          lo[j] = __ldg(src);
          hi[j] = (h0 & 7) ? __ldg(src + 1) : make_uint4(0, 0, 0, 0);
          sh[j] = h0 & 7;  // start element inside the 16-element window
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      const int64_t k = base + j * (int64_t)blockDim.x + threadIdx.x;
      if (k >= words) continue;
      const int64_t u0 = 8 * k;
      uint32_t w[4];
      if (fast[j]) {
        const uint32_t v[8] = {lo[j].x, lo[j].y, lo[j].z, lo[j].w, hi[j].x, hi[j].y, hi[j].z, hi[j].w};
        const int q = sh[j] >> 1;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          uint32_t a = 0, b = 0;
#pragma unroll
          for (int t = 0; t < 4; ++t)  // select v[q + m], v[q + m + 1] without local memory
            if (q == t) a = v[t + m], b = v[t + m + 1 < 8 ? t + m + 1 : 7];
          w[m] = (sh[j] & 1) ? __funnelshift_r(a, b, 16) : a;
        }
      } else {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int64_t ua = u0 + 2 * m, ub = ua + 1;
          const uint32_t lo16 = ua < total_u16 ? u16_at(c, tok, ring, d, ring_rows, ua) : 0u;
          const uint32_t hi16 = ub < total_u16 ? u16_at(c, tok, ring, d, ring_rows, ub) : 0u;
          w[m] = lo16 | (hi16 << 16);
        }
      }
      out[k] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

}  // namespace

uint64_t pack_blob_bytes(int rows, int d) { return 10ull + 2ull * (uint64_t)rows * (uint64_t)(d + 1); }

cudaError_t launch_pack_hidden(const PackChunkDesc* chunks_dev, int n_chunks, int max_rows,
                               const __nv_bfloat16* ring, int d, int ring_rows, uint8_t* dst_base,
                               bool desc_on_device, cudaStream_t st) {
  if (n_chunks == 0) return cudaSuccess;
  if (max_rows > kPackMaxRows) return cudaErrorInvalidValue;
  const int64_t words = (pack_blob_bytes(max_rows, d) + 15) / 16;
  const int threads = 256;
  // one word per thread when the descriptors are in device memory; over UVA
  // (small packs) few blocks per chunk: every block reads them once
  const int64_t by_words = (words + threads - 1) / threads;
  if (desc_on_device)
    return launch_k(pack_hidden_kernel<true>, dim3((unsigned)by_words, n_chunks), dim3(threads), 0, st, 1,
                    chunks_dev, ring, d, ring_rows, dst_base);
  const int bx = (int)std::max<int64_t>(1, std::min<int64_t>(by_words, (296 + n_chunks - 1) / n_chunks));
  return launch_k(pack_hidden_kernel<false>, dim3(bx, n_chunks), dim3(threads), 0, st, 1, chunks_dev, ring, d,
                  ring_rows, dst_base);
}

}  // namespace omni_dev
