// K6': persistent dataflow DiT iteration (dit_fused.cu). Internal to libomni_dev.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dit_kernels.h"

namespace omni_dev {

constexpr int kDitMaxLayers = 8;
constexpr int kDitMaxPhases = 256;  // T * (3 + 7 L)
// Row tiles are 128 rows (8 tokens) or 256 rows (16 tokens) = MMA N, chosen
// per launch by batch size (dit_tile_rows); buffers are sized for 128.
constexpr int kDitTileRows = 128;  // the smaller tile: padding unit and counter sizing
constexpr int kDitTileTok = 8;
constexpr int kDitFeat = 128;      // output features per GEMM item = MMA M (TMEM lanes)

// TMA descriptors of one DiT stage, resident in global memory (written once
// at stage creation): keeping them out of the kernel parameter block keeps
// the scalar parameters in a few constant-cache lines.
struct DitMaps {
  // weights (MMA A operand), 128-row boxes; w_out is [C_pad 128, d]
  CUtensorMap w_in, w_out;
  CUtensorMap wqkv[kDitMaxLayers], wo[kDitMaxLayers], w1[kDitMaxLayers], w2[kDitMaxLayers];
  CUtensorMap x_x[2], x_a[2], x_o[2], x_u[2];  // activations (MMA B operand), [0] 128- / [1] 256-row boxes
  // pre-tiled weight copies (16 KB SWIZZLE_128B tile images, gemm_block_weight),
  // nullptr: load the 128-row boxes of the maps above
  const uint8_t *b_in, *b_out;
  const uint8_t *b_qkv[kDitMaxLayers], *b_o[kDitMaxLayers], *b_1[kDitMaxLayers], *b_2[kDitMaxLayers];
};

// Everything else one iteration needs (a small __grid_constant__ parameter).
struct DitFusedParams {
  const DitMaps* maps;             // device copy, 64-byte aligned
  const DitTokDesc* toks;          // [n_rt * 8] (batch padded to whole row tiles)
  const __nv_bfloat16* pos_emb;    // [16][d]
  const float* mod_table;          // [T][vocab][L * 6 * d]
  float* x;                        // [rows][C] latent (fp32)
  __nv_bfloat16* xb;               // [rows][C] its bf16 copy (IN-proj operand)
  float* h;                        // [rows][d] residual stream
  __nv_bfloat16 *a, *qkv, *o, *u;  // LN out [rows][d], [rows][3d], attn out [rows][d], [rows][ff]
  float* part;                     // MLP-down first partial of each pair [n_rt * d/128][2][TR rows][128]
  float* part2;                    // first pair sum (split 4) [n_rt * d/128][TR rows][128]
  int32_t* samples;                // [rows] int32 samples (last Euler step)
  int* progress;                   // [n_rt] units completed per row tile (zeroed per launch)
  int* tile_cnt;                   // [n_rt * d/128][2] arrivals per pair (zeroed per launch)
  int* ready;                      // [n_rt * d/128][2] pair partials written (zeroed per launch)
  int* tile_cnt2;                  // [n_rt * d/128] pair sums finished (split 4)
  int* ready2;                     // [n_rt * d/128] first pair sum written
  int* next_item;                  // global item counter (zeroed per launch)
  unsigned long long* trace;       // optional [items][5]: fetch, dep ok, mma done, done, smid
  int n_rt, tile_rows, d, C, H, ff, L, T, vocab, down_split;
  float dt, sample_scale;
};

// Total items of one launch (tests / tools).
int dit_fused_items(int n_rt, int tile_rows, int d, int H, int ff, int L, int T, int down_split);
// Row tile of a batch of n_tok (padded) tokens on a persistent grid of
// `ctas`: 128 rows (more, shorter items: the per-layer dependency chain of a
// tile is the iteration's latency floor) until the batch has as many tokens
// as the grid has CTAs, 256 rows from there (throughput: half the weight
// re-reads and per-item overheads). Measured crossovers
// (profiles/r02_dit_fused_v7.txt): ~128 tokens on 148 CTAs, 16-96 on 64.
// n_tok must be a multiple of tile/16 (dit_pad_tokens).
inline int dit_tile_rows(int n_tok, int ctas) { return n_tok >= ctas && n_tok % 16 == 0 ? 256 : 128; }
// Model shapes the fused iteration covers (others run one kernel per op).
bool dit_fused_supported(int d, int C, int H, int ff, int L, int T);
// ctas: persistent grid (stages: ignored, 4-stage rings).
cudaError_t dit_fused_run(const DitFusedParams& p, int stages, int ctas, cudaStream_t st);

}  // namespace omni_dev
