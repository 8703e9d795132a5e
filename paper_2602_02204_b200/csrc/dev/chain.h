// The one-launch AR step ("step chain", chain.cu): op table + launch.
// Internal to libomni_dev.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>

#include "ar_kernels.h"
#include "gemm.h"

namespace omni_dev {

enum ChainOpKind : int {
  CHAIN_GATHER_COND = 0,  // talker: gather upstream hidden rows (item = row)
  CHAIN_EMBED = 1,        // item = row
  CHAIN_GEMM = 2,         // item = tile + n_tiles * split
  CHAIN_ATTN = 3,         // item = attention block * n_kv + kv head
  CHAIN_FINAL = 4,        // item = decode row
  CHAIN_ARGMAX = 5,       // item = decode row
  CHAIN_HEAD = 6,         // fused final norm + LM head + argmax, item = decode row
};

constexpr int kChainMaxOps = 48;
constexpr int kChainMaxSplits = 8;
constexpr int kChainCluster = 8;  // CTAs per cluster = items per ticket; ops are padded to multiples of 8

struct ChainOp {
  int kind;
  int n_items;  // CTAs of this op
  int first;    // ticket of its first item
  int units;    // completion signals that mark it done (GEMM: tiles, else items)
  // GEMM
  int w_map, x_map;  // indices into ChainParams::maps
  int epi;
  int n_tiles, splits, kb_per;
  // attention
  int layer;
  GemmArgs a;
};

struct ChainParams {
  ArStepDev sd;
  const CUtensorMap* maps;  // global-memory TMA descriptors of the stage
  int* done;                // [kChainMaxOps] completion counters + [1] ticket (zeroed per launch)
  int* ticket;
  int n_ops;
  unsigned long long* trace;  // optional: per ticket {start, dependency met, end} globaltimer ns
  // embed
  const __nv_bfloat16* emb;
  const __nv_bfloat16* emb2;
  const float* hproj;
  float* cond_table;
  int cond_rows, d, start_id;
  float* x;
  __nv_bfloat16* xb;
  float* ss;
  int ss_ld;
  // talker conditioning gather
  int cond_dim;
  __nv_bfloat16* condin;
  // attention
  const __nv_bfloat16* q;
  int n_heads, n_kv, n_layers;
  const __nv_bfloat16* kv;
  __nv_bfloat16* attn;
  float attn_scale;
  // final norm / argmax
  float eps;
  __nv_bfloat16* hbuf;
  __nv_bfloat16* ring;
  int ring_rows;
  float* logits;
  const __nv_bfloat16* lm;
  int vocab;
  int vocab_pad, argmax_lo, argmax_hi;
  int* tok;
  float* margin;
  ChainOp ops[kChainMaxOps];
};
static_assert(sizeof(ChainParams) <= 32000, "kernel parameter space");

size_t chain_smem_bytes();
int chain_max_rows();  // steps with more token rows use the per-kernel path
cudaError_t chain_launch(const ChainParams& P, int n_items, cudaStream_t st);

}  // namespace omni_dev
