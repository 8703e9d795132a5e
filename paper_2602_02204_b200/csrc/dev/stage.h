// Device-side stage runtime (one model instance on one GPU). Internal.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "ar_kernels.h"
#include "dit_fused.h"
#include "dit_kernels.h"
#include "gemm.h"
#include "omni_dev.h"
#include "pack_kernels.h"

namespace omni_dev {

constexpr int kStepTraceLaunches = 64;  // OMNI_STEP_TRACE: GEMM launches per step traced
constexpr int kStepTraceCtas = 512;     // CTA slots per traced launch

struct DevTensor {
  __nv_bfloat16* p = nullptr;
  int64_t rows = 0, rows_pad = 0, cols = 0;
  bool tiled = false;  // stored as 16 KB SWIZZLE_128B tile images (GemmWeight::blk), not row-major
};

struct ArLayer {
  DevTensor wqkv, wo, wgu, wd;
  GemmWeight gqkv, go, ggu, gd;
};

struct DitLayer {
  DevTensor wqkv, wo, w1, w2;
  GemmWeight gqkv, go, g1, g2;
};

struct SeqSlot {
  int slot = -1;
  std::vector<int> pages;
  // prefix cache (Thinker prompts): prompt tokens fed so far, chained keys of
  // its full prompt pages, positions [0, cached_upto) mapped from the cache
  std::vector<int32_t> toks;
  std::vector<uint64_t> keys;
  int cached_upto = 0;
  bool lookup_done = false;  // the first miss ends lookups (computed positions stay contiguous)
  bool no_cache = false;     // prompt fed out of order: never keyed
};

// Prefix cache over full 16-token prompt pages of a stage whose KV depends on
// the prompt tokens only (the Thinker): chained key of page p = f(key of page
// p-1, its 16 token ids) -> physical page, shared read-only by every sequence
// with that prefix. refs[page] = sequences mapping it + 1 while cached.
struct PrefixCache {
  bool enabled = false;
  std::unordered_map<uint64_t, int> page_of;
  std::unordered_map<int, uint64_t> key_of;
  std::vector<int> refs;
  uint64_t hit_tokens = 0, inserted_pages = 0, evicted_pages = 0;
};

// An instantiated CUDA graph of one step's kernel sequence.
struct StepGraph {
  cudaGraphExec_t exec = nullptr;
  int nodes = 0;  // kernels per replay (launch accounting)
};

// Pinned host staging + device mirror for per-step descriptors.
struct Staging {
  uint8_t* host = nullptr;
  uint8_t* dev = nullptr;
  size_t cap = 0;
  cudaEvent_t in_use = nullptr;  // last copy that read `host`
};

}  // namespace omni_dev

struct omni_stage {
  omni_model_desc m{};
  omni_stage_limits lim{};
  int dev = 0;
  uint64_t seed = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_start = nullptr, ev_done = nullptr, ev_link = nullptr;
  cudaEvent_t ev_pack = nullptr;  // recorded right after each connector pack
  bool pack_recorded = false;
  std::vector<void*> allocs;
  std::unordered_map<std::string, omni_dev::DevTensor> named;
  uint64_t weight_bytes = 0;

  // ---- AR model ----
  omni_dev::DevTensor emb, emb2, lm, whid;
  omni_dev::GemmWeight glm, ghid;
  std::vector<omni_dev::ArLayer> layers;
  int vocab_pad = 0, start_id = 0, argmax_lo = 0, argmax_hi = 0;
  int rows_cap = 0, max_pages = 0, ring_rows = 64, cond_rows = 64;
  float* x = nullptr;
  __nv_bfloat16* xn = nullptr;
  float* ss = nullptr;  // [rows][d/128] per-tile sums of squares (fused RMSNorm)
  __nv_bfloat16* q = nullptr;
  __nv_bfloat16* attn = nullptr;
  __nv_bfloat16* act = nullptr;
  __nv_bfloat16* hbuf = nullptr;
  __nv_bfloat16* condin = nullptr;
  float* hproj = nullptr;
  float* logits = nullptr;
  int32_t* d_tok = nullptr;  // device alias of the mapped pinned h_tok
  int top_k = 0;             // 0/1 greedy, k > 1 top-k sampling (omni_stage_set_sampling)
  uint64_t sample_seed = 0;
  float* cond_table = nullptr;
  __nv_bfloat16* ring = nullptr;
  __nv_bfloat16* kv = nullptr;
  float2* rope = nullptr;
  int32_t* page_table = nullptr;  // persistent [max_resident][max_pages]
  float* split_part = nullptr;     // split-KV attention scratch (long contexts; null: never split)
  int* split_cnt = nullptr;
  int split_groups = 0;            // >= attention blocks of any step: the split never runs out
  std::vector<omni_dev::PageDelta> pending_deltas;  // page assignments not yet shipped to the device
  omni_dev::GemmInput in_xn, in_attn, in_act, in_hbuf, in_cond;
  std::unordered_map<uint64_t, omni_dev::SeqSlot> seqs;
  std::vector<int> free_slots, free_pages;
  omni_dev::PrefixCache prefix;

  // ---- DiT model ----
  omni_dev::DevTensor w_in, pos_emb, tok_emb, t_emb, w_out, w_mod;
  omni_dev::GemmWeight g_in, g_out, g_mod;
  std::vector<omni_dev::DitLayer> dlayers;
  int tok_cap = 0, drows_cap = 0;
  float *dx = nullptr, *dh = nullptr;
  float* mod_table = nullptr;  // [T][vocab][L*6*d] adaLN modulation rows
  __nv_bfloat16 *dxin = nullptr, *da = nullptr, *dqkv = nullptr, *dout = nullptr, *du = nullptr,
                *dcvec = nullptr;
  int32_t* dsamples = nullptr;
  omni_dev::GemmInput din_x, din_a, din_o, din_u, din_c;
  // persistent dataflow iteration (dit_fused.cu): split-K scratch + counters
  float* dpart = nullptr;
  int* dctl = nullptr;
  int dctl_n = 0, down_split = 1, dit_stages = 4;
  int dit_ctas = 0;  // SM share of the fused iteration (omni_stage_set_sm_share); see dit_ctas_for
  int dit_sms_all = 0;
  omni_dev::DitMaps* dmaps = nullptr;  // device copy of the fused iteration's TMA descriptors
  unsigned long long* dit_trace = nullptr;  // OMNI_DIT_TRACE=1 (tools/dit_trace.py)
  int dit_trace_items = 0;

  // ---- step staging / results ----
  omni_dev::Staging desc, pack;
  int32_t* h_tok = nullptr;  // mapped: the sampler writes results to host memory directly
  unsigned long long* step_trace = nullptr;  // OMNI_STEP_TRACE debug stamps
  int32_t* h_samples = nullptr;
  bool pending = false;
  int pending_kind = 0;  // 1 = AR, 2 = DiT
  std::vector<int> pending_dec_entries;
  int pending_entries = 0;
  int32_t* user_tok = nullptr;
  float* user_margin = nullptr;
  int32_t* user_samples = nullptr;
  int64_t pending_samples = 0;
  float last_step_us = 0.f;
  std::unordered_map<uint64_t, omni_dev::StepGraph> graphs;  // step graphs by launch geometry
  std::unordered_map<uint64_t, int> key_hits;                 // eager runs per geometry before capture
};
