// Device step descriptor shared by the AR kernels and the host runtime.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace omni_dev {

constexpr int kHeadDim = 128;
constexpr int kPageTokens = 16;

struct ArEntryDesc {  // one IterationBatch entry (ar_engine.hpp:56-70)
  int32_t slot;       // resident slot of the sequence (hidden ring / cond table row)
  int32_t q_len;      // span
  int32_t pos0;       // first KV position
  int32_t row0;       // first flattened token row
  int32_t is_decode;
  int32_t out_index;  // decode: emitted index k
  int32_t dec_row;    // decode: row in the compact decode output, else -1
  int32_t key;        // 32-bit hash of the request id (top-k sampler draws)
};

struct ArRowDesc {  // one token row of the step
  int32_t entry;
  int32_t pos;
  int32_t token;     // -1 = stage start id
  int32_t cond_row;  // talker conditioning row j
  int32_t slot;      // resident slot of the entry's sequence (persistent page table row)
  int32_t pad;
  uint64_t cond_src; // talker prefill: device address of the upstream hidden row
};

constexpr int kAttnQTok = 4;  // query tokens per attention block (x group heads)

struct AttnBlockDesc {  // one attention CTA row: tokens [tok0, tok0+ntok) of an entry
  int32_t entry;
  int32_t tok0;
  int32_t ntok;
  // split-KV (long contexts): bits 0-7 part, 8-15 parts P
  // (P <= 1: the block owns all of its keys), 16-31 split group (scratch slot)
  int32_t split;
};
constexpr int kAttnSplitChunks = 8;   // a split part covers <= 8 chunks of 128 keys
constexpr int kAttnMaxParts = 8;
__host__ __device__ inline int attn_split_part(int32_t v) { return v & 0xff; }
__host__ __device__ inline int attn_split_parts(int32_t v) { return (v >> 8) & 0xff; }
__host__ __device__ inline int attn_split_group(int32_t v) { return (v >> 16) & 0xffff; }
__host__ __device__ inline int32_t attn_split_pack(int part, int parts, int group) {
  return part | parts << 8 | group << 16;
}

struct ArStepDev {
  const ArEntryDesc* entries;
  const ArRowDesc* rows;
  const int32_t* page_table;   // persistent [max_resident slots][max_pages] in HBM
  const int32_t* dec_entries;  // [n_dec] entry index of each decode row
  const AttnBlockDesc* attn_blocks;
  int32_t max_pages;
  // split-KV scratch: [group][kv head][part][16 rows][kHeadDim + 2] fp32
  // (unnormalised O, running max, sum) and [group][kv head] arrival counters
  // (zero between launches: the last arriver resets its counter)
  float* split_part;
  int* split_cnt;
};

cudaError_t launch_embed(const ArStepDev& s, int n_rows, const __nv_bfloat16* emb,
                         const __nv_bfloat16* emb2, const float* hproj, float* cond_table,
                         int cond_rows, int d, int start_id, float* x, __nv_bfloat16* xb, float* ss,
                         int ss_ld, const void* pf_ptr, uint64_t pf_bytes, cudaStream_t st);
cudaError_t launch_gather_cond(const ArStepDev& s, int n_rows, int d, __nv_bfloat16* out,
                               cudaStream_t st);
cudaError_t launch_attention(const ArStepDev& s, int n_blocks, const __nv_bfloat16* q,
                             int n_heads, int n_kv, int layer, int n_layers,
                             const __nv_bfloat16* kv, __nv_bfloat16* out, const void* pf_ptr,
                             uint64_t pf_bytes, cudaStream_t st);
cudaError_t launch_final_gather(const ArStepDev& s, int n_dec, const float* x, int d, float eps,
                                __nv_bfloat16* hout, __nv_bfloat16* ring, int ring_rows,
                                cudaStream_t st);
// Fused final RMSNorm + LM head (CUDA cores) + greedy argmax, vocab <= 256.
cudaError_t attn_trace_set(void* p);  // debug: per-CTA phase stamps of attention launches
// Page-table delta carried by a step's descriptor blob.
struct PageDelta {
  int32_t index;  // slot * max_pages + page ordinal
  int32_t page;
};
struct PageDeltaHeader {
  int32_t n;
  int32_t pad[3];
};
constexpr int kPageDeltaCap = 1024;
// Copies the step descriptor blob from pinned staging (UVA loads) and applies
// the page-table delta (delta_src: header + PageDelta[n], pinned host).
// Ordering contract: the kernel launched right after it must pdl_wait before
// pdl_trigger (PdlDep) -- attention and the push GEMM prologues read the
// descriptors before their own pdl_wait, relying on that chain.
cudaError_t launch_desc_copy(void* dst, const void* src, size_t bytes, const void* delta_src,
                             int32_t* page_table, cudaStream_t st);
// Greedy argmax (top_k <= 1) or top-k sampling of each decode row, + top-2 margin.
cudaError_t launch_sample(const ArStepDev& s, const float* logits, int ld, int n, int lo, int hi, int top_k,
                          uint64_t seed, int* tok, float* margin, cudaStream_t st);

}  // namespace omni_dev
