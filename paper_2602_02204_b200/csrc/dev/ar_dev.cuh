// Device bodies of the non-GEMM AR step kernels, shared by the per-kernel
// launches (ar_kernels.cu) and the one-launch step chain (chain.cu). Each
// takes its work index explicitly and a `Dep` functor that performs the wait
// on the producer of its inputs (griddepcontrol.wait for PDL launches, the
// chain's completion counters inside the step-chain kernel). Internal.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ar_kernels.h"
#include "ptx.cuh"
#include "rng.h"

namespace omni_dev {

// wait for the predecessor, THEN let dependents launch: the kernel following
// desc_copy_kernel must use this order (later kernels read step descriptors
// before their own pdl_wait)
struct PdlDep {
  __device__ __forceinline__ void operator()() const {
    pdl_wait();
    pdl_trigger();
  }
};

// ---------------------------------------------------------------------------
// Embedding.  Thinker: x = E[tok].  Talker prefill token j:
//   cond_j = E_t[tok] + (W_h h_j) (precomputed GEMM rows in `hproj`), stored
//   to the sequence's conditioning table, x = cond_j.  Talker decode step m:
//   x = E_c[prev] + cond_{m/4}.
// Also emits the first layer's fused-RMSNorm inputs: xb = bf16(x) and the
// per-128-feature sums of squares ss[row][tile] (same fixed 16-lane order as
// the EPI_RESID_NORM GEMM epilogue).
// ---------------------------------------------------------------------------
template <class Dep>
__device__ __forceinline__ void embed_row(int r, const ArStepDev& s, const __nv_bfloat16* __restrict__ emb,
                             const __nv_bfloat16* __restrict__ emb2, const float* __restrict__ hproj,
                             float* __restrict__ cond_table, int cond_rows, int d, int start_id,
                             float* __restrict__ x, __nv_bfloat16* __restrict__ xb,
                             float* __restrict__ ss_out, int ss_ld, Dep dep) {
  dep();
  const ArRowDesc rd = s.rows[r];
  const ArEntryDesc ed = s.entries[rd.entry];
  const int tok = rd.token < 0 ? start_id : rd.token;
  float* xr = x + (size_t)r * d;
  const int mode = emb2 == nullptr ? 0 : (ed.is_decode ? 2 : 1);
  float* cond = mode ? cond_table + ((size_t)ed.slot * cond_rows + rd.cond_row) * d : nullptr;
  const __nv_bfloat16* e = mode == 2 ? emb2 + (size_t)tok * d : emb + (size_t)tok * d;
  for (int base = 0; base < d; base += blockDim.x * 8) {
    const int i0 = base + threadIdx.x * 8;
    const bool live = i0 < d;
    float ss = 0.f;
    if (live) {
      float v[8];
      const uint4 raw = *reinterpret_cast<const uint4*>(e + i0);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(h2[k]);
        v[2 * k] = f.x, v[2 * k + 1] = f.y;
      }
      if (mode == 1) {
        const float* hp = hproj + (size_t)r * d + i0;
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] += hp[k];
#pragma unroll
        for (int k = 0; k < 8; ++k) cond[i0 + k] = v[k];
      } else if (mode == 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] += cond[i0 + k];
      }
      uint4 ob;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&ob);
#pragma unroll
      for (int k = 0; k < 4; ++k) o2[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
      *reinterpret_cast<uint4*>(xb + (size_t)r * d + i0) = ob;
      reinterpret_cast<float4*>(xr + i0)[0] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(xr + i0)[1] = make_float4(v[4], v[5], v[6], v[7]);
#pragma unroll
      for (int k = 0; k < 8; ++k) ss += v[k] * v[k];
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (live && (threadIdx.x & 15) == 0) ss_out[(size_t)r * ss_ld + i0 / 128] = ss;
  }
}

// Talker: gather the upstream FIX16 hidden rows (2-byte aligned inside the
// packed connector payload) into an aligned bf16 GEMM input.
template <class Dep>
__device__ __forceinline__ void gather_cond_row(int r, const ArStepDev& s, int d, __nv_bfloat16* __restrict__ out,
                                                Dep dep) {
  dep();
  const uint64_t src = s.rows[r].cond_src;
  __nv_bfloat16* o = out + (size_t)r * d;
  if (src == 0) {
    for (int i = threadIdx.x; i < d; i += blockDim.x) o[i] = __float2bfloat16_rn(0.f);
    return;
  }
  const unsigned short* p = reinterpret_cast<const unsigned short*>(src);
  unsigned short* q = reinterpret_cast<unsigned short*>(o);
  for (int i = threadIdx.x; i < d; i += blockDim.x) q[i] = p[i];
}

__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) t += red[i];  // fixed order: deterministic
  return t;
}

// ---------------------------------------------------------------------------
// Paged causal attention (K3). Grid (query block, kv_head), 8 warps.
// A query block is up to kAttnQTok tokens of one entry (decode: 1 token) and
// holds their `group` query heads that share the KV head. The block's causal
// context [0, pos0 + tok0 + ntok) is staged into smem in 128-key chunks by
// 1-D bulk TMA copies of whole 16-token pages (double buffered, one mbarrier
// per chunk). Each warp owns query vectors; QK^T has lanes split KEYS (rotated
// column order -> conflict-free smem), the chunk softmax merges online, P.V
// has lanes split the 128 head dims.
// ---------------------------------------------------------------------------
constexpr int kAttnQMax = kAttnQTok * 8;  // query vectors per block (group <= 8)

template <int kAttnWarps, int kAttnChunk>
struct AttnSmem {
  __nv_bfloat16 k[2][kAttnChunk * kHeadDim];
  __nv_bfloat16 v[2][kAttnChunk * kHeadDim];
  float2 q[kAttnQMax][kHeadDim / 2];
  float p[kAttnWarps][kAttnChunk];
  float ml[kAttnWarps][2];  // decode split: partial (max, sum) per warp
  float mrg[kAttnWarps][kHeadDim];  // decode split: partial P.V rows per warp
  uint64_t bar[2];
};

template <int kAttnWarps, int kAttnChunk, class Dep>
__device__ __forceinline__ void attention_block(int blk_idx, int kh_idx, const ArStepDev& s,
                                                const __nv_bfloat16* __restrict__ q, int n_heads, int n_kv,
                                                int layer, int n_layers, const __nv_bfloat16* __restrict__ kv,
                                                __nv_bfloat16* __restrict__ out, float scale,
                                                AttnSmem<kAttnWarps, kAttnChunk>& sm, Dep dep,
                                                unsigned long long* tr = nullptr) {
  constexpr int HD = kHeadDim;
  constexpr uint32_t PAGE_BYTES = kPageTokens * HD * 2;  // 4 KB K or V slice of one page
  constexpr int kAttnPagesPerChunk = kAttnChunk / kPageTokens;
  // Step descriptors are readable before pdl_wait: desc_copy_kernel (the
  // step's first kernel) writes them, and the kernel after it (embed /
  // gather_cond, PdlDep) waits for it BEFORE triggering its own dependents,
  // so every later kernel of the step launches after the copy completed.
  // Keep that order: a kernel right after desc_copy must use PdlDep (wait,
  // then trigger), never trigger early (ar_kernels.cu launch_desc_copy).
  const AttnBlockDesc blk = s.attn_blocks[blk_idx];
  const int kh = kh_idx;
  const ArEntryDesc ed = s.entries[blk.entry];
  const int group = n_heads / n_kv;
  const int nq = blk.ntok * group;
  const int kend = ed.pos0 + blk.tok0 + blk.ntok;  // causal context of the block
  const int n_chunks = (kend + kAttnChunk - 1) / kAttnChunk;
  const int warp = warp_id(), lane = lane_id();

  if (threadIdx.x == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    fence_barrier_init();
  }
  // KV pages holding only positions < pos0 were written by EARLIER steps:
  // they stream in before waiting on this step's QKV GEMM (PDL); only the
  // page(s) receiving this step's K/V rows are loaded after the wait.
  auto issue = [&](int c, int buf, int part) {  // part 0: history pages (+ expect_tx), 1: the rest
    const int first = c * kAttnPagesPerChunk;
    const int keys = min(kAttnChunk, kend - c * kAttnChunk);
    const int np = (keys + kPageTokens - 1) / kPageTokens;
    if (part == 0) mbar_expect_tx(&sm.bar[buf], 2u * PAGE_BYTES * np);
    for (int i = 0; i < np; ++i) {
      const bool history = (first + i + 1) * kPageTokens <= ed.pos0;
      if (history != (part == 0)) continue;
      const int page = s.page_table[ed.slot * s.max_pages + first + i];
      const size_t base = (((size_t)page * n_layers + layer) * 2) * n_kv;
      bulk_load(sm.k[buf] + i * kPageTokens * HD, kv + (base + kh) * kPageTokens * HD, PAGE_BYTES, &sm.bar[buf]);
      bulk_load(sm.v[buf] + i * kPageTokens * HD, kv + (base + n_kv + kh) * kPageTokens * HD, PAGE_BYTES,
                &sm.bar[buf]);
    }
  };
  if (threadIdx.x == 0) {
    if (tr) tr[0] = globaltimer();
    issue(0, 0, 0);
    if (n_chunks > 1) issue(1, 1, 0);
  }
  dep();
  if (tr && threadIdx.x == 0) tr[1] = globaltimer();
  if (threadIdx.x == 0) {
    issue(0, 0, 1);
    if (n_chunks > 1) issue(1, 1, 1);
  }
  // stage the (pre-scaled) query vectors
  for (int t = threadIdx.x; t < nq * (HD / 2); t += blockDim.x) {
    const int qi = t / (HD / 2), c2 = t % (HD / 2);
    const int tok = blk.tok0 + qi / group, hq = kh * group + qi % group;
    const __nv_bfloat162 v = reinterpret_cast<const __nv_bfloat162*>(
        q + (size_t)(ed.row0 + tok) * n_heads * HD + hq * HD)[c2];
    sm.q[qi][c2] = make_float2(__low2float(v) * scale, __high2float(v) * scale);
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[2] = globaltimer();

  constexpr int QW = kAttnQMax / kAttnWarps;  // query vectors per warp (prefill blocks)
  constexpr int KG = kAttnChunk / 32;          // 32-key groups per chunk
  // Decode blocks (few query vectors): `per` warps share one query vector,
  // each taking every per-th 32-key group, and merge their partial softmax
  // states at the end (flash-decoding inside the CTA) -> all 8 warps busy.
  const int per = nq >= kAttnWarps ? 1 : min(KG, kAttnWarps / nq);
  const int part = warp % per;
  float m[QW], l[QW], acc[QW][4];
#pragma unroll
  for (int j = 0; j < QW; ++j) {
    m[j] = -INFINITY;
    l[j] = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[j][t] = 0.f;
  }

  for (int c = 0; c < n_chunks; ++c) {
    const int buf = c & 1;
    mbar_wait(&sm.bar[buf], (c >> 1) & 1);
    if (tr && c == 0 && threadIdx.x == 0) tr[3] = globaltimer();
    const int kbase = c * kAttnChunk;
    const __nv_bfloat162* K2 = reinterpret_cast<const __nv_bfloat162*>(sm.k[buf]);
    const __nv_bfloat16* V = sm.v[buf];
#pragma unroll
    for (int j = 0; j < QW; ++j) {
      const int qi = per > 1 ? (j == 0 ? warp / per : nq) : warp + j * kAttnWarps;
      if (qi >= nq) break;  // warp-uniform
      const int qpos = ed.pos0 + blk.tok0 + qi / group;
      const int nk = min(kAttnChunk, qpos + 1 - kbase);  // causal keys of this chunk
      if (nk <= 0) continue;
      float sc[KG];
      float cmax = -INFINITY;
#pragma unroll
      for (int i = 0; i < KG; ++i) {
        const int key = lane + 32 * i;
        float d = -INFINITY;
        if (key < nk && i % per == part) {
          const __nv_bfloat162* kr = K2 + key * (HD / 2);
          float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
          for (int cp = 0; cp < HD / 2; ++cp) {
            const int x = (cp + lane) & (HD / 2 - 1);  // rotated: distinct banks per lane
            const float2 kv2 = __bfloat1622float2(kr[(kv_swz(x >> 2, key) << 2) | (x & 3)]);
            const float2 qv = sm.q[qi][x];
            a0 += qv.x * kv2.x;
            a1 += qv.y * kv2.y;
          }
          d = a0 + a1;
        }
        sc[i] = d;
        cmax = fmaxf(cmax, d);
      }
      cmax = warp_max(cmax);
      if (cmax == -INFINITY) continue;  // none of this warp's keys are in range (warp-uniform)
      const float mn = fmaxf(m[j], cmax);
      const float corr = __expf(m[j] - mn);
      float ps = 0.f;
#pragma unroll
      for (int i = 0; i < KG; ++i) {
        if (i % per != part) continue;
        const float pv = (lane + 32 * i < nk) ? __expf(sc[i] - mn) : 0.f;
        sm.p[warp][lane + 32 * i] = pv;
        ps += pv;
      }
      ps = warp_sum(ps);
      l[j] = l[j] * corr + ps;
      m[j] = mn;
      __syncwarp();
      float o0 = acc[j][0] * corr, o1 = acc[j][1] * corr, o2 = acc[j][2] * corr, o3 = acc[j][3] * corr;
      for (int i = part; i < KG; i += per) {
        const int kend_i = min(nk, 32 * (i + 1));
#pragma unroll 4
        for (int k = 32 * i; k < kend_i; ++k) {
          const float pk = sm.p[warp][k];
          const uint2 raw = *reinterpret_cast<const uint2*>(V + k * HD + (kv_swz(lane >> 1, k) << 3) + (lane & 1) * 4);
          const float2 v01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
          const float2 v23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
          o0 += pk * v01.x;
          o1 += pk * v01.y;
          o2 += pk * v23.x;
          o3 += pk * v23.y;
        }
      }
      acc[j][0] = o0, acc[j][1] = o1, acc[j][2] = o2, acc[j][3] = o3;
      __syncwarp();
    }
    __syncthreads();  // every warp is done with `buf`
    if (threadIdx.x == 0 && c + 2 < n_chunks) {
      issue(c + 2, buf, 0);
      issue(c + 2, buf, 1);
    }
  }
  if (tr && threadIdx.x == 0) tr[4] = globaltimer();
  if (per > 1) {
    // merge the `per` partial (max, sum, acc) states of each query vector
    const int qi = warp / per;
    if (qi < nq) {
#pragma unroll
      for (int t = 0; t < 4; ++t) sm.mrg[warp][lane * 4 + t] = acc[0][t];
      if (lane == 0) {
        sm.ml[warp][0] = m[0];
        sm.ml[warp][1] = l[0];
      }
    }
    __syncthreads();
    if (qi < nq && part == 0) {
      float mt = -INFINITY;
      for (int p = 0; p < per; ++p) mt = fmaxf(mt, sm.ml[warp + p][0]);
      float lt = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
      for (int p = 0; p < per; ++p) {
        const float mp = sm.ml[warp + p][0];
        const float f = mp == -INFINITY ? 0.f : __expf(mp - mt);
        lt += sm.ml[warp + p][1] * f;
#pragma unroll
        for (int t = 0; t < 4; ++t) o[t] += sm.mrg[warp + p][lane * 4 + t] * f;
      }
      const int tok = blk.tok0 + qi / group, hq = kh * group + qi % group;
      const float inv = 1.f / lt;
      __nv_bfloat162* op =
          reinterpret_cast<__nv_bfloat162*>(out + (size_t)(ed.row0 + tok) * n_heads * HD + hq * HD + lane * 4);
      op[0] = __floats2bfloat162_rn(o[0] * inv, o[1] * inv);
      op[1] = __floats2bfloat162_rn(o[2] * inv, o[3] * inv);
    }
    if (tr && threadIdx.x == 0) tr[5] = globaltimer();
    return;
  }
#pragma unroll
  for (int j = 0; j < QW; ++j) {
    const int qi = warp + j * kAttnWarps;
    if (qi >= nq) break;
    const int tok = blk.tok0 + qi / group, hq = kh * group + qi % group;
    const float inv = 1.f / l[j];
    __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(out + (size_t)(ed.row0 + tok) * n_heads * HD + hq * HD + lane * 4);
    op[0] = __floats2bfloat162_rn(acc[j][0] * inv, acc[j][1] * inv);
    op[1] = __floats2bfloat162_rn(acc[j][2] * inv, acc[j][3] * inv);
  }
}


// ---------------------------------------------------------------------------
// Paged causal attention on the warp MMA (blocks with <= 16 query vectors:
// every decode block, and prefill blocks of <= 16 / group tokens). The block's
// query vectors are the M = 16 rows of mma.sync m16n8k16; each warp owns 16
// keys of every staged chunk (CHUNK = 16 * W): S = Q K^T from ldmatrix'ed K
// rows (swizzled page rows, conflict-free), online softmax on the accumulator
// fragments (fp32, exp2), O += P V with P split into bf16 hi + lo halves
// (two MMAs: ~fp32 precision of the probabilities), V by ldmatrix.trans.
// The W per-warp (max, sum, O) states merge in fixed warp order at the end.
// Same staging / PDL structure as attention_block. ~10x fewer instructions
// than the CUDA-core loop (which issue-bound the decode step).
// ---------------------------------------------------------------------------
template <int W, int CHUNK, class Dep>
__device__ __forceinline__ void attention_block_mma(int blk_idx, int kh, const ArStepDev& s,
                                                    const __nv_bfloat16* __restrict__ q, int n_heads, int n_kv,
                                                    int layer, int n_layers, const __nv_bfloat16* __restrict__ kv,
                                                    __nv_bfloat16* __restrict__ out, float scale,
                                                    AttnSmem<W, CHUNK>& sm, Dep dep,
                                                    unsigned long long* tr = nullptr) {
  static_assert(CHUNK == 16 * W, "one 16-key MMA slab per warp per chunk");
  constexpr int HD = kHeadDim;
  constexpr uint32_t PAGE_BYTES = kPageTokens * HD * 2;
  constexpr int kPagesPerChunk = CHUNK / kPageTokens;
  const AttnBlockDesc blk = s.attn_blocks[blk_idx];
  const ArEntryDesc ed = s.entries[blk.entry];
  const int group = n_heads / n_kv;
  const int nq = blk.ntok * group;  // <= 16
  const int kend = ed.pos0 + blk.tok0 + blk.ntok;
  const int n_chunks = (kend + CHUNK - 1) / CHUNK;
  const int warp = warp_id(), lane = lane_id();
  const int g = lane >> 2, t4 = lane & 3;
  // split-KV: this CTA owns chunks [c_lo, c_hi) of the block's keys
  const int parts = attn_split_parts(blk.split), part = attn_split_part(blk.split);
  const bool split = parts > 1;
  const int per = split ? (n_chunks + parts - 1) / parts : n_chunks;
  const int c_lo = split ? part * per : 0;
  const int c_hi = split ? min(n_chunks, c_lo + per) : n_chunks;

  if (threadIdx.x == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    fence_barrier_init();
  }
  auto issue = [&](int c, int buf, int part) {
    const int first = c * kPagesPerChunk;
    const int keys = min(CHUNK, kend - c * CHUNK);
    const int np = (keys + kPageTokens - 1) / kPageTokens;
    if (part == 0) mbar_expect_tx(&sm.bar[buf], 2u * PAGE_BYTES * np);
    for (int i = 0; i < np; ++i) {
      const bool history = (first + i + 1) * kPageTokens <= ed.pos0;
      if (history != (part == 0)) continue;
      const int page = s.page_table[ed.slot * s.max_pages + first + i];
      const size_t base = (((size_t)page * n_layers + layer) * 2) * n_kv;
      bulk_load(sm.k[buf] + i * kPageTokens * HD, kv + (base + kh) * kPageTokens * HD, PAGE_BYTES, &sm.bar[buf]);
      bulk_load(sm.v[buf] + i * kPageTokens * HD, kv + (base + n_kv + kh) * kPageTokens * HD, PAGE_BYTES,
                &sm.bar[buf]);
    }
  };
  if (threadIdx.x == 0) {
    if (tr) tr[0] = globaltimer();
    issue(c_lo, 0, 0);
    if (c_lo + 1 < c_hi) issue(c_lo + 1, 1, 0);
  }
  dep();
  if (tr && threadIdx.x == 0) tr[1] = globaltimer();
  if (threadIdx.x == 0) {
    issue(c_lo, 0, 1);
    if (c_lo + 1 < c_hi) issue(c_lo + 1, 1, 1);
  }
  __syncthreads();  // barrier init visible before any wait

  // Q fragments (rows g, g + 8; 8 k-steps of 16 head dims) straight from the bf16 q rows
  uint32_t qa[8][4];
  int qpos_lo = -1, qpos_hi = -1;  // causal limit of rows g and g + 8 (-1: padding row)
  {
    const __nv_bfloat16* r_lo = nullptr;
    const __nv_bfloat16* r_hi = nullptr;
    if (g < nq) {
      r_lo = q + (size_t)(ed.row0 + blk.tok0 + g / group) * n_heads * HD + (kh * group + g % group) * HD;
      qpos_lo = ed.pos0 + blk.tok0 + g / group;
    }
    if (g + 8 < nq) {
      r_hi = q + (size_t)(ed.row0 + blk.tok0 + (g + 8) / group) * n_heads * HD + (kh * group + (g + 8) % group) * HD;
      qpos_hi = ed.pos0 + blk.tok0 + (g + 8) / group;
    }
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int d0 = ks * 16 + 2 * t4;
      qa[ks][0] = r_lo ? *reinterpret_cast<const uint32_t*>(r_lo + d0) : 0u;
      qa[ks][1] = r_hi ? *reinterpret_cast<const uint32_t*>(r_hi + d0) : 0u;
      qa[ks][2] = r_lo ? *reinterpret_cast<const uint32_t*>(r_lo + d0 + 8) : 0u;
      qa[ks][3] = r_hi ? *reinterpret_cast<const uint32_t*>(r_hi + d0 + 8) : 0u;
    }
  }
  if (tr && threadIdx.x == 0) tr[2] = globaltimer();
  const float sl2 = scale * 1.4426950408889634f;  // scores in log2 units
  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;
  float o[16][4];
#pragma unroll
  for (int nd = 0; nd < 16; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.f;

  for (int c = c_lo; c < c_hi; ++c) {
    const int buf = (c - c_lo) & 1;
    mbar_wait(&sm.bar[buf], ((c - c_lo) >> 1) & 1);
    if (tr && c == c_lo && threadIdx.x == 0) tr[3] = globaltimer();
    const int k0 = c * CHUNK + warp * 16;  // this warp's first key
    // warp-uniform skip: no key of the slab is visible to any row of the block
    const int blk_qmax = ed.pos0 + blk.tok0 + blk.ntok - 1;
    if (k0 <= blk_qmax) {
      const uint32_t kb = smem_addr(sm.k[buf]), vb = smem_addr(sm.v[buf]);
      // ---- S = Q K^T (16 x 16 keys) ----
      float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      {
        // ldmatrix x4: matrices (keys 0-7 | 8-15) x (dims lo 8 | hi 8) of k-step ks
        const int mi = lane >> 3, ri = lane & 7;
        const int key = warp * 16 + (mi >> 1) * 8 + ri;  // row within the chunk buffer
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const int chunk = ks * 2 + (mi & 1);
          uint32_t b[4];
          ldsm_x4(b, kb + (uint32_t)((key * HD + kv_swz(chunk, key) * 8) * 2));
          mma_bf16_16816(sc[0], qa[ks], b[0], b[1]);
          mma_bf16_16816(sc[1], qa[ks], b[2], b[3]);
        }
      }
      // ---- causal mask + online softmax (rows g / g + 8; 4 lanes per row) ----
      float mx_lo = -INFINITY, mx_hi = -INFINITY;
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int key = k0 + nb * 8 + 2 * t4 + e;
          sc[nb][e] = key <= qpos_lo ? sc[nb][e] * sl2 : -INFINITY;
          sc[nb][2 + e] = key <= qpos_hi ? sc[nb][2 + e] * sl2 : -INFINITY;
          mx_lo = fmaxf(mx_lo, sc[nb][e]);
          mx_hi = fmaxf(mx_hi, sc[nb][2 + e]);
        }
      mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
      mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
      mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
      mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
      const float mn_lo = fmaxf(m_lo, mx_lo), mn_hi = fmaxf(m_hi, mx_hi);
      const float cr_lo = mn_lo == -INFINITY ? 1.f : exp2f(m_lo - mn_lo);
      const float cr_hi = mn_hi == -INFINITY ? 1.f : exp2f(m_hi - mn_hi);
      float ps_lo = 0.f, ps_hi = 0.f;
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          sc[nb][e] = mn_lo == -INFINITY ? 0.f : exp2f(sc[nb][e] - mn_lo);
          sc[nb][2 + e] = mn_hi == -INFINITY ? 0.f : exp2f(sc[nb][2 + e] - mn_hi);
          ps_lo += sc[nb][e];
          ps_hi += sc[nb][2 + e];
        }
      ps_lo += __shfl_xor_sync(0xffffffffu, ps_lo, 1);
      ps_lo += __shfl_xor_sync(0xffffffffu, ps_lo, 2);
      ps_hi += __shfl_xor_sync(0xffffffffu, ps_hi, 1);
      ps_hi += __shfl_xor_sync(0xffffffffu, ps_hi, 2);
      l_lo = l_lo * cr_lo + ps_lo;
      l_hi = l_hi * cr_hi + ps_hi;
      m_lo = mn_lo;
      m_hi = mn_hi;
#pragma unroll
      for (int nd = 0; nd < 16; ++nd) {
        o[nd][0] *= cr_lo, o[nd][1] *= cr_lo;
        o[nd][2] *= cr_hi, o[nd][3] *= cr_hi;
      }
      // ---- O += P V: P as bf16 hi + lo A fragments ----
      uint32_t ph[4], pl[4];
      {
        const float p[4][2] = {{sc[0][0], sc[0][1]}, {sc[0][2], sc[0][3]}, {sc[1][0], sc[1][1]}, {sc[1][2], sc[1][3]}};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const __nv_bfloat162 h = __floats2bfloat162_rn(p[r][0], p[r][1]);
          const float2 hf = __bfloat1622float2(h);
          ph[r] = *reinterpret_cast<const uint32_t*>(&h);
          pl[r] = pack_bf16x2(p[r][0] - hf.x, p[r][1] - hf.y);
        }
      }
      {
        // ldmatrix.trans x4: (keys 0-7 | 8-15) x (dims nd*8 | (nd+1)*8)
        const int mi = lane >> 3, ri = lane & 7;
        const int vk = blk_qmax + 1 - k0;  // valid keys of the slab (>= 1)
        auto pair_mask = [&](int k) {
          return (k < vk ? 0x0000ffffu : 0u) | (k + 1 < vk ? 0xffff0000u : 0u);
        };
        const uint32_t vm_lo = pair_mask(2 * t4), vm_hi = pair_mask(8 + 2 * t4);
        const int key = warp * 16 + (mi & 1) * 8 + ri;
#pragma unroll
        for (int nd = 0; nd < 16; nd += 2) {
          const int chunk = nd + (mi >> 1);
          uint32_t b[4];
          ldsm_x4_t(b, vb + (uint32_t)((key * HD + kv_swz(chunk, key) * 8) * 2));
          // keys past the context hold stale smem / page bytes: P is 0 there,
          // and V must be too (0 * NaN)
          b[0] &= vm_lo, b[2] &= vm_lo;
          b[1] &= vm_hi, b[3] &= vm_hi;
          mma_bf16_16816(o[nd], ph, b[0], b[1]);
          mma_bf16_16816(o[nd], pl, b[0], b[1]);
          mma_bf16_16816(o[nd + 1], ph, b[2], b[3]);
          mma_bf16_16816(o[nd + 1], pl, b[2], b[3]);
        }
      }
    }
    __syncthreads();  // every warp is done with `buf`
    if (threadIdx.x == 0 && c + 2 < c_hi) {
      issue(c + 2, buf, 0);
      issue(c + 2, buf, 1);
    }
  }
  if (tr && threadIdx.x == 0) tr[4] = globaltimer();
  // ---- merge the W warp states in fixed warp order (K/V buffers are free) ----
  float* mo = reinterpret_cast<float*>(&sm.k[0][0]);  // [W][16][HD]
  float* ml = reinterpret_cast<float*>(&sm.v[0][0]);  // [W][16][2]
  if (t4 == 0) {
    ml[(warp * 16 + g) * 2 + 0] = m_lo;
    ml[(warp * 16 + g) * 2 + 1] = l_lo;
    ml[(warp * 16 + g + 8) * 2 + 0] = m_hi;
    ml[(warp * 16 + g + 8) * 2 + 1] = l_hi;
  }
#pragma unroll
  for (int nd = 0; nd < 16; ++nd) {
    const int d0 = nd * 8 + 2 * t4;
    if (g < nq) *reinterpret_cast<float2*>(mo + (warp * 16 + g) * HD + d0) = make_float2(o[nd][0], o[nd][1]);
    if (g + 8 < nq)
      *reinterpret_cast<float2*>(mo + (warp * 16 + g + 8) * HD + d0) = make_float2(o[nd][2], o[nd][3]);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nq * (HD / 2); idx += W * 32) {
    const int r = idx / (HD / 2), d0 = (idx % (HD / 2)) * 2;
    float mt = -INFINITY;
#pragma unroll
    for (int w = 0; w < W; ++w) mt = fmaxf(mt, ml[(w * 16 + r) * 2]);
    float lt = 0.f, a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const float mw = ml[(w * 16 + r) * 2];
      const float f = mw == -INFINITY ? 0.f : exp2f(mw - mt);
      lt += ml[(w * 16 + r) * 2 + 1] * f;
      const float2 v = *reinterpret_cast<const float2*>(mo + (w * 16 + r) * HD + d0);
      a0 += v.x * f;
      a1 += v.y * f;
    }
    if (split) {  // this part's unnormalised state -> scratch; the last part merges
      float* sp = s.split_part +
                  ((((size_t)attn_split_group(blk.split) * n_kv + kh) * kAttnMaxParts + part) * 16 + r) * (HD + 2);
      *reinterpret_cast<float2*>(sp + d0) = make_float2(a0, a1);
      if (d0 == 0) sp[HD] = mt, sp[HD + 1] = lt;
      continue;
    }
    const float inv = 1.f / lt;
    const int tok = blk.tok0 + r / group, hq = kh * group + r % group;
    *reinterpret_cast<__nv_bfloat162*>(out + (size_t)(ed.row0 + tok) * n_heads * HD + hq * HD + d0) =
        __floats2bfloat162_rn(a0 * inv, a1 * inv);
  }
  if (split) {
    // last-arriver merge in FIXED part order (bit-identical whichever part
    // finishes last); P depends only on the sequence's own context length,
    // so a sequence's output does not depend on the rest of the batch
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    int* cnt = s.split_cnt + (size_t)attn_split_group(blk.split) * n_kv + kh;
    if (threadIdx.x == 0) {
      const int old = atomicAdd(cnt, 1);
      s_last = old == parts - 1;
      if (s_last) *cnt = 0;  // ready for the next launch (every part has arrived)
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      const float* base =
          s.split_part + (((size_t)attn_split_group(blk.split) * n_kv + kh) * kAttnMaxParts) * 16 * (HD + 2);
      for (int idx = threadIdx.x; idx < nq * (HD / 2); idx += W * 32) {
        const int r = idx / (HD / 2), d0 = (idx % (HD / 2)) * 2;
        float mt = -INFINITY;
        for (int pp = 0; pp < parts; ++pp) mt = fmaxf(mt, __ldcg(base + ((size_t)pp * 16 + r) * (HD + 2) + HD));
        float lt = 0.f, a0 = 0.f, a1 = 0.f;
        for (int pp = 0; pp < parts; ++pp) {
          const float* sp = base + ((size_t)pp * 16 + r) * (HD + 2);
          const float mp = __ldcg(sp + HD);
          const float f = mp == -INFINITY ? 0.f : exp2f(mp - mt);
          lt += __ldcg(sp + HD + 1) * f;
          const float2 v = __ldcg(reinterpret_cast<const float2*>(sp + d0));
          a0 += v.x * f;
          a1 += v.y * f;
        }
        const float inv = 1.f / lt;
        const int tok = blk.tok0 + r / group, hq = kh * group + r % group;
        *reinterpret_cast<__nv_bfloat162*>(out + (size_t)(ed.row0 + tok) * n_heads * HD + hq * HD + d0) =
            __floats2bfloat162_rn(a0 * inv, a1 * inv);
      }
    }
  }
  if (tr && threadIdx.x == 0) tr[5] = globaltimer();
}

// ---------------------------------------------------------------------------
// Final norm of DECODE rows -> compact hidden rows (+ hidden ring for the
// thinker, row `out_index` of the sequence's slot).
// ---------------------------------------------------------------------------
template <class Dep>
__device__ __forceinline__ void final_gather_row(int di, const ArStepDev& s, const float* __restrict__ x, int d,
                                                 float eps, __nv_bfloat16* __restrict__ hout,
                                                 __nv_bfloat16* __restrict__ ring, int ring_rows, float* red,
                                                 Dep dep) {
  dep();
  const int e = s.dec_entries[di];
  const ArEntryDesc ed = s.entries[e];
  const float* xr = x + (size_t)ed.row0 * d;  // decode entries have exactly one row
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss += xr[i] * xr[i];
  const float tot = block_sum(ss, red);
  const float inv = rsqrtf(tot / d + eps);
  __nv_bfloat16* h = hout + (size_t)di * d;
  __nv_bfloat16* rg = ring ? ring + ((size_t)ed.slot * ring_rows + ed.out_index) * d : nullptr;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const __nv_bfloat16 v = f2bf(xr[i] * inv);
    h[i] = v;
    if (rg) rg[i] = v;
  }
}

// Greedy id over [lo, hi) of the logits row; ties -> lowest id. Also the
// top-2 margin used by the teacher-forced parity rule.
// One warp (lanes 0-31 of the block) per row.
template <class Dep>
__device__ __forceinline__ void argmax_row(int r, const float* __restrict__ logits, int ld, int lo, int hi,
                                           int* __restrict__ tok_out, float* __restrict__ margin_out, Dep dep) {
  dep();
  if (threadIdx.x >= 32) return;
  const float* row = logits + (size_t)r * ld;
  float b1 = -INFINITY, b2 = -INFINITY;
  int i1 = 0x7fffffff;
  for (int i = lo + threadIdx.x; i < hi; i += 32) {
    const float v = row[i];
    if (v > b1 || (v == b1 && i < i1)) {
      b2 = b1;
      b1 = v;
      i1 = i;
    } else if (v > b2) {
      b2 = v;
    }
  }
  // warp merge (blockDim == 32)
  for (int o = 16; o > 0; o >>= 1) {
    const float ob1 = __shfl_xor_sync(0xffffffffu, b1, o);
    const float ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
    const int oi1 = __shfl_xor_sync(0xffffffffu, i1, o);
    if (ob1 > b1 || (ob1 == b1 && oi1 < i1)) {
      b2 = fmaxf(b1, ob2);
      b1 = ob1;
      i1 = oi1;
    } else {
      b2 = fmaxf(b2, ob1);
    }
  }
  if (threadIdx.x == 0) {
    tok_out[r] = i1;
    margin_out[r] = b1 - b2;
  }
}

// ---------------------------------------------------------------------------
// Top-k sampler (north star: "warp-shuffle argmax/top-k sampler"). One warp
// per decode row; the row's logits live in registers (<= 8 per lane, V <=
// 256). top_k <= 1 is the greedy argmax above (the reference's token_of is
// greedy, reference_pipeline.hpp:34). Otherwise the k largest logits are
// extracted by k warp-argmax rounds, softmax-weighted (temperature 1), and
// one is drawn with u = sample_hash(seed, request key, emitted index): a pure
// function of the request and position, so a recompute-preempted sequence
// (ar_engine.hpp:229-257) redraws the same token and sampling stays
// batch-invariant. Ties break to the lowest id; the top-2 margin is reported
// as in the greedy path.
constexpr int kSampleMaxK = 32;
constexpr int kSamplePerLane = 8;  // V <= 256

template <class Dep>
__device__ __forceinline__ void sample_row(int r, const ArStepDev& s, const float* __restrict__ logits, int ld,
                                           int lo, int hi, int top_k, uint64_t seed,
                                           int* __restrict__ tok_out, float* __restrict__ margin_out, Dep dep) {
  if (top_k <= 1) {
    argmax_row(r, logits, ld, lo, hi, tok_out, margin_out, dep);
    return;
  }
  dep();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const float* row = logits + (size_t)r * ld;
  float v[kSamplePerLane];
#pragma unroll
  for (int j = 0; j < kSamplePerLane; ++j) {
    const int i = lo + lane + 32 * j;
    v[j] = i < hi ? row[i] : -INFINITY;
  }
  const int k = min(min(top_k, kSampleMaxK), hi - lo);
  float top_v = -INFINITY;  // lane t keeps the t-th largest (t < k)
  int top_i = 0x7fffffff;
  for (int t = 0; t < k; ++t) {
    float b = -INFINITY;
    int bi = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < kSamplePerLane; ++j) {
      const int i = lo + lane + 32 * j;
      if (v[j] > b || (v[j] == b && i < bi)) b = v[j], bi = i;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, b, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > b || (ob == b && oi < bi)) b = ob, bi = oi;
    }
    if (lane == t) top_v = b, top_i = bi;
#pragma unroll
    for (int j = 0; j < kSamplePerLane; ++j)
      if (lo + lane + 32 * j == bi) v[j] = -INFINITY;
  }
  const float vmax = __shfl_sync(0xffffffffu, top_v, 0);
  const float p = lane < k ? __expf(top_v - vmax) : 0.f;
  // inclusive prefix sum in lane order (= descending logit order)
  float c = p;
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, c, o);
    if (lane >= o) c += y;
  }
  const float total = __shfl_sync(0xffffffffu, c, 31);
  const int e = s.dec_entries[r];
  const ArEntryDesc ed = s.entries[e];
  const uint64_t h = sample_hash(seed, (uint32_t)ed.key, (uint32_t)ed.out_index);
  const float u = (float)(h >> 40) * (1.0f / 16777216.0f) * total;
  const unsigned hit = __ballot_sync(0xffffffffu, lane < k && c > u);
  const int pick = hit ? __ffs(hit) - 1 : k - 1;
  const int tok = __shfl_sync(0xffffffffu, top_i, pick);
  const float m2 = __shfl_sync(0xffffffffu, top_v, 1);
  if (lane == 0) {
    tok_out[r] = tok;
    margin_out[r] = vmax - m2;
  }
}

}  // namespace omni_dev
