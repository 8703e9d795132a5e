// K6': the whole DiT denoise iteration (T Euler steps x L layers) as ONE
// persistent dataflow kernel.
//
// Replaces the per-job denoise() of diffusion_engine.hpp:28-43 (called at
// :98). The model is token-local: the S = 16 sample rows of a conditioning
// token only ever interact with each other (attention is among a token's own
// samples), so a tile of 128 rows (8 tokens) can run through the iteration
// independently of every other tile. The kernel exploits that instead of
// global barriers:
//
//  * work = a fixed, totally ordered list of ITEMS, phase-major:
//    (Euler step, phase, row tile, item-in-phase). Phases per step:
//    IN-proj, then per layer LN1 | QKV | ATTN | O (+adaLN gate, residual) |
//    LN2 | MLP-up (+GELU) | MLP-down (+gate, residual; split-K 2), then the
//    final LN and OUT-proj (+Euler update, int32 samples on the last step);
//  * every CTA (one per SM, persistent) takes the next item index from a
//    global counter; an item of phase p on row tile r waits only until
//    progress[r] (units of that tile completed so far, monotone) covers all
//    earlier phases of the tile. Items only wait on smaller indices, all
//    held by resident CTAs, so the schedule cannot deadlock, and tiles at
//    different phases overlap freely (no grid-wide barrier, no launch gaps);
//  * GEMM items: 128 output features x 128 rows, swap-AB tcgen05 kind::f16
//    (weights = MMA A / TMEM lanes, rows = MMA B), TMA (SWIZZLE_128B) into a
//    4-deep ring, one elected thread issues the MMAs, accumulators
//    double-buffered in TMEM (2 x 128 columns) so an item's epilogue overlaps
//    the next mainloop; weight tiles are requested BEFORE the dependency wait;
//  * epilogue thread = one output feature, so each warp store covers one
//    row's 32 consecutive features (one 64 / 128-byte line): TMEM ->
//    registers -> global, the residual update h += gate * acc as
//    red.global.add.f32 (each element receives exactly one add per phase:
//    deterministic, no read of h). Measured: shared-memory staging + TMA
//    stores stall on the mainloop's smem traffic, and row-per-thread 16-byte
//    stores touch 32 lines per warp instruction -- both 2-4x slower;
//  * MLP-down (K = 4 d) is split in two K halves: the first arriving half
//    writes its partial, the second adds it to its own TMEM accumulator
//    (a + b is commutative: bit-identical whichever half arrives first);
//  * LN and attention items run on the four epilogue warps (same arithmetic
//    as the standalone kernels in dit_kernels.cu).
//
// Warp roles (320 threads): 0 = scheduler + TMA producer, 1 = MMA issuer,
// 2..9 = epilogue / LN / attention (TMEM lane quadrant = warp % 4; the two
// warps of a quadrant take alternate 16-row chunks of an item). Measured
// (profiles/r02_dit_fused_v7.txt): 128-row tiles halve every item's
// mainloop and the 8 epilogue warps halve its epilogue, which together set
// the per-layer latency of a row tile through the dependency chain.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>

#include "dit_fused.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace omni_dev {
namespace {

constexpr int kEpiWarps = 8;  // two warps per TMEM lane quadrant, each half of an item's 16-row chunks
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kThreadsF = 64 + kEpiThreads;
constexpr int kQ = 1;  // item ring depth: fetch item i+1 once item i started (deeper run-ahead
                       // strands short LN / attention items behind long GEMM items of the same CTA)
constexpr int kABytes = kDitFeat * 64 * 2;  // weight tile (128 features x 64 k)
static_assert(16 % kEpiWarps == 0, "LN rows per warp");

// Row-tile geometry: TR rows = TR / 16 tokens = MMA N (128 or 256).
template <int TR>
struct Tile {
  static constexpr int rows = TR, tok = TR / 16;
  static constexpr int chunks = TR / 16;                  // 16-row chunks (one token each) per item
  static constexpr int my_chunks = chunks / (kEpiWarps / 4);  // chunks per epilogue warp
  static constexpr int b_bytes = TR * 64 * 2;             // row tile (TR rows x 64 k)
  static constexpr int stage_bytes = kABytes + b_bytes;
  static constexpr int att_groups = tok / kEpiWarps;      // attention items per head (a warp per token)
  static constexpr uint32_t idesc = idesc_bf16_f32(kDitFeat, TR);
  static_assert(tok % kEpiWarps == 0 && chunks % 2 == 0, "attention groups / chunk halves");
};

enum Kind : int { K_IN = 0, K_LN1, K_QKV, K_ATT, K_O, K_LN2, K_UP, K_DOWN, K_LNF, K_OUT, K_END };

__device__ __forceinline__ bool is_gemm(int k) {
  return k == K_IN || k == K_QKV || k == K_O || k == K_UP || k == K_DOWN || k == K_OUT;
}

struct Item {
  int kind, layer, step, tp, r, j, idx;
};

struct PhaseInfo {
  int kind, layer, items, units;
};

// Phase ph of one Euler step (P = 3 + 7 L phases); items / units per row tile.
template <int TR>
__device__ __forceinline__ PhaseInfo phase_info(const DitFusedParams& p, int ph) {
  using T = Tile<TR>;
  const int nf = p.d / kDitFeat, P = 3 + 7 * p.L;
  if (ph == 0) return {K_IN, 0, nf, nf};
  if (ph == P - 2) return {K_LNF, 0, T::tok, T::tok};
  if (ph == P - 1) return {K_OUT, 0, 1, 1};
  const int l = (ph - 1) / 7;
  switch ((ph - 1) % 7) {
    case 0: return {K_LN1, l, T::tok, T::tok};
    case 1: return {K_QKV, l, 3 * nf, 3 * nf};
    case 2: return {K_ATT, l, p.H * T::att_groups, p.H * T::att_groups};  // (head, 8-token group)
    case 3: return {K_O, l, nf, nf};
    case 4: return {K_LN2, l, T::tok, T::tok};
    case 5: return {K_UP, l, p.ff / kDitFeat, p.ff / kDitFeat};
    default: return {K_DOWN, l, nf * p.down_split, nf};
  }
}

// Spin with relaxed loads (an acquire load compiles to LDG.STRONG + an L1
// invalidate per poll), then one acquire fence.
__device__ __forceinline__ void wait_ge(const int* ptr, int target) {
  int v;
  for (;;) {
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
    if (v >= target) break;
    __nanosleep(20);
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// gelu_tanh with one MUFU tanh.approx.f32 (|rel err| <= 2^-10.99 on tanh,
// below the bf16 rounding of the result): ~6 instructions per element -- the
// MLP-up epilogue was instruction-bound on the exp / divide form
__device__ __forceinline__ float gelu_fast(float x) {
  const float y = x * fmaf(0.0356774081f, x * x, 0.7978845608f);  // sqrt(2/pi) (x + 0.044715 x^3)
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(y));
  const float hx = 0.5f * x;
  return fmaf(hx, t, hx);
}
// 4x4 transpose inside each group of 4 lanes: lane 4g+k holds feature 4g+k
// of rows 0..3 on entry, and rows... on exit lane 4g+t holds row t of
// features 4g..4g+3 (two shfl_xor stages, selects only, no divergence).
__device__ __forceinline__ void tr4(float& a0, float& a1, float& a2, float& a3, int lane) {
  const bool b1 = lane & 2, b0 = lane & 1;
  float s0 = b1 ? a0 : a2, s1 = b1 ? a1 : a3;
  float r0 = __shfl_xor_sync(0xffffffffu, s0, 2), r1 = __shfl_xor_sync(0xffffffffu, s1, 2);
  if (b1) a0 = r0, a1 = r1;
  else a2 = r0, a3 = r1;
  s0 = b0 ? a0 : a1;
  s1 = b0 ? a2 : a3;
  r0 = __shfl_xor_sync(0xffffffffu, s0, 1);
  r1 = __shfl_xor_sync(0xffffffffu, s1, 1);
  if (b0) a0 = r0, a2 = r1;
  else a1 = r0, a3 = r1;
}
__device__ __forceinline__ void st_f4_cg(float* p, float a, float b, float c, float d) {
  __stcg(reinterpret_cast<float4*>(p), make_float4(a, b, c, d));
}
__device__ __forceinline__ void st_bf16x4(__nv_bfloat16* p, float a, float b, float c, float d) {
  *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16x2(a, b), pack_bf16x2(c, d));
}
__device__ __forceinline__ void ep_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory"); }

// a = bf16(LN(h) * (1 + scale) + shift) for NR consecutive rows of one token
// (one warp; the token's modulation rows preloaded), same arithmetic as
// dit_ln_mod_kernel. The two rows of a pair have their loads in flight together.
template <int PER, int NR>
__device__ __forceinline__ void ln_rows(const float* hr, bool mod, const float4 (&sc)[PER], const float4 (&sh)[PER],
                                         __nv_bfloat16* out_row, int lane) {
  constexpr int d = PER * 128;
#pragma unroll 1
  for (int q0 = 0; q0 < NR; q0 += 2) {
    float4 x[2][PER];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int k = 0; k < PER; ++k)
        x[q][k] = __ldcg(reinterpret_cast<const float4*>(hr + (size_t)(q0 + q) * d) + lane + 32 * k);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float sum = 0.f;
#pragma unroll
      for (int k = 0; k < PER; ++k) sum += (x[q][k].x + x[q][k].y) + (x[q][k].z + x[q][k].w);
      const float mean = warp_sum(sum) / d;
      float var = 0.f;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const float a0 = x[q][k].x - mean, a1 = x[q][k].y - mean, a2 = x[q][k].z - mean, a3 = x[q][k].w - mean;
        var += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
      }
      const float inv = rsqrtf(warp_sum(var) / d + 1e-6f);
      uint2* o = reinterpret_cast<uint2*>(out_row + (size_t)(q0 + q) * d);
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        float y[4] = {(x[q][k].x - mean) * inv, (x[q][k].y - mean) * inv, (x[q][k].z - mean) * inv,
                      (x[q][k].w - mean) * inv};
        if (mod) {
          y[0] = y[0] * (1.f + sc[k].x) + sh[k].x;
          y[1] = y[1] * (1.f + sc[k].y) + sh[k].y;
          y[2] = y[2] * (1.f + sc[k].z) + sh[k].z;
          y[3] = y[3] * (1.f + sc[k].w) + sh[k].w;
        }
        const __nv_bfloat162 lo = __floats2bfloat162_rn(y[0], y[1]), hi = __floats2bfloat162_rn(y[2], y[3]);
        o[lane + 32 * k] =
            make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
      }
    }
  }
}

__device__ __forceinline__ uint32_t ldcg_u32(const __nv_bfloat16* p) {
  return __ldcg(reinterpret_cast<const unsigned int*>(p));
}

// Attention among the 16 samples of token `tok`, head h (one warp), all on
// the warp MMA (mma.sync m16n8k16): S = Q K^T, softmax on the S accumulators,
// O = P V with P kept in registers -- the S accumulator fragments ARE the A
// fragments of the PV product (rows = samples, k = keys), split into bf16 hi
// + lo halves (two MMAs: ~fp32 precision of the probabilities). Every global
// access is 16 bytes (24 loads + 8 stores per lane instead of 96 + 32 narrow
// ones, which made attention items ~10 us):
//  * Q / K: lane (g, t) loads 8 consecutive dims of rows g and g + 8; the head
//    dimension is consumed in a permuted order (the fragment's k slots 2t /
//    8 + 2t of k-step 2c + e take dims 32c + 8t + 4e + {0,1} / {2,3}),
//    identical for Q and K, so S is the same dot product;
//  * V: a 4x4 lane transpose (tr4) turns the quad's 16-byte row segments into
//    rows of 8x8 tiles, and movmatrix.trans into the PV B fragments;
//  * O: the transpose back turns the C fragments into 16-byte row segments.
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}
__device__ __forceinline__ void tr4u(uint32_t (&a)[4], int lane) {
  float f0 = __uint_as_float(a[0]), f1 = __uint_as_float(a[1]), f2 = __uint_as_float(a[2]),
        f3 = __uint_as_float(a[3]);
  tr4(f0, f1, f2, f3, lane);
  a[0] = __float_as_uint(f0), a[1] = __float_as_uint(f1), a[2] = __float_as_uint(f2), a[3] = __float_as_uint(f3);
}
__device__ __forceinline__ void attn_token_head(const __nv_bfloat16* qkv, int tok, int h, int d,
                                                __nv_bfloat16* out, int lane) {
  constexpr int S = 16, HD = 128, NC = HD / 32;
  const int g = lane >> 2, t = lane & 3;
  const size_t ld = 3 * (size_t)d;
  const __nv_bfloat16* Q = qkv + (size_t)tok * S * ld + h * HD + 8 * t;
  const __nv_bfloat16* K = Q + d;
  const __nv_bfloat16* V = Q + 2 * d;
  uint4 q0[NC], q1[NC], k0[NC], k1[NC], v0[NC], v1[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    q0[c] = __ldcg(reinterpret_cast<const uint4*>(Q + (size_t)g * ld + 32 * c));
    q1[c] = __ldcg(reinterpret_cast<const uint4*>(Q + (size_t)(g + 8) * ld + 32 * c));
    k0[c] = __ldcg(reinterpret_cast<const uint4*>(K + (size_t)g * ld + 32 * c));
    k1[c] = __ldcg(reinterpret_cast<const uint4*>(K + (size_t)(g + 8) * ld + 32 * c));
    v0[c] = __ldcg(reinterpret_cast<const uint4*>(V + (size_t)g * ld + 32 * c));
    v1[c] = __ldcg(reinterpret_cast<const uint4*>(V + (size_t)(g + 8) * ld + 32 * c));
  }
  float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const uint32_t qa0[4] = {q0[c].x, q1[c].x, q0[c].y, q1[c].y}, qa1[4] = {q0[c].z, q1[c].z, q0[c].w, q1[c].w};
    mma_bf16_16816(c0, qa0, k0[c].x, k0[c].y);
    mma_bf16_16816(c1, qa0, k1[c].x, k1[c].y);
    mma_bf16_16816(c0, qa1, k0[c].z, k0[c].w);
    mma_bf16_16816(c1, qa1, k1[c].z, k1[c].w);
  }
  const float scale = rsqrtf((float)HD);
  // rows g (c*[0..1]) and g + 8 (c*[2..3]); keys 2t, 2t + 1 (c0) and 8 + 2t, 9 + 2t (c1)
  float r0[4] = {c0[0] * scale, c0[1] * scale, c1[0] * scale, c1[1] * scale};
  float r1[4] = {c0[2] * scale, c0[3] * scale, c1[2] * scale, c1[3] * scale};
  float m0 = fmaxf(fmaxf(r0[0], r0[1]), fmaxf(r0[2], r0[3]));
  float m1 = fmaxf(fmaxf(r1[0], r1[1]), fmaxf(r1[2], r1[3]));
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
    m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
  }
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    r0[i] = expf(r0[i] - m0);
    r1[i] = expf(r1[i] - m1);
    s0 += r0[i];
    s1 += r1[i];
  }
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  const float i0 = 1.f / s0, i1 = 1.f / s1;
  // A fragments of P (m16 x k16): {row g keys 2t..}, {row g+8 keys 2t..}, {row g keys 8+2t..}, {row g+8 keys 8+2t..}
  const float pv[4][2] = {{r0[0] * i0, r0[1] * i0}, {r1[0] * i1, r1[1] * i1}, {r0[2] * i0, r0[3] * i0},
                          {r1[2] * i1, r1[3] * i1}};
  uint32_t ph[4], pl[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const __nv_bfloat162 hb = __floats2bfloat162_rn(pv[r][0], pv[r][1]);
    const float2 hf = __bfloat1622float2(hb);
    ph[r] = *reinterpret_cast<const uint32_t*>(&hb);
    pl[r] = pack_bf16x2(pv[r][0] - hf.x, pv[r][1] - hf.y);
  }
  __nv_bfloat16* orow0 = out + ((size_t)tok * S + g) * d + h * HD + 8 * t;
  __nv_bfloat16* orow1 = orow0 + (size_t)8 * d;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    // lane (g, t) holds dims 32c + 8t .. +7 of key rows g / g + 8 = row g of
    // 8x8 tile 4c + t; after the transpose: u32 t of row g of tiles 4c .. 4c+3
    uint32_t a[4] = {v0[c].x, v0[c].y, v0[c].z, v0[c].w}, b[4] = {v1[c].x, v1[c].y, v1[c].z, v1[c].w};
    tr4u(a, lane);
    tr4u(b, lane);
    uint32_t o0[4], o1[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // tile 4c + u: dims 32c + 8u .. +7
      const uint32_t bb0 = movmatrix_t(a[u]), bb1 = movmatrix_t(b[u]);  // (keys 2t.., dim g) / (keys 8+2t..)
      float o[4] = {0.f, 0.f, 0.f, 0.f};
      mma_bf16_16816(o, ph, bb0, bb1);
      mma_bf16_16816(o, pl, bb0, bb1);
      o0[u] = pack_bf16x2(o[0], o[1]);  // row g, dims 32c + 8u + 2t, +1
      o1[u] = pack_bf16x2(o[2], o[3]);  // row g + 8
    }
    tr4u(o0, lane);  // -> lane t: row g, dims 32c + 8t .. +7
    tr4u(o1, lane);
    *reinterpret_cast<uint4*>(orow0 + 32 * c) = make_uint4(o0[0], o0[1], o0[2], o0[3]);
    *reinterpret_cast<uint4*>(orow1 + 32 * c) = make_uint4(o1[0], o1[1], o1[2], o1[3]);
  }
}

// The epilogue of one GEMM item for one kind. MLP-down K parts meet in a
// fixed binary tree of commutative two-way sums, (p0 + p1) + (p2 + p3), so
// the result does not depend on which part arrives first. MODE: 0 plain;
// 1 write my partial to `dst` (first of a pair); 2 final: gate * (acc + s1)
// (split 2); 3 pair sum acc + s1 to `dst` (first pair to finish, split 4);
// 4 final: gate * ((acc + s1) + s2) (split 4). Each chunk = 16 rows (one
// token) x this warp's 32 features; after a 4x4 lane-group transpose (tr4)
// lane 4g+t owns row 4m+t, features fw .. fw+3 of group m, so every store is
// 8 / 16 bytes per thread (4x fewer store instructions than one feature per
// thread). aux: IN pos_emb[sample][own feature]; O / DOWN the adaLN gate of
// token c (rotated one per chunk).
template <int TR, int KIND, int MODE>
__device__ __forceinline__ void epi_chunks(const DitFusedParams& p, uint32_t ta, int row0, int ft, const float* s1b,
                                           const float* s2b, float* dstb, int quad, int half, int lane,
                                           float (&aux)[16], int step) {
  constexpr bool kGated = KIND == K_O || KIND == K_DOWN;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int fw = ft * kDitFeat + quad * 32 + 4 * g4;  // first of my 4 features after the transpose
  const int d = p.d;
  if (KIND == K_OUT && quad * 32 >= p.C) return;  // OUT: the C channels are the first C lanes
  constexpr int kChunks = Tile<TR>::chunks, kMyChunks = Tile<TR>::my_chunks;
  const int off4 = quad * 32 + 4 * g4;  // my 4 features within the 128-feature partial tile
  const float* s1 = s1b + off4;
  const float* s2 = s2b + off4;
  float* dst4 = dstb + off4;
  // side inputs (x / partial sums) of chunk cc, my 4 rows 4m + t4
  // (post-transpose layout); the next chunk's are in flight
  auto load_side = [&](int cc, float4(&dst)[4], float4(&dst2)[4]) {
    if constexpr (KIND == K_OUT)
#pragma unroll
      for (int m = 0; m < 4; ++m)
        dst[m] = __ldcg(reinterpret_cast<const float4*>(p.x + (size_t)(row0 + cc * 16 + 4 * m + t4) * p.C + fw));
    if constexpr (MODE >= 2)
#pragma unroll
      for (int m = 0; m < 4; ++m)
        dst[m] = __ldcg(reinterpret_cast<const float4*>(s1 + (size_t)(cc * 16 + 4 * m + t4) * kDitFeat));
    if constexpr (MODE == 4)
#pragma unroll
      for (int m = 0; m < 4; ++m)
        dst2[m] = __ldcg(reinterpret_cast<const float4*>(s2 + (size_t)(cc * 16 + 4 * m + t4) * kDitFeat));
  };
  // this warp's chunks: c = half, half + 2, ... (its quadrant partner takes the
  // others); the next chunk's TMEM load and side inputs are in flight while
  // this one is processed
  float4 nx[4] = {}, nx2[4] = {};
  load_side(half, nx, nx2);
  uint32_t tr[16];
  tmem_ld16_issue(ta + half * 16, tr);
#pragma unroll 1
  for (int c = half; c < kChunks; c += 2) {
    float4 ld[4], ld2[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) ld[m] = nx[m], ld2[m] = nx2[m];
    if (c + 2 < kChunks) load_side(c + 2, nx, nx2);
    tmem_ld16_wait(tr);
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(tr[i]);
    if (c + 2 < kChunks) tmem_ld16_issue(ta + (c + 2) * 16, tr);
    const int rb = row0 + c * 16;  // rows of token row0 / 16 + c
    if constexpr (KIND == K_IN) {
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) v[jj] += aux[jj];
    } else if constexpr (KIND == K_UP) {
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) v[jj] = gelu_fast(v[jj]);
    } else if constexpr (kGated && MODE == 0) {
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) v[jj] *= aux[0];
    }
    float gq[4];  // MODE 2 / 4: the gates of my 4 post-transpose features
    if constexpr (MODE == 2 || MODE == 4)
#pragma unroll
      for (int i = 0; i < 4; ++i) gq[i] = __shfl_sync(0xffffffffu, aux[0], 4 * g4 + i);
#pragma unroll
    for (int m = 0; m < 4; ++m) tr4(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3], lane);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int row = rb + 4 * m + t4;
      const float* q = v + 4 * m;
      if constexpr (KIND == K_IN) {
        st_f4_cg(p.h + (size_t)row * d + fw, q[0], q[1], q[2], q[3]);
      } else if constexpr (KIND == K_QKV) {
        st_bf16x4(p.qkv + (size_t)row * 3 * d + fw, q[0], q[1], q[2], q[3]);
      } else if constexpr (KIND == K_UP) {
        st_bf16x4(p.u + (size_t)row * p.ff + fw, q[0], q[1], q[2], q[3]);
      } else if constexpr (KIND == K_OUT) {  // Euler update, int32 samples (channel 0) on the last step
        const float x[4] = {ld[m].x + p.dt * q[0], ld[m].y + p.dt * q[1], ld[m].z + p.dt * q[2], ld[m].w + p.dt * q[3]};
        st_f4_cg(p.x + (size_t)row * p.C + fw, x[0], x[1], x[2], x[3]);
        st_bf16x4(p.xb + (size_t)row * p.C + fw, x[0], x[1], x[2], x[3]);
        if (fw == 0 && step == p.T - 1) {
          float sq = rintf(p.sample_scale * x[0]);
          sq = fminf(fmaxf(sq, -64.f), 63.f);
          p.samples[row] = (int32_t)sq;
        }
      } else if constexpr (MODE == 1) {
        st_f4_cg(dst4 + (size_t)(c * 16 + 4 * m + t4) * kDitFeat, q[0], q[1], q[2], q[3]);
      } else if constexpr (MODE == 3) {
        st_f4_cg(dst4 + (size_t)(c * 16 + 4 * m + t4) * kDitFeat, q[0] + ld[m].x, q[1] + ld[m].y, q[2] + ld[m].z,
                 q[3] + ld[m].w);
      } else if constexpr (MODE == 2) {
        red_add_v4(p.h + (size_t)row * d + fw, gq[0] * (q[0] + ld[m].x), gq[1] * (q[1] + ld[m].y),
                   gq[2] * (q[2] + ld[m].z), gq[3] * (q[3] + ld[m].w));
      } else if constexpr (MODE == 4) {
        red_add_v4(p.h + (size_t)row * d + fw, gq[0] * ((q[0] + ld[m].x) + ld2[m].x),
                   gq[1] * ((q[1] + ld[m].y) + ld2[m].y), gq[2] * ((q[2] + ld[m].z) + ld2[m].z),
                   gq[3] * ((q[3] + ld[m].w) + ld2[m].w));
      } else {
        red_add_v4(p.h + (size_t)row * d + fw, q[0], q[1], q[2], q[3]);
      }
    }
    if constexpr (kGated)
#pragma unroll
      for (int k = 0; k < kMyChunks - 1; ++k) aux[k] = aux[k + 1];  // static indices: aux stays in registers
  }
}

struct Smem {
  uint64_t full[8], empty[8];
  uint64_t acc_full[2], acc_empty[2];
  uint64_t q_full[kQ], q_empty[kQ];
  Item ring[kQ];
  uint32_t tmem;
  int mode;
  int item_start[kDitMaxPhases + 1];  // global item index where (step, phase) tp starts
  int unit_cum[kDitMaxPhases + 1];    // per-tile units completed before tp
};

template <int PER, int STAGES, int TR>
__global__ void __launch_bounds__(kThreadsF, 1) dit_fused_kernel(const __grid_constant__ DitFusedParams p) {
  static_assert(STAGES <= 8, "barrier slots");
  using Tl = Tile<TR>;
  constexpr int kBBytes = Tl::b_bytes, kStageBytes = Tl::stage_bytes;
  constexpr uint32_t kIdesc = Tl::idesc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + STAGES * kABytes;
  Smem& sm = *reinterpret_cast<Smem*>(base + STAGES * kStageBytes);
  const int warp = warp_id(), lane = lane_id();
  const int P = 3 + 7 * p.L, TP = p.T * P;
  const int nf = p.d / kDitFeat;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&sm.full[s], 1), mbar_init(&sm.empty[s], 1);
    for (int a = 0; a < 2; ++a) mbar_init(&sm.acc_full[a], 1), mbar_init(&sm.acc_empty[a], kEpiWarps);
    for (int q = 0; q < kQ; ++q) mbar_init(&sm.q_full[q], 1), mbar_init(&sm.q_empty[q], 1 + kEpiWarps);
    int items = 0, units = 0;
    for (int tp = 0; tp < TP; ++tp) {
      const PhaseInfo ph = phase_info<TR>(p, tp % P);
      sm.item_start[tp] = items;
      sm.unit_cum[tp] = units;
      items += ph.items * p.n_rt;
      units += ph.units;
    }
    sm.item_start[TP] = items;
    sm.unit_cum[TP] = units;
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  pdl_wait();  // descriptors / noise / counters of this iteration are written by the predecessors

  if (warp == 0) {
    // ---------------- scheduler + TMA producer ----------------
    if (lane == 0) {
      const DitMaps* mp = p.maps;
      constexpr int ti = TR == 256 ? 1 : 0;  // activation maps with TR-row boxes
      const uint64_t pol = policy_evict_last();  // weights re-read by every row tile; activations hot
      int tp = 0;
      uint32_t qi = 0, kbi = 0;
      const int total = sm.item_start[TP];
      for (;;) {
        const int idx = atomicAdd(p.next_item, 1);
        const int slot = qi % kQ;
        mbar_wait_sleep(&sm.q_empty[slot], ((qi / kQ) & 1) ^ 1);
        Item it;
        it.kind = K_END;
        if (idx < total) {
          while (idx >= sm.item_start[tp + 1]) ++tp;
          const PhaseInfo ph = phase_info<TR>(p, tp % P);
          const int local = idx - sm.item_start[tp];
          it.kind = ph.kind;
          it.layer = ph.layer;
          it.step = tp / P;
          it.tp = tp;
          it.r = local / ph.items;
          it.j = local % ph.items;
          it.idx = idx;
          if (p.trace) {
            unsigned int smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            p.trace[(size_t)idx * 8 + 0] = globaltimer();
            p.trace[(size_t)idx * 8 + 4] = smid;
          }
        }
        sm.ring[slot] = it;
        mbar_arrive(&sm.q_full[slot]);
        ++qi;
        if (it.kind == K_END) break;
        if (!is_gemm(it.kind)) continue;
        const CUtensorMap* wm;
        const CUtensorMap* xm;
        const uint8_t* wb;  // pre-tiled weight (or nullptr)
        int nkb, kb0 = 0, wrow = it.j * kDitFeat, kbt = p.d / 64;  // kbt: k-blocks of the whole weight
        switch (it.kind) {
          case K_IN: wm = &mp->w_in; wb = mp->b_in; xm = &mp->x_x[ti]; nkb = kbt = p.C / 64; break;
          case K_QKV: wm = &mp->wqkv[it.layer]; wb = mp->b_qkv[it.layer]; xm = &mp->x_a[ti]; nkb = p.d / 64; break;
          case K_O: wm = &mp->wo[it.layer]; wb = mp->b_o[it.layer]; xm = &mp->x_o[ti]; nkb = p.d / 64; break;
          case K_UP: wm = &mp->w1[it.layer]; wb = mp->b_1[it.layer]; xm = &mp->x_a[ti]; nkb = p.d / 64; break;
          case K_DOWN:
            wm = &mp->w2[it.layer];
            wb = mp->b_2[it.layer];
            xm = &mp->x_u[ti];
            kbt = p.ff / 64;
            nkb = kbt / p.down_split;
            kb0 = (it.j % p.down_split) * nkb;
            wrow = (it.j / p.down_split) * kDitFeat;
            break;
          default: wm = &mp->w_out; wb = mp->b_out; xm = &mp->x_a[ti]; nkb = p.d / 64; wrow = 0; break;
        }
        auto load_a = [&](int s, int kb) {
          if (wb)
            bulk_load_hint(sA + s * kABytes, wb + ((size_t)(wrow / kDitFeat) * kbt + kb) * kABytes, kABytes,
                           &sm.full[s], pol);
          else
            tma_load_2d(sA + s * kABytes, wm, &sm.full[s], kb * 64, wrow, pol);
        };
        const int xrow = it.r * TR;
        const int pre = nkb < STAGES ? nkb : STAGES;
        for (int i = 0; i < pre; ++i) {  // weights first: they never depend on another item
          const uint32_t k = kbi + i;
          const int s = k % STAGES;
          mbar_wait_sleep(&sm.empty[s], ((k / STAGES) & 1) ^ 1);
          mbar_expect_tx(&sm.full[s], kStageBytes);
          load_a(s, kb0 + i);
        }
        wait_ge(p.progress + it.r, sm.unit_cum[tp]);
        fence_proxy_async_global();
        if (p.trace) p.trace[(size_t)idx * 8 + 1] = globaltimer();
        for (int i = 0; i < pre; ++i) {
          const int s = (kbi + i) % STAGES;
          tma_load_2d(sB + s * kBBytes, xm, &sm.full[s], (kb0 + i) * 64, xrow, pol);
        }
        for (int i = pre; i < nkb; ++i) {
          const uint32_t k = kbi + i;
          const int s = k % STAGES;
          mbar_wait_sleep(&sm.empty[s], ((k / STAGES) & 1) ^ 1);
          mbar_expect_tx(&sm.full[s], kStageBytes);
          load_a(s, kb0 + i);
          tma_load_2d(sB + s * kBBytes, xm, &sm.full[s], (kb0 + i) * 64, xrow, pol);
        }
        kbi += nkb;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      uint32_t qi = 0, kbi = 0, gi = 0;
      for (;;) {
        const int slot = qi % kQ;
        mbar_wait_sleep(&sm.q_full[slot], (qi / kQ) & 1);
        const Item it = sm.ring[slot];
        mbar_arrive(&sm.q_empty[slot]);
        ++qi;
        if (it.kind == K_END) break;
        if (!is_gemm(it.kind)) continue;
        const int nkb = it.kind == K_IN ? p.C / 64 : it.kind == K_DOWN ? p.ff / 64 / p.down_split : p.d / 64;
        const int acc = gi & 1;
        mbar_wait_sleep(&sm.acc_empty[acc], ((gi >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t td = tmem + acc * TR;
        for (int i = 0; i < nkb; ++i) {
          const uint32_t k = kbi + i;
          const int s = k % STAGES;
          mbar_wait_sleep(&sm.full[s], (k / STAGES) & 1);
          tc_fence_after();
          const uint64_t ad = sdesc_k_sw128(smem_addr(sA + s * kABytes));
          const uint64_t bd = sdesc_k_sw128(smem_addr(sB + s * kBBytes));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) tc_mma_bf16(td, ad + 2 * kk, bd + 2 * kk, kIdesc, (i | kk) != 0);
          tc_commit(&sm.empty[s]);
        }
        tc_commit(&sm.acc_full[acc]);
        kbi += nkb;
        ++gi;
      }
    }
  } else {
    // ---------------- epilogue / LN / attention (warps 2..5) ----------------
    const int ew = warp - 2;          // 0..7 worker index
    const int half = ew >> 2;         // which half of the item's chunks (quadrant partner: ew ^ 4)
    const int quad = warp & 3;        // TMEM lane quadrant this warp may access
    const int et = ew * 32 + lane;    // 0..255
    const int fl = quad * 32 + lane;  // output feature (TMEM lane) of this thread within a tile
    const int ld_mod = p.L * 6 * p.d;
    uint32_t qi = 0, gi = 0;
    for (;;) {
      const int slot = qi % kQ;
      mbar_wait_sleep(&sm.q_full[slot], (qi / kQ) & 1);
      const Item it = sm.ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.q_empty[slot]);
      ++qi;
      if (it.kind == K_END) break;
      const float* mod_t = p.mod_table + (size_t)it.step * p.vocab * ld_mod;
      const int row0 = it.r * TR;
      const int tok0 = it.r * Tl::tok;
      if (is_gemm(it.kind)) {
        const bool gated = it.kind == K_O || it.kind == K_DOWN;
        const int ft = it.kind == K_DOWN ? it.j / p.down_split : it.kind == K_OUT ? 0 : it.j;
        const int f = ft * kDitFeat + fl;  // this thread's output feature
        const int tix = it.r * nf + ft;
        // static side inputs first, overlapping the item's mainloop: the adaLN
        // gate of every token of the tile (O / DOWN) or pos_emb (IN)
        float aux[16];
        if (it.kind == K_IN) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) aux[jj] = bf2f(p.pos_emb[(size_t)jj * p.d + f]);  // row % 16 = sample
        } else if (gated) {
          const int goff = it.layer * 6 * p.d + (it.kind == K_O ? 2 : 5) * p.d + f;
          int id[Tile<TR>::my_chunks];
#pragma unroll
          for (int c = 0; c < Tl::my_chunks; ++c) id[c] = p.toks[tok0 + half + 2 * c].id;  // my chunks' tokens
#pragma unroll
          for (int c = 0; c < Tl::my_chunks; ++c) aux[c] = mod_t[(size_t)id[c] * ld_mod + goff];
        }
        const int acc = gi & 1;
        mbar_wait_sleep(&sm.acc_full[acc], (gi >> 1) & 1);
        tc_fence_after();
        ++gi;
        if (p.trace && et == 0) p.trace[(size_t)it.idx * 8 + 2] = globaltimer();
        // split MLP-down: parts meet pairwise, (p0 + p1) [+ (p2 + p3)]; in
        // each pair / between the pairs the first arriver writes its partial
        // and the second adds it (commutative: arrival order never changes bits)
        int mode = 0;
        const int pr = it.kind == K_DOWN ? (it.j % p.down_split) / 2 : 0;  // my pair
        const int tix2 = tix * 2 + pr;
        if (it.kind == K_DOWN && p.down_split > 1) {
          if (et == 0) {
            const int old1 = atomicAdd(p.tile_cnt + tix2, 1);
            int md = 1;
            if (old1 & 1) {  // second of my pair: the pair sum is mine
              wait_ge(p.ready + tix2, (old1 + 1) / 2);
              md = 2;
              if (p.down_split == 4) {
                const int old2 = atomicAdd(p.tile_cnt2 + tix, 1);
                md = 3;
                if (old2 & 1) {
                  wait_ge(p.ready2 + tix, (old2 + 1) / 2);
                  md = 4;
                }
              }
            }
            sm.mode = md;
          }
          ep_bar();
          mode = sm.mode;
        }
        const float* part1 = p.part + (size_t)tix2 * TR * kDitFeat;  // my pair's first partial
        float* part2 = p.part2 + (size_t)tix * TR * kDitFeat;        // the first pair sum
        const uint32_t ta = tmem + acc * TR + (static_cast<uint32_t>(quad * 32) << 16);
        switch (it.kind) {  // once per item: the chunk loop is specialised per kind (no jump table inside)
          case K_IN: epi_chunks<TR, K_IN, 0>(p, ta, row0, ft, part1, part2, part2, quad, half, lane, aux, it.step); break;
          case K_QKV: epi_chunks<TR, K_QKV, 0>(p, ta, row0, ft, part1, part2, part2, quad, half, lane, aux, it.step); break;
          case K_UP: epi_chunks<TR, K_UP, 0>(p, ta, row0, ft, part1, part2, part2, quad, half, lane, aux, it.step); break;
          case K_OUT: epi_chunks<TR, K_OUT, 0>(p, ta, row0, ft, part1, part2, part2, quad, half, lane, aux, it.step); break;
          case K_O: epi_chunks<TR, K_O, 0>(p, ta, row0, ft, part1, part2, part2, quad, half, lane, aux, it.step); break;
          default:
            switch (mode) {
              case 1: epi_chunks<TR, K_DOWN, 1>(p, ta, row0, ft, part1, part2, const_cast<float*>(part1), quad, half, lane, aux, it.step); break;
              case 2: epi_chunks<TR, K_DOWN, 2>(p, ta, row0, ft, part1, part2, part2, quad, half, lane, aux, it.step); break;
              case 3: epi_chunks<TR, K_DOWN, 3>(p, ta, row0, ft, part1, part2, part2, quad, half, lane, aux, it.step); break;
              case 4: epi_chunks<TR, K_DOWN, 4>(p, ta, row0, ft, part1, part2, part2, quad, half, lane, aux, it.step); break;
              default: epi_chunks<TR, K_DOWN, 0>(p, ta, row0, ft, part1, part2, part2, quad, half, lane, aux, it.step); break;
            }
            break;
        }
        if (p.trace && et == 0) p.trace[(size_t)it.idx * 8 + 5] = globaltimer();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.acc_empty[acc]);
        if (mode == 1 || mode == 3) {
          ep_bar();
          if (et == 0) {
            __threadfence();
            atomicAdd(mode == 1 ? p.ready + tix2 : p.ready2 + tix, 1);
            if (p.trace) p.trace[(size_t)it.idx * 8 + 3] = globaltimer();
          }
          continue;  // no unit of progress: the final sum completes the tile
        }
      } else {
        // LN / attention items: wait for the tile's earlier phases
        float4 sc[PER], sh[PER];
        const bool mod = it.kind == K_LN1 || it.kind == K_LN2;
        if (mod) {  // the token's adaLN rows are static: load them before the wait
          const float* mr = mod_t + (size_t)p.toks[tok0 + it.j].id * ld_mod + it.layer * 6 * p.d;
          const int sh_off = it.kind == K_LN1 ? 0 : 3 * p.d, sc_off = it.kind == K_LN1 ? p.d : 4 * p.d;
#pragma unroll
          for (int k = 0; k < PER; ++k) {
            sc[k] = *reinterpret_cast<const float4*>(mr + sc_off + 4 * (lane + 32 * k));
            sh[k] = *reinterpret_cast<const float4*>(mr + sh_off + 4 * (lane + 32 * k));
          }
        }
        if (et == 0) {
          wait_ge(p.progress + it.r, sm.unit_cum[it.tp]);
          if (p.trace) p.trace[(size_t)it.idx * 8 + 1] = p.trace[(size_t)it.idx * 8 + 2] = globaltimer();
        }
        ep_bar();
        if (it.kind == K_ATT) {
          const int h = it.j % p.H, grp = it.j / p.H;  // item = (head, group of kEpiWarps tokens)
          attn_token_head(p.qkv, tok0 + grp * kEpiWarps + ew, h, p.d, p.o, lane);
        } else {
          constexpr int kRows = 16 / kEpiWarps;  // rows of the token per warp
          const int row = (tok0 + it.j) * 16 + ew * kRows;
          ln_rows<PER, kRows>(p.h + (size_t)row * p.d, mod, sc, sh, p.a + (size_t)row * p.d, lane);
        }
      }
      // completion: publish this item's writes (generic proxy; the consumers
      // read them through TMA), then count one unit of the tile
      fence_proxy_async_global();
      ep_bar();
      if (et == 0) {
        if (p.trace) p.trace[(size_t)it.idx * 8 + 6] = globaltimer();
        __threadfence();
        atomicAdd(p.progress + it.r, 1);
        if (p.trace) p.trace[(size_t)it.idx * 8 + 3] = globaltimer();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<512>(tmem);
}

template <int STAGES, int TR>
constexpr size_t smem_bytes() {
  return 1024 + (size_t)STAGES * Tile<TR>::stage_bytes + sizeof(Smem);
}
static_assert(smem_bytes<4, 256>() <= 227 * 1024, "4-stage 256-row ring must fit");

template <int PER, int STAGES, int TR>
cudaError_t launch_fused(const DitFusedParams& p, int ctas, cudaStream_t st) {
  auto kern = dit_fused_kernel<PER, STAGES, TR>;
  constexpr size_t smem = smem_bytes<STAGES, TR>();
  static std::atomic<uint64_t> configured{0};
  if (cudaError_t e = smem_attr_once(kern, smem, configured); e != cudaSuccess) return e;
  return launch_k(kern, dim3(ctas), dim3(kThreadsF), smem, st, 1, p);
}

}  // namespace

int dit_fused_items(int n_rt, int tile_rows, int d, int H, int ff, int L, int T, int down_split) {
  const int nf = d / kDitFeat, tok = tile_rows / 16, att = H * tok / kEpiWarps;
  const int per_step = nf + L * (tok + 3 * nf + att + nf + tok + ff / kDitFeat + nf * down_split) + tok + 1;
  return per_step * T * n_rt;
}

bool dit_fused_supported(int d, int C, int H, int ff, int L, int T) {
  return (d == 256 || d == 512 || d == 1024) && ff % kDitFeat == 0 && C == 64 && H * 128 == d &&
         L <= kDitMaxLayers && T * (3 + 7 * L) <= kDitMaxPhases;
}

cudaError_t dit_fused_run(const DitFusedParams& p, int stages, int ctas, cudaStream_t st) {
  if (!dit_fused_supported(p.d, p.C, p.H, p.ff, p.L, p.T) || (p.down_split != 1 && p.down_split != 2 && p.down_split != 4) ||
      (p.ff / 64) % p.down_split != 0 || p.n_rt <= 0)
    return cudaErrorInvalidValue;
  // 4-stage rings for both tiles (128 rows: 32 KB stages -- 6 stages measured slower, r02_dit_fused_v7.txt)
  const bool wide = p.tile_rows == 256;
  if (!wide && p.tile_rows != 128) return cudaErrorInvalidValue;
  (void)stages;
  switch (p.d / 128) {
    case 2: return wide ? launch_fused<2, 4, 256>(p, ctas, st) : launch_fused<2, 4, 128>(p, ctas, st);
    case 4: return wide ? launch_fused<4, 4, 256>(p, ctas, st) : launch_fused<4, 4, 128>(p, ctas, st);
    case 8: return wide ? launch_fused<8, 4, 256>(p, ctas, st) : launch_fused<8, 4, 128>(p, ctas, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace omni_dev
