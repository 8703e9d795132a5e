// Device-side pieces shared by the per-GEMM kernel (gemm_tc.cu) and the
// step-chain kernel (chain.cu): tile constants, vector helpers, the fused
// GEMM epilogues. Internal to libomni_dev.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ar_kernels.h"
#include "gemm.h"
#include "ptx.cuh"

namespace omni_dev {
namespace gemm_dev {

constexpr int kBlockM = 128;  // weight rows per tile (MMA M)
constexpr int kBlockK = 64;   // 128-byte swizzle atom of bf16
constexpr int kThreads = 128;

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.f + tanhf(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float silu(float x) { return x / (1.f + expf(-x)); }

__device__ __forceinline__ void ld8(const float* p, float (&v)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
}
__device__ __forceinline__ void st8(float* p, const float (&v)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void st8_bf16(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 u;
  __nv_bfloat162 h[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  u.x = *reinterpret_cast<uint32_t*>(&h[0]);
  u.y = *reinterpret_cast<uint32_t*>(&h[1]);
  u.z = *reinterpret_cast<uint32_t*>(&h[2]);
  u.w = *reinterpret_cast<uint32_t*>(&h[3]);
  *reinterpret_cast<uint4*>(p) = u;
}

// Per-token input-RMS scale of the fused RMSNorm (GemmEpilogue::ss_in):
// inv[c] = rsqrt(sum_j ss_in[tok0 + c][j] / d + eps), j in fixed order.
__device__ __forceinline__ void input_scales(const GemmArgs& a, int tok0, int ncols, float* inv,
                                             int tid, int nthreads) {
  for (int c = tid; c < ncols; c += nthreads) {
    float s = 0.f;
    if (a.ss_in) {
      const float* p = a.ss_in + (size_t)(tok0 + c) * a.ss_ld;
      for (int j = 0; j < a.ss_n; ++j) s += p[j];
      inv[c] = rsqrtf(s / a.norm_d + a.norm_eps);
    } else {
      inv[c] = 1.f;
    }
  }
}

// Applies the fused epilogue to `ncols` finished accumulator columns held in
// smem as acc[c * 128 + row] (fp32), column c = token tok0 + c. Each thread
// owns 8 consecutive output features of one token, so every global access
// is a 16-byte vector (bf16) or 2x16-byte (fp32); SWIGLU pairs gate row f
// with up row f + 64 of the same tile, ROPE_KV rotates feature f with f + 64.
// `pre` (optional, push path): smem staged during the mainloop -- RESID_NORM:
// the residual rows pre[c * 128 + feature] = x[tok0 + c][tile]; ROPE_KV: the
// tokens' positions, KV pages and RoPE (cos, sin) rows.
template <int EPI>
__device__ __forceinline__ void epi_cols(const GemmArgs& a, int n_tile, int tok0, int ncols,
                                         const float* acc, const float* inv, const float* pre = nullptr) {
  __syncthreads();
  const int t = threadIdx.x;
  if constexpr (EPI == EPI_SWIGLU) {
    const int f0 = (t & 7) * 8;
    for (int c = t >> 3; c < ncols; c += kThreads / 8) {
      float g[8], u[8], o[8];
      ld8(acc + c * 128 + f0, g);
      ld8(acc + c * 128 + 64 + f0, u);
      const float sc = inv[c];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = silu(g[i] * sc) * (u[i] * sc);
      st8_bf16(static_cast<__nv_bfloat16*>(a.out) + (size_t)(tok0 + c) * a.ldo + n_tile * 64 + f0, o);
    }
  } else if constexpr (EPI == EPI_ROPE_KV) {
    const RopeKvArgs& rp = a.rope;
    const ArRowDesc* rows = static_cast<const ArRowDesc*>(rp.rows);
    const int f0 = (t & 7) * 8;
    const int head = n_tile;
    for (int c = t >> 3; c < ncols; c += kThreads / 8) {
      const int tok = tok0 + c;
      float lo[8], hi[8];
      ld8(acc + c * 128 + f0, lo);
      ld8(acc + c * 128 + 64 + f0, hi);
      const float sc = inv[c];
      // `pre` (push path): pos[16] | page[16] | (cos, sin)[c][64], staged
      // during the mainloop; else straight from the descriptors / table
      const int* pre_i = reinterpret_cast<const int*>(pre);
      const float2* pre_cs = reinterpret_cast<const float2*>(pre + 32);
      ArRowDesc rd;
      if (pre) rd.pos = pre_i[c], rd.entry = 0;
      else rd = rows[tok];
      float o0[8], o1[8];
      if (head < rp.n_heads + rp.n_kv) {
        const float4* cs4 = reinterpret_cast<const float4*>(pre ? pre_cs + c * 64 + f0
                                                                : rp.table + (size_t)rd.pos * 64 + f0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 w = cs4[i];  // (cos, sin) of pairs 2i, 2i+1
          const float a0 = lo[2 * i] * sc, b0 = hi[2 * i] * sc;
          const float a1 = lo[2 * i + 1] * sc, b1 = hi[2 * i + 1] * sc;
          o0[2 * i] = a0 * w.x - b0 * w.y;
          o1[2 * i] = b0 * w.x + a0 * w.y;
          o0[2 * i + 1] = a1 * w.z - b1 * w.w;
          o1[2 * i + 1] = b1 * w.z + a1 * w.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) o0[i] = lo[i] * sc, o1[i] = hi[i] * sc;
      }
      __nv_bfloat16* dst;
      if (head < rp.n_heads) {
        dst = rp.q_out + (size_t)tok * rp.n_heads * 128 + head * 128;
      } else {
        const int is_v = head >= rp.n_heads + rp.n_kv;
        const int kh = head - rp.n_heads - (is_v ? rp.n_kv : 0);
        const int page = pre ? pre_i[16 + c] : rp.page_table[rd.slot * rp.max_pages + rd.pos / kPageTokens];
        const int pt = rd.pos % kPageTokens;
        dst = rp.kv +
              ((((size_t)page * rp.n_layers + rp.layer) * 2 + is_v) * rp.n_kv + kh) * kPageTokens * 128 +
              (size_t)pt * 128;
        st8_bf16(dst + kv_swz(f0 >> 3, pt) * 8, o0);  // swizzled 16-byte chunks (ptx.cuh kv_swz)
        st8_bf16(dst + kv_swz(8 + (f0 >> 3), pt) * 8, o1);
        continue;
      }
      st8_bf16(dst + f0, o0);
      st8_bf16(dst + 64 + f0, o1);
    }
  } else if constexpr (EPI == EPI_RESID_NORM) {
    // warp-uniform trip count so the 16-lane sum-of-squares shuffle is safe
    const int r0 = (t & 15) * 8;
    const int n0 = n_tile * kBlockM + r0;
    for (int cb = 0; cb < ncols; cb += kThreads / 16) {
      const int c = cb + (t >> 4);
      const bool live = c < ncols;
      float ss = 0.f;
      if (live) {
        const int tok = tok0 + c;
        float v[8], x[8];
        ld8(acc + c * 128 + r0, v);
        float* r = static_cast<float*>(a.out) + (size_t)tok * a.ldo + n0;
        if (pre) ld8(pre + c * 128 + r0, x);
        else ld8(r, x);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          x[i] += v[i];
          ss += x[i] * x[i];
        }
        st8(r, x);
        st8_bf16(a.xb + (size_t)tok * a.ldo + n0, x);
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (live && (t & 15) == 0) a.ss_out[(size_t)(tok0 + c) * a.ss_ld + n_tile] = ss;
    }
  } else {
    const int r0 = (t & 15) * 8;
    const int n0 = n_tile * kBlockM + r0;
    if (n0 >= a.n_valid) return;
    for (int c = t >> 4; c < ncols; c += kThreads / 16) {
      const int tok = tok0 + c;
      float v[8];
      ld8(acc + c * 128 + r0, v);
      const float sc = inv[c];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] *= sc;
      if constexpr (EPI == EPI_BF16) {
        st8_bf16(static_cast<__nv_bfloat16*>(a.out) + (size_t)tok * a.ldo + n0, v);
      } else if constexpr (EPI == EPI_F32) {
        if (a.row_bias) {
          const uint4 raw = *reinterpret_cast<const uint4*>(a.row_bias + (size_t)(tok % a.bias_period) * a.N + n0);
          const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(b2[i]);
            v[2 * i] += f.x, v[2 * i + 1] += f.y;
          }
        }
        st8(static_cast<float*>(a.out) + (size_t)tok * a.ldo + n0, v);
      } else if constexpr (EPI == EPI_RESID) {
        float* r = static_cast<float*>(a.out) + (size_t)tok * a.ldo + n0;
        float x[8];
        ld8(r, x);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] += v[i];
        st8(r, x);
      } else if constexpr (EPI == EPI_GATED_RESID) {
        float g[8], x[8];
        const int grp = tok / a.rows_per_group;
        const int grow = a.gate_index ? a.gate_index[(size_t)grp * a.gate_index_stride] : grp;
        ld8(a.gate + (size_t)grow * a.ldg + a.gate_off + n0, g);
        float* r = static_cast<float*>(a.out) + (size_t)tok * a.ldo + n0;
        if (pre) ld8(pre + c * 128 + r0, x);
        else ld8(r, x);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] += g[i] * v[i];
        st8(r, x);
      } else if constexpr (EPI == EPI_EULER) {
        float* xr = static_cast<float*>(a.out) + (size_t)tok * a.ldo + n0;
        float x[8];
        ld8(xr, x);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] += a.dt * v[i];
        st8(xr, x);
        st8_bf16(a.xb + (size_t)tok * a.ldo + n0, x);
        if (a.samples && n0 == 0) {
          float q = rintf(a.sample_scale * x[0]);
          q = fminf(fmaxf(q, -64.f), 63.f);
          a.samples[tok] = (int32_t)q;
        }
      } else if constexpr (EPI == EPI_GELU) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = gelu_tanh(v[i]);
        st8_bf16(static_cast<__nv_bfloat16*>(a.out) + (size_t)tok * a.ldo + n0, v);
      }
    }
  }
}

}  // namespace gemm_dev
}  // namespace omni_dev
