// K1: batch-invariant tcgen05/TMA bf16 GEMM  Y[M,N] = X[M,K] · W[N,K]^T.
//
// Swap-AB: the weight tile (128 output features) is the MMA "A" operand
// (M=128), the token tile (BN = 16..256 tokens) the "B" operand, so a decode
// batch of 1..16 rows still issues full-height MMAs while W streams from HBM
// exactly once.  Operands are staged by TMA (SWIZZLE_128B) into a STAGES-deep
// mbarrier ring; one elected thread issues tcgen05.mma into a TMEM accumulator
// (128 lanes x BN fp32 columns); all four warps drain TMEM with tcgen05.ld and
// apply the fused epilogue.
//
// Batch invariance (SURVEY §0.7a, §7 hard part 1): the split-K factor is a
// property of the weight (fixed at load time from (N, K)), the split CTAs of
// a tile form one thread-block cluster and reduce their fp32 partials over
// DSMEM in fixed rank order, and every output element depends only on its
// own row of X — so a row's bits are identical for any batch size M.
//
// Replaces the per-sequence StageModel::prefill/decode loop
// (ar_engine.hpp:308-337, reference_pipeline.hpp:96-154) for the dense
// projections; reused by the DiT (diffusion_engine.hpp:28-43 replacement).
#include <cuda.h>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ar_kernels.h"
#include "gemm.h"
#include "gemm_epi.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace omni_dev {

// debug marks (omni_k_debug_traces, tools/attn_trace.py; null = off)
__device__ unsigned long long* g_gemm_marks = nullptr;
cudaError_t gemm_marks_set(void* p) { return cudaMemcpyToSymbol(g_gemm_marks, &p, sizeof(p)); }

static int bn_for(const GemmWeight& w, int M);  // token-tile width for (weight, batch)
bool gemm_push_enabled();

namespace {

using namespace gemm_dev;

// PUSH (decode tiles BN <= 32 with split-K): instead of cluster barrier ->
// DSMEM pull -> cluster barrier, every split CTA pushes its fp32 partials for
// the column slice each peer owns straight from the TMEM registers into that
// peer's receive buffer (st.async, complete_tx on the owner's mbarrier); the
// owner waits for its bytes only and sums in the same fixed rank order, so
// results are bit-identical to the pull variant. No barrier at exit: a CTA's
// smem is only written by peers before its own wait completes.
template <int BN, int STAGES, int EPI, int kPushS = 0>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const GemmArgs a) {
  constexpr bool PUSH = kPushS > 0;
  constexpr uint32_t kABytes = kBlockM * kBlockK * 2;
  constexpr uint32_t kBBytes = BN * kBlockK * 2;
  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
  constexpr uint32_t kIdesc = idesc_bf16_f32(kBlockM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * kABytes;
  constexpr size_t kPipe = (size_t)STAGES * (kABytes + kBBytes);
  constexpr size_t kEpi = (size_t)BN * 128 * 4 * 3 / 2;  // own partial + reduced slice (S >= 2)
  constexpr size_t kMain = kPipe > kEpi ? kPipe : kEpi;
  constexpr size_t kRecv = PUSH ? (size_t)BN * 128 * 4 : 0;  // [S][128][per] fp32, S * per <= BN
  // own-slice residual (RESID_NORM) / positions, pages, RoPE rows (ROPE_KV)
  constexpr size_t kPre = PUSH ? (size_t)(BN / (kPushS > 0 ? kPushS : 1)) * 128 * 4 + 128 : 0;
  float* recv = reinterpret_cast<float*>(smem + kMain);
  float* pre = reinterpret_cast<float*>(smem + kMain + kRecv);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kMain + kRecv + kPre);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  float* inv_s = reinterpret_cast<float*>(done + 2);  // [BN] input-RMS scales
  uint64_t* recv_bar = reinterpret_cast<uint64_t*>(inv_s + BN);

  const int warp = warp_id(), lane = lane_id();
  const int n_tile = blockIdx.x, m_tile = blockIdx.y, split = blockIdx.z;
  const int kb_per = (a.K / kBlockK) / a.splits;
  unsigned long long* tr = a.trace ? a.trace + 8ull * ((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x)
                                   : nullptr;
  const long long c0 = clock64();
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  const int kb0 = split * kb_per;
  // weight tile (n_tile, kb): a 16 KB block of the pre-tiled copy, or a 2-D TMA box
  auto load_w = [&](uint8_t* dst, uint64_t* bar, int kb, uint64_t pol) {
    if (a.w_blk)
      bulk_load_hint(dst, a.w_blk + ((size_t)n_tile * (a.K / kBlockK) + kb) * kABytes, kABytes, bar, pol);
    else
      tma_load_2d(dst, &tmW, bar, kb * kBlockK, n_tile * kBlockM, pol);
  };

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmX);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    if (PUSH) mbar_init(recv_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (PUSH) cluster_arrive_relaxed();  // recv_bar initialised; waited on before the first push
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();  // the next kernel may start its own prologue / weight prefetch
  if (tr && threadIdx.x == 0) tr[1] = clock64() - c0;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();  // weights: streamed once per step
      const uint64_t pol_x = policy_evict_last();   // activations: shared by all n-tiles
      // Weights never depend on the previous kernel: fill the ring with W
      // tiles BEFORE waiting on the predecessor (PDL), then add the X tiles.
      const int pre = kb_per < STAGES ? kb_per : STAGES;
      for (int i = 0; i < pre; ++i) {
        mbar_expect_tx(&full[i], kABytes + kBBytes);
        load_w(sA + i * kABytes, &full[i], kb0 + i, pol_w);
      }
      pdl_wait();
      if (g_gemm_marks && EPI == EPI_RESID_NORM && a.K == 2048) atomicMax(g_gemm_marks + 1, globaltimer());
      if (tr) tr[2] = clock64() - c0;
      for (int i = 0; i < pre; ++i)
        tma_load_2d(sB + i * kBBytes, &tmX, &full[i], (kb0 + i) * kBlockK, m_tile * BN, pol_x);
      for (int i = pre; i < kb_per; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], kABytes + kBBytes);
        const int kx = (kb0 + i) * kBlockK;
        load_w(sA + s * kABytes, &full[s], kb0 + i, pol_w);
        tma_load_2d(sB + s * kBBytes, &tmX, &full[s], kx, m_tile * BN, pol_x);
      }
      if (tr) tr[3] = clock64() - c0;
      // own stream fully issued: pull this CTA's share of the successor's
      // weights into L2 so the kernel boundary does not idle HBM
      const uint32_t cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      prefetch_l2_share(a.pf_ptr, a.pf_bytes, cta, gridDim.x * gridDim.y * gridDim.z);
    }
  } else if (warp >= 2) {
    // idle warps: input-RMS scales of this token tile, overlapped with the mainloop
    if constexpr (PUSH && EPI == EPI_ROPE_KV) {
      // positions / KV pages / RoPE rows of this rank's token slice: step
      // descriptors (written by desc_copy_kernel, complete before any GEMM
      // of the step launches -- see launch_desc_copy's ordering contract) and
      // static tables, readable before the PDL wait
      constexpr int kPer = BN / kPushS;
      const int cb0 = m_tile * BN + split * kPer;
      const int n_me = min(kPer, a.M - cb0);
      const RopeKvArgs& rp = a.rope;
      int* pre_i = reinterpret_cast<int*>(pre);
      float2* pre_cs = reinterpret_cast<float2*>(pre + 32);
      const int q = threadIdx.x - 64;
      if (q < n_me) {
        const ArRowDesc rd = static_cast<const ArRowDesc*>(rp.rows)[cb0 + q];
        pre_i[q] = rd.pos;
        pre_i[16 + q] = n_tile >= rp.n_heads ? rp.page_table[rd.slot * rp.max_pages + rd.pos / kPageTokens] : 0;
      }
      asm volatile("bar.sync 1, 64;" ::: "memory");  // warps 2-3 only
      if (n_tile < rp.n_heads + rp.n_kv)
        for (int i = q; i < n_me * 64; i += kThreads - 64)
          pre_cs[i] = rp.table[(size_t)pre_i[i >> 6] * 64 + (i & 63)];
    }
    pdl_wait();
    const int m0 = m_tile * BN;
    input_scales(a, m0, min(BN, a.M - m0), inv_s, threadIdx.x - 64, kThreads - 64);
    if constexpr (PUSH && EPI == EPI_RESID_NORM) {
      // stage this rank's residual slice while the MMAs run (the epilogue
      // would otherwise start with a dependent L2 round trip)
      constexpr int kPer = BN / kPushS;
      const int cb0 = m0 + split * kPer;
      const int n_me = min(kPer, a.M - cb0);
      const int n0 = n_tile * kBlockM;
      for (int q = threadIdx.x - 64; q < n_me * 32; q += kThreads - 64) {
        const int c = q >> 5, f = (q & 31) * 4;
        *reinterpret_cast<float4*>(pre + c * 128 + f) =
            *reinterpret_cast<const float4*>(static_cast<const float*>(a.out) + (size_t)(cb0 + c) * a.ldo + n0 + f);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      for (int i = 0; i < kb_per; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t ad = sdesc_k_sw128(smem_addr(sA + s * kABytes));
        const uint64_t bd = sdesc_k_sw128(smem_addr(sB + s * kBBytes));
#pragma unroll
        for (int k = 0; k < kBlockK / 16; ++k) {
          // +32 bytes per K=16 step inside the 128-byte swizzle atom (>>4 encoded)
          tc_mma_bf16(tmem, ad + 2 * k, bd + 2 * k, kIdesc, (i | k) != 0);
        }
        tc_commit(&empty[s]);
      }
      tc_commit(done);
    }
  }
  __syncwarp();
  pdl_wait();  // epilogue reads / writes activations of the predecessor

  // ---- epilogue: TMEM -> smem (fp32, column-major) -> [cluster split-K
  // reduction over DSMEM in fixed rank order] -> fused op -------------------
  mbar_wait(done, 0);
  tc_fence_after();
  if (tr && threadIdx.x == 0) tr[4] = clock64() - c0;
  const int row = warp * 32 + lane;  // TMEM lane == output feature within tile
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const int m0 = m_tile * BN;
  const int cols = min(BN, a.M - m0);           // live token columns
  const int chunks = (cols + 15) / 16;
  float* red = reinterpret_cast<float*>(smem);  // pipeline smem is free now
  if constexpr (PUSH) {
    // Fixed slices of kPer = BN / kPushS token columns per rank (compile-time:
    // fully unrolled, vector stores); a rank whose slice holds no live column
    // receives nothing. Which rank sums a column does not change its sum order.
    constexpr int S = kPushS, kPer = BN / kPushS;
    const int cb0 = split * kPer;
    const int n_me = min(kPer, cols - cb0);  // live columns of my slice (<= 0: none)
    if (threadIdx.x == 0 && n_me > 0) mbar_expect_tx(recv_bar, (uint32_t)((S - 1) * 128 * kPer * 4));
    cluster_wait();  // every peer's recv_bar is initialised
    const uint32_t recv_s = smem_addr(recv) + (uint32_t)((split * 128 + row) * kPer * 4), bar_s = smem_addr(recv_bar);
    float v[BN];
#pragma unroll
    for (int c = 0; c < BN / 16; ++c)
      if (c < chunks) tmem_ld16(trow + c * 16, *reinterpret_cast<float(*)[16]>(v + c * 16));
#pragma unroll
    for (int r = 0; r < S; ++r) {
      if (r * kPer >= cols) break;  // no live column from here on (uniform)
      if (r == split) {
#pragma unroll
        for (int k = 0; k < kPer; ++k) red[k * 128 + row] = v[r * kPer + k];
      } else {
        const uint32_t dst = dsmem_map(recv_s, r), bar = dsmem_map(bar_s, r);
        if constexpr (kPer == 2) {
          st_async_f32x2(dst, v[r * 2], v[r * 2 + 1], bar);
        } else {
          static_assert(kPer % 4 == 0, "push slices of 2 or 4k columns");
#pragma unroll
          for (int k = 0; k < kPer; k += 4)
            st_async_f32x4(dst + k * 4, v[r * kPer + k], v[r * kPer + k + 1], v[r * kPer + k + 2],
                           v[r * kPer + k + 3], bar);
        }
      }
    }
    if (tr && threadIdx.x == 0) tr[5] = clock64() - c0;
    if (n_me > 0) {
      mbar_wait(recv_bar, 0);
      // fixed rank order, own partial in place: identical sums to the pull variant
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int z = 0; z < S; ++z) {
          const float x = z == split ? red[k * 128 + row] : recv[(z * 128 + row) * kPer + k];
          acc = z == 0 ? x : acc + x;
        }
        red[k * 128 + row] = acc;
      }
      // syncs before reading the slice (and the staged residual)
      epi_cols<EPI>(a, n_tile, m0 + cb0, n_me, red, inv_s + cb0,
                    (EPI == EPI_RESID_NORM || EPI == EPI_ROPE_KV) ? pre : nullptr);
    }
  } else {
  for (int c = 0; c < chunks; ++c) {
    float v[16];
    tmem_ld16(trow + c * 16, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) red[(c * 16 + j) * 128 + row] = v[j];
  }
  if (tr && threadIdx.x == 0) tr[5] = clock64() - c0;
  if (a.splits == 1) {
    epi_cols<EPI>(a, n_tile, m0, cols, red, inv_s);  // epi_cols syncs before reading inv_s
  } else {
    // The split CTAs of this tile form one cluster (rank == split). Each
    // reduces a slice of token columns across all ranks, in rank order, so
    // the sum order never depends on the batch. All S remote 16-byte loads
    // of an element group are issued before the ordered sum.
    cluster_sync();
    const int S = a.splits;
    const int per = (cols + S - 1) / S;
    const int c0 = split * per;
    const int c1 = min(cols, c0 + per);
    float* fin = red + BN * 128;
    const uint32_t red_s = smem_addr(red);
    const int n4 = (c1 > c0 ? c1 - c0 : 0) * 32;  // float4 groups in the slice
    for (int q = threadIdx.x; q < n4; q += kThreads) {
      const int c = c0 + q / 32, r4 = (q % 32) * 4;
      const uint32_t off = static_cast<uint32_t>((c * 128 + r4) * 4);
      float4 v[16];
#pragma unroll
      for (int z = 0; z < 16; ++z)
        if (z < S) v[z] = dsmem_ld_f32x4(dsmem_map(red_s + off, z));
      float4 acc = v[0];
#pragma unroll
      for (int z = 1; z < 16; ++z)
        if (z < S) acc.x += v[z].x, acc.y += v[z].y, acc.z += v[z].z, acc.w += v[z].w;
      *reinterpret_cast<float4*>(fin + (c - c0) * 128 + r4) = acc;
    }
    if (c1 > c0) epi_cols<EPI>(a, n_tile, m0 + c0, c1 - c0, fin, inv_s + c0);
    cluster_sync();  // keep our partial alive until every rank has read it
  }
  }  // !PUSH

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<kTmemCols>(tmem);
  if (g_gemm_marks && threadIdx.x == 0) {
    if (EPI == EPI_ROPE_KV) atomicMax(g_gemm_marks + 0, globaltimer());
    if (EPI == EPI_RESID_NORM && a.K == 2048) atomicMax(g_gemm_marks + 2, globaltimer());
  }
  if (tr && threadIdx.x == 0) {
    tr[6] = clock64() - c0;
    tr[7] = globaltimer();
  }
}

template <int BN>
constexpr int stages_for() {
  // Decode tiles: <= ~112 KB (two CTAs per SM; a decode grid has <= 192
  // CTAs, so every SM keeps a slot for the NEXT kernel's CTA to start (PDL)
  // and prefetch its weights while this one drains). Measured (in-chain,
  // tools/gemm_sweep.py): 6 stages beat 4 on the 67 MB gate-up weight.
  // Wide tiles (prefill / DiT): deep rings, one CTA per SM.
  return BN <= 16 ? 6 : BN <= 32 ? 5 : BN <= 64 ? 4 : BN <= 128 ? 6 : 4;
}
template <int BN>
constexpr size_t epi_smem_for() {
  return (size_t)BN * 128 * 4 * 3 / 2;  // own partial + reduced slice (S >= 2)
}
template <int BN, int STAGES = stages_for<BN>(), int kPushS = 0>
constexpr size_t smem_for() {
  constexpr bool PUSH = kPushS > 0;
  constexpr size_t pipe = STAGES * (kBlockM * kBlockK * 2 + BN * kBlockK * 2);
  // + [push receive buffer] + barriers / tmem slot (256 B) + per-column
  // input-RMS scales (4 B x BN) + flag / receive barrier
  return 1024 + (pipe > epi_smem_for<BN>() ? pipe : epi_smem_for<BN>()) + (PUSH ? (size_t)BN * 128 * 4 : 0) +
         (PUSH ? (size_t)BN / (PUSH ? kPushS : 1) * 128 * 4 + 128 : 0) + 256 + 4 * BN + 16;  // + staged epilogue inputs
}
// push split-K variants keep two CTAs per SM (<= ~113 KB): one stage less
static_assert(smem_for<16, 5, 2>() <= 113 * 1024, "BN16 push tile must fit twice per SM");
static_assert(smem_for<32, 4, 2>() <= 113 * 1024, "BN32 push tile must fit twice per SM");
static_assert(smem_for<128, 3>() <= 113 * 1024, "BN128 3-stage tile must fit twice per SM");

template <int BN, int EPI, int STAGES = stages_for<BN>(), int kPushS = 0>
cudaError_t launch_bn(const GemmWeight& w, const GemmInput& x, const GemmArgs& a,
                      cudaStream_t st) {
  auto kern = gemm_tc_kernel<BN, STAGES, EPI, kPushS>;
  constexpr size_t smem = smem_for<BN, STAGES, kPushS>();
  static std::atomic<uint64_t> configured{0};  // per instantiation, per device
  if (cudaError_t e = smem_attr_once(kern, smem, configured); e != cudaSuccess) return e;
  if (a.splits > 8) {  // 16-CTA clusters are non-portable (opt-in)
    static std::atomic<uint64_t> np{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (!(np.load() & bit)) {
      if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
          e != cudaSuccess)
        return e;
      np.fetch_or(bit);
    }
  }
  return launch_k(kern, dim3(w.N_pad / kBlockM, (a.M + BN - 1) / BN, a.splits), dim3(kThreads), smem, st,
                  a.splits, w.tmap, x.tmap_for(BN), a);
}

template <int EPI>
cudaError_t launch_epi(const GemmWeight& w, const GemmInput& x, const GemmArgs& a,
                       cudaStream_t st) {
  // compute-bound weights (DiT per-op path, fill_sms): the widest token tile;
  // the per-element result does not depend on BN
  const bool push = gemm_push_enabled();
  switch (bn_for(w, a.M)) {
    case 16:
      if (push && a.splits == 8) return launch_bn<16, EPI, 5, 8>(w, x, a, st);
      if (push && a.splits == 2) return launch_bn<16, EPI, 5, 2>(w, x, a, st);
      return launch_bn<16, EPI>(w, x, a, st);
    case 32:
      if (push && a.splits == 8) return launch_bn<32, EPI, 4, 8>(w, x, a, st);
      if (push && a.splits == 2) return launch_bn<32, EPI, 4, 2>(w, x, a, st);
      return launch_bn<32, EPI>(w, x, a, st);
    case 64: return launch_bn<64, EPI>(w, x, a, st);  // push needs a 3-stage ring here: measured slower
    case 128: {
      // decode weights (prefill / mixed steps): a 6-stage 128-token tile holds
      // a whole SM -- grids over 148 CTAs (QKV: 192) run in two waves and the
      // next kernel's CTAs cannot co-reside to prefetch (PDL). A 3-stage ring
      // (96 KB in flight, as much as the 16-token 6-stage tile) fits two CTAs
      // per SM. OMNI_BN128_2CTA=0: 6 stages; =2: only for grids > 148 CTAs.
      static const int two = [] {
        const char* e = std::getenv("OMNI_BN128_2CTA");
        return e ? std::atoi(e) : 1;
      }();
      const int ctas = (w.N_pad / kBlockM) * ((a.M + 127) / 128) * a.splits;
      if (!w.fill_sms && (two == 1 || (two == 2 && ctas > 148))) return launch_bn<128, EPI, 3>(w, x, a, st);
      return launch_bn<128, EPI>(w, x, a, st);
    }
    default: return launch_bn<256, EPI>(w, x, a, st);
  }
}

}  // namespace

bool gemm_push_enabled() {  // OMNI_SPLITK_PUSH=0: cluster-barrier + DSMEM-pull reduction
  static const bool push = [] {
    const char* e = std::getenv("OMNI_SPLITK_PUSH");
    return !(e && e[0] == '0');
  }();
  return push;
}

static int bn_for(const GemmWeight& w, int M) {
  int bn = gemm_block_n(M);
  if (!w.fill_sms && bn > 128) {
    // decode weights in big prefill steps: two 128-token tiles (3-stage,
    // two CTAs per SM) instead of one 256-token tile that holds a whole SM
    // (OMNI_BN256_SPLIT=0: keep 256)
    static const bool split = [] {
      const char* e = std::getenv("OMNI_BN256_SPLIT");
      return !(e && e[0] == '0');
    }();
    if (split) return 128;
  }
  if (w.fill_sms && bn > 64) {
    // Widest token tile (fewest CTAs), not the isolated-latency optimum: the
    // DiT shares the GPU with two latency-bound AR chains, and fat tiles leave
    // them SMs -- measured +6.5 % pipeline req/s over a fill-the-SMs cost
    // model (profiles/r01_bench_dit_bn_ab.log) although each DiT GEMM alone is
    // up to 1.6x slower at <= 1k rows (profiles/r01_dit_gemm_sweep_forced_bn.txt).
    bn = M <= 128 ? 128 : 256;
  }
  return bn;
}

// dst 16-byte chunk (tile, kb, row r, position j') <- source chunk
// j = j' ^ (r & 7) of row tile*128 + r, columns kb*64 + 8j .. +7: the
// SWIZZLE_128B image TMA would write for a 1024-byte aligned box.
__global__ void block_weight_kernel(const uint4* __restrict__ w, int K, int64_t n_chunks, uint4* __restrict__ blk) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_chunks) return;
  const int kbt = K / kBlockK;
  const int jp = (int)(q & 7), r = (int)((q >> 3) & 127);
  const int64_t box = q >> 10;  // 1024 chunks of 16 B per 16 KB block
  const int64_t tile = box / kbt, kb = box % kbt;
  const int j = jp ^ (r & 7);
  blk[q] = w[((tile * kBlockM + r) * (int64_t)K + kb * kBlockK) / 8 + j];
}

bool gemm_decode_weights_blocked() {  // OMNI_WBLOCK=0: row-major weights, 2-D TMA boxes (A/B)
  static const bool on = [] {
    const char* e = std::getenv("OMNI_WBLOCK");
    return !(e && e[0] == '0');
  }();
  return on;
}

cudaError_t gemm_block_weight(const __nv_bfloat16* w, int N_pad, int K, uint8_t* blk, cudaStream_t st) {
  if (N_pad % kBlockM != 0 || K % kBlockK != 0) return cudaErrorInvalidValue;
  const int64_t n_chunks = (int64_t)N_pad * K / 8;
  block_weight_kernel<<<(unsigned)((n_chunks + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const uint4*>(w), K, n_chunks, reinterpret_cast<uint4*>(blk));
  return cudaGetLastError();
}

int gemm_block_n(int M) {
  return M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256;
}

cudaError_t gemm_make_args(const GemmWeight& w, const GemmInput& x, int M, int epi, const GemmEpilogue& e,
                           GemmArgs& a) {
  // vectorised epilogue: 8-element aligned rows
  if (e.ldo % 8 != 0 || (reinterpret_cast<uintptr_t>(e.out) & 15) != 0 || w.N % 8 != 0) return cudaErrorInvalidValue;
  if (epi == EPI_GATED_RESID && (e.ldg % 4 != 0 || e.gate_off % 4 != 0)) return cudaErrorInvalidValue;
  if (M > x.rows_cap || w.K != x.K) return cudaErrorInvalidValue;
  a = GemmArgs{};
  a.M = M;
  a.N = w.N_pad;
  a.K = w.K;
  a.n_valid = w.N;
  a.splits = w.splits;
  a.out = e.out;
  a.ldo = e.ldo;
  a.gate = e.gate;
  a.ldg = e.ldg;
  a.gate_off = e.gate_off;
  a.rows_per_group = e.rows_per_group > 0 ? e.rows_per_group : 1;
  a.gate_index = e.gate_index;
  a.gate_index_stride = e.gate_index_stride;
  a.ss_in = e.ss_in;
  a.ss_ld = e.ss_ld;
  a.ss_n = e.ss_n;
  a.norm_d = e.norm_d;
  a.norm_eps = e.norm_eps;
  a.xb = e.xb;
  a.ss_out = e.ss_out;
  a.rope = e.rope;
  a.trace = e.trace;
  a.dt = e.dt;
  a.sample_scale = e.sample_scale;
  a.samples = e.samples;
  if (epi == EPI_EULER && (e.xb == nullptr || e.ss_in != nullptr)) return cudaErrorInvalidValue;
  a.row_bias = e.row_bias;
  a.bias_period = e.bias_period > 0 ? e.bias_period : 1;
  if (e.row_bias && (epi != EPI_F32 || w.N != w.N_pad)) return cudaErrorInvalidValue;
  a.w_blk = w.blk;
  a.pf_ptr = e.pf_ptr;
  a.pf_bytes = e.pf_bytes & ~uint64_t(15);
  if (epi == EPI_RESID_NORM && (e.xb == nullptr || e.ss_out == nullptr || w.N != w.N_pad))
    return cudaErrorInvalidValue;
  if (epi == EPI_ROPE_KV && (e.rope.rows == nullptr || e.rope.kv == nullptr || e.rope.q_out == nullptr ||
                             w.K % 64 != 0 || w.N != (e.rope.n_heads + 2 * e.rope.n_kv) * 128))
    return cudaErrorInvalidValue;
  if (e.ss_in && (e.ss_n <= 0 || e.norm_d <= 0.f)) return cudaErrorInvalidValue;
  if (w.splits > 16 || (a.K / kBlockK) % w.splits != 0) return cudaErrorInvalidValue;
  return cudaSuccess;
}

cudaError_t gemm_run(const GemmWeight& w, const GemmInput& x, int M, int epi, const GemmEpilogue& e,
                     cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  GemmArgs a;
  if (cudaError_t err = gemm_make_args(w, x, M, epi, e, a); err != cudaSuccess) return err;
  switch (epi) {
    case EPI_BF16: return launch_epi<EPI_BF16>(w, x, a, st);
    case EPI_F32: return launch_epi<EPI_F32>(w, x, a, st);
    case EPI_RESID: return launch_epi<EPI_RESID>(w, x, a, st);
    case EPI_GATED_RESID: return launch_epi<EPI_GATED_RESID>(w, x, a, st);
    case EPI_SWIGLU: return launch_epi<EPI_SWIGLU>(w, x, a, st);
    case EPI_GELU: return launch_epi<EPI_GELU>(w, x, a, st);
    case EPI_RESID_NORM: return launch_epi<EPI_RESID_NORM>(w, x, a, st);
    case EPI_ROPE_KV: return launch_epi<EPI_ROPE_KV>(w, x, a, st);
    case EPI_EULER: return launch_epi<EPI_EULER>(w, x, a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace omni_dev
