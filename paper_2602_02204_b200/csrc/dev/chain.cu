// The AR step as ONE launch ("step chain").
//
// Every kernel of a decode step (embed, per layer: QKV GEMM -> attention ->
// O GEMM -> gate-up GEMM -> down GEMM, final norm, LM head, argmax) becomes a
// range of CTA-sized work items of a single grid. A CTA takes a ticket when
// it starts (atomicAdd on a per-launch counter) and runs the item with that
// ticket; items are numbered in op order, so an item only ever waits (spins
// on the previous op's completion counter) for items with SMALLER tickets,
// which belong to CTAs that have already started -> no deadlock, whatever
// the residency and whatever else runs on the GPU.
//
// What it buys over the PDL kernel chain (ar_kernels.cu / gemm_tc.cu): the
// CTAs of op o+1 become resident the moment ANY slot frees (not when op o's
// whole grid has drained), stream their weight tiles into smem before they
// wait, and leave the wait ~1 us after op o's last tile signals, instead of
// paying a grid completion + dependent launch per op.
//
// The grid runs in clusters of 8 CTAs; a cluster takes one ticket (8 items).
// GEMM items are BN = 16 tiles (decode / small steps, rows <= 16) and the S
// splits of a tile sit in one cluster and reduce over DSMEM in rank order
// (same fp32 order as the per-kernel path -> bit-identical outputs). Replaces the same reference
// functions as the per-kernel path: ArEngine::run_batch / StageModel hooks
// (ar_engine.hpp:308-337, registry.hpp:79-89).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ar_dev.cuh"
#include "chain.h"
#include "gemm_epi.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace omni_dev {

using namespace gemm_dev;

namespace {

constexpr int kChainThreads = 128;
constexpr int kChainBN = 16;
constexpr int kChainStages = 6;
constexpr int kChainAttnWarps = kChainThreads / 32;
constexpr int kChainAttnChunk = 64;
using ChainAttnSmem = AttnSmem<kChainAttnWarps, kChainAttnChunk>;

constexpr uint32_t kABytes = kBlockM * kBlockK * 2;
constexpr uint32_t kBBytes = kChainBN * kBlockK * 2;
constexpr size_t kPipeBytes = (size_t)kChainStages * (kABytes + kBBytes);
constexpr size_t kGemmSmem = 1024 + kPipeBytes + 256 + 4 * kChainBN + 16;
static_assert(kPipeBytes >= (size_t)kChainBN * 128 * 4 * 3 / 2, "split-K staging fits the ring");
constexpr size_t kChainSmem = kGemmSmem > sizeof(ChainAttnSmem) + 128 ? kGemmSmem : sizeof(ChainAttnSmem) + 128;

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Wait for the previous op of the chain (thread 0 spins, the CTA barrier
// extends the acquire to every thread).
struct ChainDep {
  const int* cnt;
  int target;
  unsigned long long* tr;
  __device__ __forceinline__ void spin() const {
    if (cnt != nullptr) {
      int ns = 32;
      while (ld_acquire(cnt) < target) {
        __nanosleep(ns);
        ns = ns < 256 ? ns * 2 : 256;
      }
    }
    if (tr) tr[1] = globaltimer();
  }
  __device__ __forceinline__ void operator()() const {
    if (threadIdx.x == 0) spin();
    __syncthreads();
  }
};

__device__ __forceinline__ void signal_done(int* done) {
  __syncthreads();  // every thread's global writes of this item precede the release
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(done, 1);
  }
}

__device__ __forceinline__ void epi_dispatch(int epi, const GemmArgs& a, int n_tile, int tok0, int ncols,
                                             const float* acc, const float* inv) {
  switch (epi) {
    case EPI_ROPE_KV: epi_cols<EPI_ROPE_KV>(a, n_tile, tok0, ncols, acc, inv); break;
    case EPI_RESID_NORM: epi_cols<EPI_RESID_NORM>(a, n_tile, tok0, ncols, acc, inv); break;
    case EPI_SWIGLU: epi_cols<EPI_SWIGLU>(a, n_tile, tok0, ncols, acc, inv); break;
    case EPI_F32: epi_cols<EPI_F32>(a, n_tile, tok0, ncols, acc, inv); break;
    default: epi_cols<EPI_BF16>(a, n_tile, tok0, ncols, acc, inv); break;
  }
}

// One BN=16 output tile x one K split of a GEMM op. A cluster of 8 CTAs
// hosts 8/S tiles x S splits (rank r: tile r/S, split r%S); the S splits of
// a tile reduce over DSMEM in fixed rank order (as gemm_tc.cu does).
__device__ __forceinline__ void gemm_item(const ChainParams& P, const ChainOp& op, int o, int item,
                                          const ChainDep& dep, uint8_t* smem_raw) {
  constexpr int BN = kChainBN, STAGES = kChainStages;
  constexpr uint32_t kTmemCols = 32;
  constexpr uint32_t kIdesc = idesc_bf16_f32(kBlockM, BN);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPipeBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint64_t* dep_bar = done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dep_bar + 1);
  float* inv_s = reinterpret_cast<float*>(dep_bar + 2);
  int* last = reinterpret_cast<int*>(inv_s + BN);

  const GemmArgs& a = op.a;
  const int warp = warp_id(), lane = lane_id();
  const int S = op.splits;
  const int rank = item % kChainCluster;
  const int n_tile = (item / kChainCluster) * (kChainCluster / S) + rank / S, split = rank % S;
  const int kb_per = op.kb_per;
  const int kb0 = split * kb_per;
  const CUtensorMap* tmW = P.maps + op.w_map;
  const CUtensorMap* tmX = P.maps + op.x_map;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(tmW);
    prefetch_tmap(tmX);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init(dep_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      // weights are static: stream them in before waiting on the previous op
      const int pre = kb_per < STAGES ? kb_per : STAGES;
      for (int i = 0; i < pre; ++i) {
        mbar_expect_tx(&full[i], kABytes + kBBytes);
        tma_load_2d(sA + i * kABytes, tmW, &full[i], (kb0 + i) * kBlockK, n_tile * kBlockM, pol_w);
      }
      dep.spin();
      mbar_arrive(dep_bar);
      for (int i = 0; i < pre; ++i)
        tma_load_2d(sB + i * kBBytes, tmX, &full[i], (kb0 + i) * kBlockK, 0, pol_x);
      for (int i = pre; i < kb_per; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], kABytes + kBBytes);
        const int kx = (kb0 + i) * kBlockK;
        tma_load_2d(sA + s * kABytes, tmW, &full[s], kx, n_tile * kBlockM, pol_w);
        tma_load_2d(sB + s * kBBytes, tmX, &full[s], kx, 0, pol_x);
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
        for (int k = 0; k < kBlockK / 16; ++k) tc_mma_bf16(tmem, ad + 2 * k, bd + 2 * k, kIdesc, (i | k) != 0);
        tc_commit(&empty[s]);
      }
      tc_commit(done);
    }
  } else {
    // idle warps: input-RMS scales, once the producer has seen the dependency
    mbar_wait(dep_bar, 0);
    input_scales(a, 0, min(BN, a.M), inv_s, threadIdx.x - 64, kChainThreads - 64);
  }
  __syncwarp();
  mbar_wait(dep_bar, 0);  // orders this thread's epilogue reads after the previous op
  mbar_wait(done, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const int cols = min(BN, a.M);
  float* red = reinterpret_cast<float*>(smem);  // pipeline smem is free now
  {
    float v[16];
    tmem_ld16(trow, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) red[j * 128 + row] = v[j];
  }
  if (S == 1) {
    epi_dispatch(op.epi, a, n_tile, 0, cols, red, inv_s);
  } else {
    // ranks [base, base + S) hold the partials of this tile; each reduces a
    // slice of token columns across them in rank order, then runs the epilogue
    cluster_sync();
    const int base = (rank / S) * S;
    const int per = (cols + S - 1) / S;
    const int c0 = split * per;
    const int c1 = min(cols, c0 + per);
    float* fin = red + BN * 128;
    const uint32_t red_s = smem_addr(red);
    const int n4 = (c1 > c0 ? c1 - c0 : 0) * 32;
    for (int q = threadIdx.x; q < n4; q += kChainThreads) {
      const int c = c0 + q / 32, r4 = (q % 32) * 4;
      const uint32_t off = static_cast<uint32_t>((c * 128 + r4) * 4);
      float4 v[8];
#pragma unroll
      for (int z = 0; z < 8; ++z)
        if (z < S) v[z] = dsmem_ld_f32x4(dsmem_map(red_s + off, base + z));
      float4 acc = v[0];
#pragma unroll
      for (int z = 1; z < 8; ++z)
        if (z < S) acc.x += v[z].x, acc.y += v[z].y, acc.z += v[z].z, acc.w += v[z].w;
      *reinterpret_cast<float4*>(fin + (c - c0) * 128 + r4) = acc;
    }
    if (c1 > c0) epi_dispatch(op.epi, a, n_tile, c0, c1 - c0, fin, inv_s + c0);
    cluster_sync();  // keep our partial alive until every rank of the tile has read it
  }
  signal_done(P.done + o);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<kTmemCols>(tmem);
}

__global__ void __launch_bounds__(kChainThreads, 2) step_chain_kernel(const __grid_constant__ ChainParams P) {
  extern __shared__ __align__(1024) uint8_t chain_smem[];
  __shared__ int s_ticket;
  __shared__ float s_red[32];
  // one ticket per cluster of 8 CTAs: rank 0 draws it and writes it into
  // every rank's smem over DSMEM; item = 8 * ticket + rank
  const uint32_t rank = cluster_rank();
  if (rank == 0 && threadIdx.x == 0) {
    const int tc = atomicAdd(P.ticket, 1);
    const uint32_t loc = smem_addr(&s_ticket);
    for (uint32_t r = 0; r < kChainCluster; ++r)
      asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(dsmem_map(loc, r)), "r"(tc) : "memory");
  }
  cluster_sync();
  const int t = s_ticket * kChainCluster + (int)rank;
  unsigned long long* tr = P.trace ? P.trace + 3ull * t : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  int o = 0;
  while (o + 1 < P.n_ops && t >= P.ops[o + 1].first) ++o;
  const ChainOp& op = P.ops[o];
  const int item = t - op.first;
  if (item >= op.n_items) {  // cluster padding
    if (op.kind == CHAIN_GEMM && op.splits > 1) {  // the split-K reduction syncs the whole cluster
      cluster_sync();
      cluster_sync();
    }
    return;
  }
  const ChainDep dep{o > 0 ? P.done + (o - 1) : nullptr, o > 0 ? P.ops[o - 1].units : 0, tr};
  switch (op.kind) {
    case CHAIN_GEMM:
      gemm_item(P, op, o, item, dep, chain_smem);
      break;
    case CHAIN_EMBED:
      embed_row(item, P.sd, P.emb, P.emb2, P.hproj, P.cond_table, P.cond_rows, P.d, P.start_id, P.x, P.xb, P.ss,
                P.ss_ld, dep);
      signal_done(P.done + o);
      break;
    case CHAIN_GATHER_COND:
      gather_cond_row(item, P.sd, P.cond_dim, P.condin, dep);
      signal_done(P.done + o);
      break;
    case CHAIN_ATTN:
      if (P.sd.attn_blocks[item / P.n_kv].ntok * (P.n_heads / P.n_kv) <= 16)
        attention_block_mma<kChainAttnWarps, kChainAttnChunk>(
            item / P.n_kv, item % P.n_kv, P.sd, P.q, P.n_heads, P.n_kv, op.layer, P.n_layers, P.kv, P.attn,
            P.attn_scale, *reinterpret_cast<ChainAttnSmem*>(chain_smem), dep);
      else
        attention_block<kChainAttnWarps, kChainAttnChunk>(
            item / P.n_kv, item % P.n_kv, P.sd, P.q, P.n_heads, P.n_kv, op.layer, P.n_layers, P.kv, P.attn,
            P.attn_scale, *reinterpret_cast<ChainAttnSmem*>(chain_smem), dep);
      signal_done(P.done + o);
      break;
    case CHAIN_FINAL:
      final_gather_row(item, P.sd, P.x, P.d, P.eps, P.hbuf, P.ring, P.ring_rows, s_red, dep);
      signal_done(P.done + o);
      break;
    case CHAIN_ARGMAX:
      argmax_row(item, P.logits, P.vocab_pad, P.argmax_lo, P.argmax_hi, P.tok, P.margin, dep);
      signal_done(P.done + o);
      break;
    case CHAIN_HEAD: {
      float* hs = reinterpret_cast<float*>(chain_smem);
      head_row(item, 0, P.vocab, 1, nullptr, P.sd, P.x, P.d, P.eps, P.hbuf, P.ring, P.ring_rows, P.lm, P.logits,
               P.vocab_pad, P.argmax_lo, P.argmax_hi, P.tok, P.margin, hs, s_red, dep);
      signal_done(P.done + o);
      break;
    }
  }
  if (tr && threadIdx.x == 0) tr[2] = globaltimer();
}

}  // namespace

size_t chain_smem_bytes() { return kChainSmem; }
int chain_max_rows() { return kChainBN; }

cudaError_t chain_launch(const ChainParams& P, int n_items, cudaStream_t st) {
  static std::atomic<uint64_t> configured{0};
  if (cudaError_t e = smem_attr_once(step_chain_kernel, kChainSmem, configured); e != cudaSuccess) return e;
  if (cudaError_t e = cudaMemsetAsync(P.done, 0, sizeof(int) * (kChainMaxOps + 1), st); e != cudaSuccess)
    return e;
  // plain (non-PDL) launch: the kernel does its own dependency tracking
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_items);
  cfg.blockDim = dim3(kChainThreads);
  cfg.dynamicSmemBytes = kChainSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kChainCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, step_chain_kernel, P);
}

}  // namespace omni_dev
