// Host runtime of libomni_dev: stage construction (random-init weights
// materialised on device), paged-KV bookkeeping, and the batched AR / DiT
// step drivers behind the C ABI (include/omni_dev.h).
#include "stage.h"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <tuple>

#include "common.h"
#include "kernels.h"
#include "rng.h"

using namespace omni_dev;

namespace {

constexpr float kNormEps = 1e-6f;

int round_up(int v, int m) { return (v + m - 1) / m * m; }

template <typename T>
T* dev_alloc(omni_stage* st, size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(&p, count * sizeof(T));
  if (e != cudaSuccess)
    throw DevError(OMNI_E_OOM, std::string("cudaMalloc ") + std::to_string(count * sizeof(T)) +
                                   " bytes: " + cudaGetErrorString(e));
  st->allocs.push_back(p);
  return static_cast<T*>(p);
}

// A streaming decode weight is stored pre-tiled (gemm_decode_weights_blocked):
// generated row-major into a scratch buffer, rewritten as 16 KB tile images.
template <class Fill>
void materialise(omni_stage* st, DevTensor& t, Fill fill) {
  const size_t n = (size_t)t.rows_pad * t.cols;
  t.p = dev_alloc<__nv_bfloat16>(st, n);
  if (!t.tiled) {
    OMNI_KERNEL(fill(t.p));
    return;
  }
  __nv_bfloat16* tmp = nullptr;
  OMNI_CUDA(cudaMalloc(&tmp, n * sizeof(__nv_bfloat16)));
  const cudaError_t e1 = fill(tmp);
  const cudaError_t e2 = e1 == cudaSuccess ? gemm_block_weight(tmp, (int)t.rows_pad, (int)t.cols,
                                                               reinterpret_cast<uint8_t*>(t.p), st->stream)
                                           : e1;
  const cudaError_t e3 = cudaStreamSynchronize(st->stream);
  cudaFree(tmp);
  OMNI_CUDA(e2);
  OMNI_CUDA(e3);
}

DevTensor make_weight(omni_stage* st, const std::string& name, int64_t rows, int64_t rows_pad,
                      int64_t cols, uint32_t tid, float scale, bool tiled = false) {
  DevTensor t;
  t.rows = rows;
  t.rows_pad = rows_pad;
  t.cols = cols;
  t.tiled = tiled;
  materialise(st, t, [&](__nv_bfloat16* dst) {
    return fill_weights(dst, rows_pad, rows, cols, st->seed, tid, scale, st->stream);
  });
  st->weight_bytes += (uint64_t)rows * cols * 2;
  st->named[tiled ? name + ".tiled" : name] = t;
  return t;
}

DevTensor make_swiglu(omni_stage* st, const std::string& name, int64_t ff, int64_t cols,
                      uint32_t tid_gate, uint32_t tid_up, float scale, bool tiled = false) {
  DevTensor t;
  t.rows = t.rows_pad = 2 * ff;
  t.cols = cols;
  t.tiled = tiled;
  materialise(st, t, [&](__nv_bfloat16* dst) {
    return fill_swiglu(dst, ff, cols, st->seed, tid_gate, tid_up, scale, st->stream);
  });
  st->weight_bytes += (uint64_t)2 * ff * cols * 2;
  st->named[tiled ? name + ".tiled" : name] = t;
  return t;
}

GemmWeight gemm_of(const DevTensor& t, int max_splits, int target_ctas = 192) {
  GemmWeight g;
  OMNI_REQUIRE(gemm_make_weight(g, t.p, (int)t.rows, (int)t.rows_pad, (int)t.cols, max_splits, target_ctas),
               OMNI_E_BADARG, "weight tensor map encode failed");
  if (t.tiled) g.blk = reinterpret_cast<const uint8_t*>(t.p);
  return g;
}

GemmInput input_of(const __nv_bfloat16* p, int rows_cap, int K) {
  GemmInput x;
  OMNI_REQUIRE(gemm_make_input(x, p, rows_cap, K), OMNI_E_BADARG, "input tensor map encode failed");
  return x;
}

// Returns true when the buffers were (re)allocated.
bool staging_reserve(Staging& s, size_t bytes) {
  if (bytes <= s.cap) return false;
  if (s.in_use) OMNI_CUDA(cudaEventSynchronize(s.in_use));
  if (s.host) cudaFreeHost(s.host);
  if (s.dev) cudaFree(s.dev);
  size_t cap = std::max<size_t>(bytes, 64 * 1024);
  OMNI_CUDA(cudaMallocHost(&s.host, cap));
  OMNI_CUDA(cudaMalloc(&s.dev, cap));
  s.cap = cap;
  if (!s.in_use) OMNI_CUDA(cudaEventCreateWithFlags(&s.in_use, cudaEventDisableTiming));
  return true;
}

void drop_graphs(omni_stage* st) {
  for (auto& kv : st->graphs) cudaGraphExecDestroy(kv.second.exec);
  st->graphs.clear();
  st->key_hits.clear();
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw DevError(OMNI_E_NOGPU, "no CUDA device visible (libomni_dev has no CPU fallback)");
}

void ensure_idle(omni_stage* st) {
  OMNI_REQUIRE(!st->pending, OMNI_E_BADARG,
               "stage has an unfinished step; call omni_stage_wait/omni_stage_query first");
}

// ---------------------------------------------------------------------------
// construction
// ---------------------------------------------------------------------------
void build_ar(omni_stage* st) {
  const auto& m = st->m;
  OMNI_REQUIRE(m.head_dim == kHeadDim, OMNI_E_BADARG, "head_dim must be 128");
  OMNI_REQUIRE(m.n_heads % m.n_kv_heads == 0, OMNI_E_BADARG, "n_heads % n_kv_heads != 0");
  OMNI_REQUIRE(m.d_model % 128 == 0 && m.d_ff % 128 == 0, OMNI_E_BADARG, "dims must be multiples of 128");
  const int d = m.d_model, L = m.n_layers, H = m.n_heads, KVH = m.n_kv_heads, ff = m.d_ff;
  const bool talker = m.kind == OMNI_MODEL_TALKER;
  const float s_d = 1.f / std::sqrt((float)d);

  st->emb = make_weight(st, "embed", 256, 256, d, 1, 1.0f);  // byte-valued token ids
  st->vocab_pad = round_up(m.vocab, 128);
  st->lm = make_weight(st, "lm_head", m.vocab, st->vocab_pad, d, 2, 4.0f * s_d);
  st->glm = gemm_of(st->lm, 8);
  if (talker) {
    OMNI_REQUIRE(m.cond_dim % 64 == 0 && m.cond_dim > 0, OMNI_E_BADARG, "talker cond_dim");
    st->emb2 = make_weight(st, "embed_codec", m.vocab + 1, m.vocab + 1, d, 3, 1.0f);
    st->whid = make_weight(st, "w_hid", d, d, m.cond_dim, 4, 1.f / std::sqrt((float)m.cond_dim));
    st->ghid = gemm_of(st->whid, 8);
    st->start_id = m.vocab;  // codec start id
    st->argmax_lo = 0;
  } else {
    st->start_id = 0;  // reserved id 0 is the thinker start token
    st->argmax_lo = 1; // outputs live in [1, 255] like token_of (reference_pipeline.hpp:34)
  }
  st->argmax_hi = m.vocab;
  const int qkv_rows = (H + 2 * KVH) * kHeadDim;
  st->layers.resize(L);
  for (int l = 0; l < L; ++l) {
    auto& ly = st->layers[l];
    const uint32_t b = 16u * (l + 1);
    const std::string p = "L" + std::to_string(l) + ".";
    ly.wqkv = make_weight(st, p + "wqkv", qkv_rows, qkv_rows, d, b + 0, s_d);
    ly.wo = make_weight(st, p + "wo", d, d, H * kHeadDim, b + 1, 1.f / std::sqrt((float)(H * kHeadDim)));
    // the two streaming weights (67 + 33.5 MB per Thinker layer) are stored
    // pre-tiled: one contiguous 16 KB bulk copy per tile instead of a 2-D box
    // of 128 strided 128-byte rows (in-chain gate-up 12.2 -> 11.8 us, down
    // 7.8 -> 7.3 us at 16 rows; QKV / O measured ~3 % slower pre-tiled, their
    // slices sit in the prefetch ring: profiles/r02_weight_tiles.txt)
    const bool tiled = gemm_decode_weights_blocked();
    ly.wgu = make_swiglu(st, p + "wgu", ff, d, b + 2, b + 3, s_d, tiled);
    ly.wd = make_weight(st, p + "wd", d, d, ff, b + 4, 1.f / std::sqrt((float)ff), tiled);
    ly.gqkv = gemm_of(ly.wqkv, 8);
    ly.go = gemm_of(ly.wo, 8);
    ly.ggu = gemm_of(ly.wgu, 1);  // 128 n-tiles: no split-K (a 2-way split measured neutral)
    ly.gd = gemm_of(ly.wd, 8);    // 16 n-tiles x 8-way split-K (16-way measured slower)
  }

  // activations
  const int R = st->rows_cap = std::max(16, st->lim.max_batch_tokens);
  st->x = dev_alloc<float>(st, (size_t)R * d);
  st->xn = dev_alloc<__nv_bfloat16>(st, (size_t)R * d);
  st->ss = dev_alloc<float>(st, (size_t)R * (d / 128));
  st->q = dev_alloc<__nv_bfloat16>(st, (size_t)R * H * kHeadDim);
  st->attn = dev_alloc<__nv_bfloat16>(st, (size_t)R * H * kHeadDim);
  st->act = dev_alloc<__nv_bfloat16>(st, (size_t)R * ff);
  st->hbuf = dev_alloc<__nv_bfloat16>(st, (size_t)R * d);
  st->logits = dev_alloc<float>(st, (size_t)R * st->vocab_pad);
  st->in_xn = input_of(st->xn, R, d);
  st->in_attn = input_of(st->attn, R, H * kHeadDim);
  st->in_act = input_of(st->act, R, ff);
  st->in_hbuf = input_of(st->hbuf, R, d);

  if (talker) {
    st->condin = dev_alloc<__nv_bfloat16>(st, (size_t)R * m.cond_dim);
    st->hproj = dev_alloc<float>(st, (size_t)R * d);
    st->in_cond = input_of(st->condin, R, m.cond_dim);
    st->cond_table = dev_alloc<float>(st, (size_t)st->lim.max_resident * st->cond_rows * d);
  } else {
    st->ring = dev_alloc<__nv_bfloat16>(st, (size_t)st->lim.max_resident * st->ring_rows * d);
  }
  // paged KV: [page][layer][k|v][kv_head][16][128] bf16
  st->max_pages = (st->lim.max_seq_len + kPageTokens - 1) / kPageTokens;
  int pages = st->lim.kv_pages > 0 ? st->lim.kv_pages : st->lim.max_resident * st->max_pages;
  st->page_table = dev_alloc<int32_t>(st, (size_t)st->lim.max_resident * st->max_pages);
  OMNI_CUDA(cudaMemsetAsync(st->page_table, 0, (size_t)st->lim.max_resident * st->max_pages * sizeof(int32_t),
                            st->stream));
  st->kv = dev_alloc<__nv_bfloat16>(st, (size_t)pages * L * 2 * KVH * kPageTokens * kHeadDim);
  if (st->lim.max_seq_len > kAttnSplitChunks * 128) {  // contexts long enough to split (attention CHUNK 128)
    st->split_groups = st->lim.max_resident + (st->rows_cap + kAttnQTok - 1) / kAttnQTok;
    st->split_part = dev_alloc<float>(st, (size_t)st->split_groups * KVH * kAttnMaxParts * 16 * (kHeadDim + 2));
    st->split_cnt = dev_alloc<int>(st, (size_t)st->split_groups * KVH);
    OMNI_CUDA(cudaMemsetAsync(st->split_cnt, 0, (size_t)st->split_groups * KVH * sizeof(int), st->stream));
  }
  st->free_pages.resize(pages);
  for (int i = 0; i < pages; ++i) st->free_pages[i] = pages - 1 - i;
  // prefix cache: the Thinker's KV is a function of the prompt tokens alone
  // (the Talker's also of its conditioning rows: never cached)
  st->prefix.enabled = m.kind == OMNI_MODEL_THINKER;
  st->prefix.refs.assign(pages, 0);
  st->free_slots.resize(st->lim.max_resident);
  for (int i = 0; i < st->lim.max_resident; ++i) st->free_slots[i] = st->lim.max_resident - 1 - i;
  // RoPE table (theta 10000, rotate-half), computed in double, stored fp32
  std::vector<float2> rt((size_t)st->lim.max_seq_len * (kHeadDim / 2));
  for (int pos = 0; pos < st->lim.max_seq_len; ++pos)
    for (int i = 0; i < kHeadDim / 2; ++i) {
      const double inv = std::pow(10000.0, -(double)i / (kHeadDim / 2));
      const double a = pos * inv;
      rt[(size_t)pos * (kHeadDim / 2) + i] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
  st->rope = dev_alloc<float2>(st, rt.size());
  OMNI_CUDA(cudaMemcpyAsync(st->rope, rt.data(), rt.size() * sizeof(float2), cudaMemcpyHostToDevice,
                            st->stream));
  // OMNI_STEP_TRACE=1 (tools/step_trace.py): every GEMM launch of a step
  // records its per-CTA phase stamps in its own slot (baked into the graphs).
  if (const char* e = std::getenv("OMNI_STEP_TRACE"); e && e[0] == '1') {
    st->step_trace = dev_alloc<unsigned long long>(st, (size_t)kStepTraceLaunches * kStepTraceCtas * 8);
    OMNI_CUDA(cudaMemsetAsync(st->step_trace, 0, (size_t)kStepTraceLaunches * kStepTraceCtas * 8 * 8, st->stream));
  }
  // Step results [n_dec tokens | n_dec margins]: the argmax kernel stores
  // them straight into mapped pinned host memory (no D2H copy on the step's
  // tail: -2..3 µs per step, profiles/r01_zc_tok_ab.txt).
  OMNI_CUDA(cudaHostAlloc(&st->h_tok, 2 * (size_t)R * sizeof(int32_t), cudaHostAllocMapped));
  {
    void* dp = nullptr;
    OMNI_CUDA(cudaHostGetDevicePointer(&dp, st->h_tok, 0));
    st->d_tok = static_cast<int32_t*>(dp);
  }
  OMNI_CUDA(cudaStreamSynchronize(st->stream));
}

void build_dit(omni_stage* st) {
  const auto& m = st->m;
  OMNI_REQUIRE(m.head_dim == 128 && m.dit_samples == kDitSamples, OMNI_E_BADARG,
               "DiT needs head_dim 128 and 16 samples per token");
  OMNI_REQUIRE(m.dit_channels % 64 == 0 && m.dit_channels <= 128, OMNI_E_BADARG, "DiT channels");
  const int d = m.d_model, L = m.n_layers, C = m.dit_channels, ff = m.d_ff;
  const float s_d = 1.f / std::sqrt((float)d);
  // the DiT's GEMM weights pre-tiled like the AR streaming weights: each
  // item's weight tiles are single 16 KB bulk copies (isolated iteration
  // 1018 -> 998 us at 8 tokens, within 1 % at 64-512; profiles/r02_weight_tiles.txt)
  const bool dt = gemm_decode_weights_blocked();
  st->w_in = make_weight(st, "w_in", d, d, C, 1, 1.f / std::sqrt((float)C), dt);
  st->pos_emb = make_weight(st, "pos_emb", kDitSamples, kDitSamples, d, 2, 0.5f);
  st->tok_emb = make_weight(st, "tok_emb", m.vocab, m.vocab, d, 3, 1.0f);
  st->t_emb = make_weight(st, "t_emb", m.dit_steps, m.dit_steps, d, 4, 1.0f);
  st->w_out = make_weight(st, "w_out", C, round_up(C, 128), d, 5, s_d, dt);
  st->w_mod = make_weight(st, "w_mod", (int64_t)L * 6 * d, (int64_t)L * 6 * d, d, 6, 0.5f * s_d);
  st->g_in = gemm_of(st->w_in, 1);
  st->g_in.fill_sms = true;
  st->g_out = gemm_of(st->w_out, 1);
  st->g_out.fill_sms = true;
  st->g_mod = gemm_of(st->w_mod, 1);
  st->dlayers.resize(L);
  for (int l = 0; l < L; ++l) {
    auto& ly = st->dlayers[l];
    const uint32_t b = 16u * (l + 1);
    const std::string p = "L" + std::to_string(l) + ".";
    ly.wqkv = make_weight(st, p + "wqkv", 3 * d, 3 * d, d, b + 1, s_d, dt);
    ly.wo = make_weight(st, p + "wo", d, d, d, b + 2, s_d, dt);
    ly.w1 = make_weight(st, p + "w1", ff, ff, d, b + 3, s_d, dt);
    ly.w2 = make_weight(st, p + "w2", d, d, ff, b + 4, 1.f / std::sqrt((float)ff), dt);
    ly.gqkv = gemm_of(ly.wqkv, 1);
    ly.gqkv.fill_sms = true;
    ly.go = gemm_of(ly.wo, 1, 64);
    ly.go.fill_sms = true;
    ly.g1 = gemm_of(ly.w1, 1);
    ly.g1.fill_sms = true;
    ly.g2 = gemm_of(ly.w2, 1, 64);
    ly.g2.fill_sms = true;
  }
  const int T = st->tok_cap = round_up(std::max(16, st->lim.dit_max_tokens), 2 * kDitTileTok);  // whole 256-row tiles
  const int R = st->drows_cap = T * kDitSamples;
  st->dx = dev_alloc<float>(st, (size_t)R * C);
  st->dxin = dev_alloc<__nv_bfloat16>(st, (size_t)R * C);
  st->dh = dev_alloc<float>(st, (size_t)R * d);
  st->da = dev_alloc<__nv_bfloat16>(st, (size_t)R * d);
  st->dqkv = dev_alloc<__nv_bfloat16>(st, (size_t)R * 3 * d);
  st->dout = dev_alloc<__nv_bfloat16>(st, (size_t)R * d);
  st->du = dev_alloc<__nv_bfloat16>(st, (size_t)R * ff);
  // fused iteration: MLP-down split in two K halves (fixed per weight shape:
  // batch invariance) so its items match the others' K = d mainloop
  // K halves meet in a commutative pair sum (dit_fused.cu). Four parts (a
  // tree of pair sums, also supported) measured slower at every batch size:
  // 3x the partial-sum traffic (profiles/r02_dit_fused_v7.txt)
  st->down_split = (ff >= 2 * d && (ff / 64) % 2 == 0) ? 2 : 1;
  const int n_rt = R / kDitTileRows, nfd = d / kDitFeat;
  st->dpart = dev_alloc<float>(st, (size_t)3 * n_rt * nfd * kDitTileRows * kDitFeat);  // [2 pairs] + pair sum
  st->dctl_n = n_rt + 6 * n_rt * nfd + 1;
  st->dctl = dev_alloc<int>(st, (size_t)st->dctl_n);
  {
    int sms = 0;
    OMNI_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, st->dev));
    st->dit_ctas = st->dit_sms_all = sms;
  }
  if (const char* e = std::getenv("OMNI_DIT_TRACE"); e && e[0] == '1') {
    st->dit_trace_items = dit_fused_items(n_rt, kDitTileRows, d, m.n_heads, ff, L, m.dit_steps, st->down_split);
    st->dit_trace = dev_alloc<unsigned long long>(st, (size_t)st->dit_trace_items * 8);
  }
  const int cvec_rows = std::max(T, m.vocab);  // per-step rows / adaLN table rows
  const bool fused = dit_fused_supported(d, C, m.n_heads, ff, L, m.dit_steps);
  st->dcvec = dev_alloc<__nv_bfloat16>(st, (size_t)cvec_rows * d);
  st->din_x = input_of(st->dxin, R, C);
  st->din_a = input_of(st->da, R, d);
  st->din_o = input_of(st->dout, R, d);
  st->din_u = input_of(st->du, R, ff);
  st->din_c = input_of(st->dcvec, cvec_rows, d);
  if (fused) {  // TMA descriptors of the fused iteration, resident on the device
    DitMaps mp{};
    mp.w_in = st->g_in.tmap;  // 128-row boxes: MMA A (swap-AB)
    mp.w_out = st->g_out.tmap;
    mp.b_in = st->g_in.blk;
    mp.b_out = st->g_out.blk;
    for (int l = 0; l < L; ++l) {
      const auto& ly = st->dlayers[l];
      mp.wqkv[l] = ly.gqkv.tmap;
      mp.wo[l] = ly.go.tmap;
      mp.w1[l] = ly.g1.tmap;
      mp.w2[l] = ly.g2.tmap;
      mp.b_qkv[l] = ly.gqkv.blk;
      mp.b_o[l] = ly.go.blk;
      mp.b_1[l] = ly.g1.blk;
      mp.b_2[l] = ly.g2.blk;
    }
    for (int i = 0; i < 2; ++i) {  // 128- and 256-row boxes (dit_tile_rows)
      mp.x_x[i] = st->din_x.tmap_for(128 << i);
      mp.x_a[i] = st->din_a.tmap_for(128 << i);
      mp.x_o[i] = st->din_o.tmap_for(128 << i);
      mp.x_u[i] = st->din_u.tmap_for(128 << i);
    }
    st->dmaps = dev_alloc<DitMaps>(st, 1);
    OMNI_CUDA(cudaMemcpyAsync(st->dmaps, &mp, sizeof(mp), cudaMemcpyHostToDevice, st->stream));
  }

  // adaLN modulation table: mod[t][id] = W_mod . silu(tok_emb[id] + t_emb[t])
  // for every (Euler step, conditioning id) — the per-token GEMM of the
  // reference-shaped model depends on nothing else, so it is evaluated once
  // here with the same kernel (batch invariance => identical rows).
  const int ld_mod = L * 6 * d;
  st->mod_table = dev_alloc<float>(st, (size_t)m.dit_steps * m.vocab * ld_mod);
  {
    std::vector<DitTokDesc> ids(m.vocab);
    for (int i = 0; i < m.vocab; ++i) ids[i] = DitTokDesc{0, 0, i};
    DitTokDesc* ids_dev = dev_alloc<DitTokDesc>(st, m.vocab);
    OMNI_CUDA(cudaMemcpyAsync(ids_dev, ids.data(), ids.size() * sizeof(DitTokDesc), cudaMemcpyHostToDevice,
                              st->stream));
    for (int t = 0; t < m.dit_steps; ++t) {
      OMNI_KERNEL(dit_cond(ids_dev, m.vocab, st->tok_emb.p, st->t_emb.p, t, d, st->dcvec, st->stream));
      GemmEpilogue e;
      e.out = st->mod_table + (size_t)t * m.vocab * ld_mod;
      e.ldo = ld_mod;
      OMNI_KERNEL(gemm_run(st->g_mod, st->din_c, m.vocab, EPI_F32, e, st->stream));
    }
  }
  // Zero-copy waveform samples: the Euler epilogue of the last step stores
  // them straight into the pinned host buffer (UVA).
  OMNI_CUDA(cudaMallocHost(&st->h_samples, (size_t)R * sizeof(int32_t)));
  st->dsamples = st->h_samples;
  OMNI_CUDA(cudaStreamSynchronize(st->stream));
}

void destroy_stage(omni_stage* st) {
  if (!st) return;
  cudaSetDevice(st->dev);
  if (st->stream) cudaStreamSynchronize(st->stream);
  drop_graphs(st);
  for (void* p : st->allocs) cudaFree(p);
  for (Staging* s : {&st->desc, &st->pack}) {
    if (s->host) cudaFreeHost(s->host);
    if (s->dev) cudaFree(s->dev);
    if (s->in_use) cudaEventDestroy(s->in_use);
  }
  if (st->h_tok) cudaFreeHost(st->h_tok);
  if (st->h_samples) cudaFreeHost(st->h_samples);
  for (cudaEvent_t e : {st->ev_start, st->ev_done, st->ev_link, st->ev_pack})
    if (e) cudaEventDestroy(e);
  if (st->stream) cudaStreamDestroy(st->stream);
  delete st;
}

// ---------------------------------------------------------------------------
// AR step
// ---------------------------------------------------------------------------
SeqSlot& seq_for(omni_stage* st, uint64_t id) {
  auto it = st->seqs.find(id);
  if (it != st->seqs.end()) return it->second;
  OMNI_REQUIRE(!st->free_slots.empty(), OMNI_E_OOM, "no free resident slot on stage");
  SeqSlot s;
  s.slot = st->free_slots.back();
  st->free_slots.pop_back();
  return st->seqs.emplace(id, std::move(s)).first->second;
}

void prefix_evict(omni_stage* st);

void ensure_pages(omni_stage* st, SeqSlot& s, int upto) {
  const int need = (upto + kPageTokens - 1) / kPageTokens;
  OMNI_REQUIRE(need <= st->max_pages, OMNI_E_OOM,
               "sequence longer than max_seq_len (" + std::to_string(st->lim.max_seq_len) + ")");
  while ((int)s.pages.size() < need) {
    if (st->free_pages.empty()) prefix_evict(st);
    OMNI_REQUIRE(!st->free_pages.empty(), OMNI_E_OOM, "paged-KV pool exhausted");
    const int page = st->free_pages.back();
    st->pending_deltas.push_back(PageDelta{s.slot * st->max_pages + (int)s.pages.size(), page});
    s.pages.push_back(page);
    st->free_pages.pop_back();
    if (!st->prefix.refs.empty()) st->prefix.refs[page] = 1;
  }
}

// ---- prefix cache -------------------------------------------
uint64_t prefix_page_key(uint64_t prev, const int32_t* t) {
  uint64_t h = mix64(prev ^ 0x5be0cd19137e2179ull);
  for (int i = 0; i < kPageTokens; ++i) h = mix64(h ^ (uint64_t)(uint32_t)t[i] ^ ((uint64_t)i << 40));
  return h | 1;  // never 0
}

void page_unref(omni_stage* st, int page) {
  auto& pc = st->prefix;
  if (pc.refs.empty() || --pc.refs[page] == 0) st->free_pages.push_back(page);
}

// Drops every cached page no sequence maps (refs == 1: only the cache).
void prefix_evict(omni_stage* st) {
  auto& pc = st->prefix;
  for (auto it = pc.key_of.begin(); it != pc.key_of.end();) {
    if (pc.refs[it->first] == 1) {
      pc.page_of.erase(it->second);
      pc.refs[it->first] = 0;
      st->free_pages.push_back(it->first);
      ++pc.evicted_pages;
      it = pc.key_of.erase(it);
    } else {
      ++it;
    }
  }
}

// A prefill span of `s`: record its tokens and map every further full
// prompt page already in the cache (stopping at the first miss).
void prefix_lookup(omni_stage* st, SeqSlot& s, int pos0, int span, const int32_t* tokens) {
  auto& pc = st->prefix;
  if (s.no_cache) return;
  if (pos0 > (int)s.toks.size()) {  // a gap: not a continuation of the recorded prompt
    s.no_cache = true;
    return;
  }
  // record the span's new tokens (a span may be seen twice: reserve, then step)
  const int have = (int)s.toks.size() - pos0;
  if (have < span) s.toks.insert(s.toks.end(), tokens + have, tokens + span);
  while (!s.lookup_done && s.pages.size() == s.keys.size() &&
         (s.keys.size() + 1) * kPageTokens <= s.toks.size()) {
    const size_t p = s.keys.size();
    const uint64_t k = prefix_page_key(p ? s.keys.back() : 0, s.toks.data() + p * kPageTokens);
    auto hit = pc.page_of.find(k);
    if (hit == pc.page_of.end()) {
      s.lookup_done = true;
      break;
    }
    ++pc.refs[hit->second];
    st->pending_deltas.push_back(PageDelta{s.slot * st->max_pages + (int)p, hit->second});
    s.pages.push_back(hit->second);
    s.keys.push_back(k);
    s.cached_upto = (int)(p + 1) * kPageTokens;
  }
}

// After a step computed prompt positions below `upto`: key and cache its
// full pages.
void prefix_insert(omni_stage* st, SeqSlot& s, int upto) {
  auto& pc = st->prefix;
  if (s.no_cache || upto <= s.cached_upto) return;  // this step computed nothing of it
  s.lookup_done = true;  // computed pages follow: no more lookups for this sequence
  while ((s.keys.size() + 1) * kPageTokens <= (size_t)std::min<int>(upto, (int)s.toks.size())) {
    const size_t p = s.keys.size();
    const uint64_t k = prefix_page_key(p ? s.keys.back() : 0, s.toks.data() + p * kPageTokens);
    s.keys.push_back(k);
    const int page = s.pages[p];
    if (pc.page_of.count(k) || pc.key_of.count(page)) continue;  // already cached (another copy)
    pc.page_of.emplace(k, page);
    pc.key_of.emplace(page, k);
    ++pc.refs[page];
    ++pc.inserted_pages;
  }
}

size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

// eager launches of a geometry before it is captured (OMNI_GRAPH_HITS)
int graph_after_hits() {
  static const int n = [] {
    const char* e = std::getenv("OMNI_GRAPH_HITS");
    return e ? std::max(1, std::atoi(e)) : 12;
  }();
  return n;
}

// OMNI_GRAPHS=0 launches every step eagerly (A/B measurements).
bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("OMNI_GRAPHS");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Runs the kernel sequence `body` on the stage stream through a CUDA graph
// cached under `key` (the launch geometry of the step: every pointer the
// kernels see is fixed per stage, every per-step value lives in the device
// descriptor blob copied before the launch). The first occurrence of a key
// is captured (PDL launch attributes become programmatic graph edges) and
// instantiated; later steps replay it with one cudaGraphLaunch.
template <typename F>
StepGraph& capture_graph(omni_stage* st, uint64_t key, F&& body) {
  cudaStream_t s = st->stream;
  if (st->graphs.size() >= 4096) drop_graphs(st);
  const uint64_t l0 = counters().launches;
  OMNI_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
  cudaGraph_t g = nullptr;
  try {
    body();
  } catch (...) {
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    counters().launches = l0;
    throw;
  }
  OMNI_CUDA(cudaStreamEndCapture(s, &g));
  StepGraph sg;
  sg.nodes = (int)(counters().launches - l0);
  counters().launches = l0;  // counted per replay
  const cudaError_t e = cudaGraphInstantiate(&sg.exec, g, 0);
  cudaGraphDestroy(g);
  OMNI_CUDA(e);
  ++counters().graph_captures;
  return st->graphs.emplace(key, sg).first->second;
}

template <class F>
void run_graph(omni_stage* st, uint64_t key, F&& body) {
  cudaStream_t s = st->stream;
  if (!graphs_enabled()) {
    body();
    return;
  }
  auto it = st->graphs.find(key);
  StepGraph* sg = it == st->graphs.end() ? nullptr : &it->second;
  if (!sg) {
    // Capture + instantiate costs ~1 ms of host time: a launch geometry is
    // only graphed once it has recurred (timing-dependent batches produce a
    // long tail of one-off geometries); until then the step runs eagerly
    // (still PDL-chained). Decode-only geometries are captured up front
    // (prewarm_decode_graphs).
    if (++st->key_hits[key] < graph_after_hits()) {
      body();
      return;
    }
    sg = &capture_graph(st, key, body);
  }
  ++counters().graph_replays;
  OMNI_CUDA(cudaGraphLaunch(sg->exec, s));
  counters().launches += sg->nodes;
}

// Descriptor blob at FIXED offsets (capacity-sized regions, so the device
// pointers baked into a captured step graph never change):
//   entries | decode entry list | attention blocks | rows | page-table delta
// The page table itself is persistent in HBM ([slot][max_pages], indexed by
// the resident slot); a step's blob carries only the page assignments made
// since the previous step ({index, page} pairs, count in the delta header),
// which the step's first kernel applies. So the blob stays ~20 KB even when
// max_seq_len is the 8192-token kv budget (516 pages per sequence).
struct ArDescLayout {
  size_t off_dec, off_blk, off_rows, off_delta, reserve, cap_delta;
};
ArDescLayout ar_desc_layout(const omni_stage* st) {
  const size_t cap_e = (size_t)st->lim.max_resident, cap_r = (size_t)st->rows_cap;
  ArDescLayout l;
  // the attention blocks come last: a step graph (keyed by n_blocks) copies
  // only [0, off_blk + n_blocks) -- the block region is sized for split-KV
  // worst cases (kAttnMaxParts per block) that ordinary steps never use
  l.off_dec = align16(cap_e * sizeof(ArEntryDesc));
  l.off_rows = l.off_dec + align16(cap_e * sizeof(int32_t));
  l.off_blk = l.off_rows + align16(cap_r * sizeof(ArRowDesc));
  l.off_delta = l.off_blk + align16((cap_r + cap_e) * kAttnMaxParts * sizeof(AttnBlockDesc));
  l.cap_delta = kPageDeltaCap;
  l.reserve = l.off_delta + sizeof(PageDeltaHeader) + l.cap_delta * sizeof(PageDelta);
  return l;
}
ArStepDev ar_step_dev(const omni_stage* st, const ArDescLayout& lay) {
  ArStepDev sd;
  sd.entries = reinterpret_cast<const ArEntryDesc*>(st->desc.dev);
  sd.rows = reinterpret_cast<const ArRowDesc*>(st->desc.dev + lay.off_rows);
  sd.page_table = st->page_table;
  sd.dec_entries = reinterpret_cast<const int32_t*>(st->desc.dev + lay.off_dec);
  sd.attn_blocks = reinterpret_cast<const AttnBlockDesc*>(st->desc.dev + lay.off_blk);
  sd.max_pages = st->max_pages;
  sd.split_part = st->split_part;
  sd.split_cnt = st->split_cnt;
  return sd;
}
// The per-kernel AR step (PDL chain) for one launch geometry; everything
// step-specific is read from the fixed-offset descriptor blob, so the launch
// sequence depends on (n_rows, n_blocks, n_dec, cond_prefill) only -- the
// step-graph key.
//
// Ordering contract of the blob: desc_copy_kernel (first kernel) copies it
// from pinned staging and applies the page-table delta; the next kernel
// (embed / gather_cond) waits for it (PdlDep: griddepcontrol.wait BEFORE its
// launch_dependents), so every later kernel -- including the attention and
// RoPE-epilogue reads that run before their own griddepcontrol.wait -- sees
// a completed copy. Keep that wait-before-trigger order in the kernel after
// desc_copy.
void launch_ar_kernels(omni_stage* st, const ArStepDev& sd, int n_rows, int n_blocks, int n_dec,
                       bool cond_prefill) {
  const auto& m = st->m;
  const int d = m.d_model, H = m.n_heads, KVH = m.n_kv_heads, L = m.n_layers;
  const bool talker = m.kind == OMNI_MODEL_TALKER;
  cudaStream_t s = st->stream;
  {
    const ArDescLayout lay = ar_desc_layout(st);
    OMNI_KERNEL(launch_desc_copy(st->desc.dev, st->desc.host, align16(lay.off_blk + (size_t)n_blocks * sizeof(AttnBlockDesc)),
                                 st->desc.host + lay.off_delta,
                                 st->page_table, s));
  }
  int trace_slot = 0;  // OMNI_STEP_TRACE: one slot per GEMM launch, in launch order
  auto traced = [&](GemmEpilogue e) {
    if (st->step_trace && trace_slot < kStepTraceLaunches)
      e.trace = st->step_trace + (size_t)(trace_slot++) * kStepTraceCtas * 8;
    return e;
  };
  if (cond_prefill) {
    OMNI_KERNEL(launch_gather_cond(sd, n_rows, m.cond_dim, st->condin, s));
    GemmEpilogue e;
    e.out = st->hproj;
    e.ldo = d;
    OMNI_KERNEL(gemm_run(st->ghid, st->in_cond, n_rows, EPI_F32, traced(e), s));
  }
  // st->xn holds bf16(x) (un-normalised); the RMSNorm scale is applied in
  // the consuming GEMM's epilogue from the per-tile sums of squares st->ss.
  const int ss_ld = d / 128;
  OMNI_KERNEL(launch_embed(sd, n_rows, st->emb.p, talker ? st->emb2.p : nullptr, st->hproj,
                         st->cond_table, st->cond_rows, d, st->start_id, st->x, st->xn, st->ss, ss_ld,
                         nullptr, 0, s));
  GemmEpilogue norm_in;  // fused RMSNorm of the GEMM input
  norm_in.ss_in = st->ss;
  norm_in.ss_ld = ss_ld;
  norm_in.ss_n = ss_ld;
  norm_in.norm_d = (float)d;
  norm_in.norm_eps = kNormEps;
  for (int l = 0; l < L; ++l) {
    const auto& ly = st->layers[l];
    GemmEpilogue e = norm_in;  // QKV: norm scale -> RoPE -> q rows / paged KV
    e.out = st->q;
    e.ldo = H * kHeadDim;
    e.rope.rows = sd.rows;
    e.rope.page_table = sd.page_table;
    e.rope.max_pages = sd.max_pages;
    e.rope.table = st->rope;
    e.rope.q_out = st->q;
    e.rope.kv = st->kv;
    e.rope.n_heads = H;
    e.rope.n_kv = KVH;
    e.rope.layer = l;
    e.rope.n_layers = L;
    OMNI_KERNEL(gemm_run(ly.gqkv, st->in_xn, n_rows, EPI_ROPE_KV, traced(e), s));
    OMNI_KERNEL(launch_attention(sd, n_blocks, st->q, H, KVH, l, L, st->kv, st->attn, nullptr, 0, s));
    GemmEpilogue r;  // x += attn W_o^T; xb = bf16(x); ss = sums of squares
    r.out = st->x;
    r.ldo = d;
    r.xb = st->xn;
    r.ss_out = st->ss;
    r.ss_ld = ss_ld;
    OMNI_KERNEL(gemm_run(ly.go, st->in_attn, n_rows, EPI_RESID_NORM, traced(r), s));
    e = norm_in;
    e.out = st->act;
    e.ldo = m.d_ff;
    OMNI_KERNEL(gemm_run(ly.ggu, st->in_xn, n_rows, EPI_SWIGLU, traced(e), s));
    OMNI_KERNEL(gemm_run(ly.gd, st->in_act, n_rows, EPI_RESID_NORM, traced(r), s));
  }
  if (n_dec > 0) {
    OMNI_KERNEL(launch_final_gather(sd, n_dec, st->x, d, kNormEps, st->hbuf,
                                    talker ? nullptr : st->ring, st->ring_rows, s));
    GemmEpilogue e;
    e.out = st->logits;
    e.ldo = st->vocab_pad;
    OMNI_KERNEL(gemm_run(st->glm, st->in_hbuf, n_dec, EPI_F32, traced(e), s));
    OMNI_KERNEL(launch_sample(sd, st->logits, st->vocab_pad, n_dec, st->argmax_lo, st->argmax_hi, st->top_k,
                              st->sample_seed, st->d_tok, reinterpret_cast<float*>(st->d_tok + n_dec), s));
  }
}

uint64_t ar_graph_key(int n_rows, int n_blocks, int n_dec, bool cond_prefill) {
  return ((uint64_t)n_rows << 40) | ((uint64_t)n_blocks << 20) | ((uint64_t)n_dec << 1) | (cond_prefill ? 1u : 0u);
}

// Decode-only steps (every entry feeds one token: n_rows = n_blocks = n_dec)
// are the steady state of both AR stages; capture their step graphs at stage
// creation (~1 ms host time each) instead of stalling the serving loop the
// third time a batch size shows up. OMNI_PREWARM=<max decode rows> (0 = off).
void prewarm_decode_graphs(omni_stage* st) {
  if (!graphs_enabled()) return;
  static const int cap_env = [] {
    const char* e = std::getenv("OMNI_PREWARM");
    return e ? std::atoi(e) : -1;
  }();
  int upto = std::min(st->lim.max_resident, st->rows_cap);
  if (cap_env >= 0) upto = std::min(upto, cap_env);
  if (upto <= 0) return;
  const ArDescLayout lay = ar_desc_layout(st);
  if (staging_reserve(st->desc, lay.reserve)) drop_graphs(st);
  const ArStepDev sd = ar_step_dev(st, lay);
  for (int n = 1; n <= upto; ++n) {
    const uint64_t key = ar_graph_key(n, n, n, false);
    if (!st->graphs.count(key)) capture_graph(st, key, [&] { launch_ar_kernels(st, sd, n, n, n, false); });
  }
}

void ar_step(omni_stage* st, const omni_ar_batch* b, int32_t* tok_out, float* margin_out) {
  ensure_idle(st);
  const int ne = b->n_entries;
  OMNI_REQUIRE(ne >= 0, OMNI_E_BADARG, "n_entries < 0");
  const bool talker = st->m.kind == OMNI_MODEL_TALKER;
  int n_rows = 0;
  for (int e = 0; e < ne; ++e) {
    OMNI_REQUIRE(b->span[e] >= 1, OMNI_E_BADARG, "entry span < 1");
    OMNI_REQUIRE(b->phase[e] != OMNI_PHASE_DECODE || b->span[e] == 1, OMNI_E_BADARG,
                 "decode entries feed exactly one token");
    n_rows += b->span[e];
  }
  OMNI_REQUIRE(n_rows <= st->rows_cap, OMNI_E_BADARG,
               "batch of " + std::to_string(n_rows) + " tokens exceeds max_batch_tokens");
  if (talker) OMNI_REQUIRE(b->cond_row != nullptr, OMNI_E_BADARG, "talker step needs cond_row");

  OMNI_REQUIRE(ne <= st->lim.max_resident, OMNI_E_BADARG, "more entries than max_resident_requests");
  const ArDescLayout lay = ar_desc_layout(st);
  if (staging_reserve(st->desc, lay.reserve)) drop_graphs(st);
  // prefix cache: map cached prompt pages before any fresh page is assigned
  if (st->prefix.enabled)
    for (int e = 0, i = 0; e < ne; i += b->span[e], ++e)
      if (b->phase[e] == OMNI_PHASE_PREFILL)
        prefix_lookup(st, seq_for(st, b->seq_id[e]), b->pos0[e], b->span[e], b->tokens + i);
  // every entry's pages first: a failure leaves the step unlaunched
  for (int e = 0; e < ne; ++e) ensure_pages(st, seq_for(st, b->seq_id[e]), b->pos0[e] + b->span[e]);
  OMNI_REQUIRE(st->pending_deltas.size() <= lay.cap_delta, OMNI_E_OOM,
               "more page assignments than one step's page-table delta holds");
  auto* ents = reinterpret_cast<ArEntryDesc*>(st->desc.host);
  auto* rows = reinterpret_cast<ArRowDesc*>(st->desc.host + lay.off_rows);
  auto* dec = reinterpret_cast<int32_t*>(st->desc.host + lay.off_dec);
  auto* blks = reinterpret_cast<AttnBlockDesc*>(st->desc.host + lay.off_blk);
  auto* dh = reinterpret_cast<PageDeltaHeader*>(st->desc.host + lay.off_delta);
  auto* dl = reinterpret_cast<PageDelta*>(st->desc.host + lay.off_delta + sizeof(PageDeltaHeader));
  int n_blocks = 0, n_groups = 0;
  std::vector<int> dec_list;
  int r = 0, ir = 0, de = 0, n_prefill_rows = 0;
  for (int e = 0; e < ne; ++e, ir += b->span[e - 1]) {
    SeqSlot& s = st->seqs.at(b->seq_id[e]);
    const bool is_dec = b->phase[e] == OMNI_PHASE_DECODE;
    // prefill positions below cached_upto come from the prefix cache: the
    // device runs only [pos0, pos0 + span) past them (prefill emits nothing,
    // so the trim is invisible to the caller)
    const int skip = is_dec ? 0 : std::clamp(s.cached_upto - b->pos0[e], 0, b->span[e]);
    const int pos0 = b->pos0[e] + skip, span = b->span[e] - skip, ir0 = ir + skip;
    st->prefix.hit_tokens += skip;
    if (span == 0) continue;  // the whole prefill span was cached
    ArEntryDesc& ed = ents[de];
    ed.slot = s.slot;
    ed.q_len = span;
    ed.pos0 = pos0;
    ed.row0 = r;
    ed.is_decode = is_dec ? 1 : 0;
    ed.out_index = is_dec ? b->out_index[e] : -1;
    ed.dec_row = is_dec ? (int)dec_list.size() : -1;
    ed.key = (int32_t)(uint32_t)mix64(b->seq_id[e]);
    if (is_dec) {
      if (!talker)
        OMNI_REQUIRE(ed.out_index >= 0 && ed.out_index < st->ring_rows, OMNI_E_BADARG,
                     "thinker out_index outside the 64-row hidden ring");
      dec[dec_list.size()] = de;
      dec_list.push_back(e);  // results go back to the caller's entry e
    }
    for (int t0 = 0; t0 < span; t0 += kAttnQTok) {
      const int ntok = std::min(kAttnQTok, span - t0);
      // long contexts: split the keys over P CTAs (flash-decoding), merged
      // in fixed part order by the last arriver. P is a function of this
      // block's own context length only (batch invariance).
      const int n_chunks = (pos0 + t0 + ntok + 127) / 128;
      const int parts = std::min(kAttnMaxParts, (n_chunks + kAttnSplitChunks - 1) / kAttnSplitChunks);
      if (parts > 1 && st->split_part) {
        OMNI_REQUIRE(n_groups < st->split_groups, OMNI_E_BADARG, "split-KV groups exhausted");
        for (int pp = 0; pp < parts; ++pp)
          blks[n_blocks++] = AttnBlockDesc{de, t0, ntok, attn_split_pack(pp, parts, n_groups)};
        ++n_groups;
      } else {
        blks[n_blocks++] = AttnBlockDesc{de, t0, ntok, 0};
      }
    }
    for (int t = 0; t < span; ++t, ++r) {
      const int i = ir0 + t;  // caller's token row
      ArRowDesc& rd = rows[r];
      rd.entry = de;
      rd.pos = pos0 + t;
      rd.token = b->tokens[i];
      rd.cond_row = talker ? b->cond_row[i] : 0;
      rd.slot = s.slot;
      rd.pad = 0;
      rd.cond_src = (talker && !is_dec && b->cond_src) ? b->cond_src[i] : 0;
      if (talker) {
        OMNI_REQUIRE(rd.cond_row >= 0 && rd.cond_row < st->cond_rows, OMNI_E_BADARG,
                     "talker cond_row outside the 64-row conditioning table");
        if (!is_dec) {
          OMNI_REQUIRE(rd.cond_src != 0, OMNI_E_BADARG, "talker prefill token without hidden row");
          ++n_prefill_rows;
        }
      }
      OMNI_REQUIRE(rd.token >= -1 && rd.token < (talker && is_dec ? st->m.vocab : 256),
                   OMNI_E_BADARG, "input token id out of range");
    }
    ++de;
  }
  n_rows = r;
  // full prompt pages this step computes become cache entries (reads of
  // them by later steps are ordered on this stream)
  if (st->prefix.enabled)
    for (int e = 0; e < ne; ++e)
      if (b->phase[e] == OMNI_PHASE_PREFILL) prefix_insert(st, st->seqs.at(b->seq_id[e]), b->pos0[e] + b->span[e]);
  // page assignments since the previous step (applied by the step's first kernel)
  dh->n = (int32_t)st->pending_deltas.size();
  for (size_t i = 0; i < st->pending_deltas.size(); ++i) dl[i] = st->pending_deltas[i];
  st->pending_deltas.clear();
  const int n_dec = (int)dec_list.size();
  cudaStream_t s = st->stream;
  OMNI_CUDA(cudaEventRecord(st->ev_start, s));
  counters().h2d_bytes += align16(lay.off_blk + (size_t)n_blocks * sizeof(AttnBlockDesc)) + sizeof(PageDeltaHeader) +
                          dh->n * sizeof(PageDelta);
  const ArStepDev sd = ar_step_dev(st, lay);
  if (n_rows > 0) {
    const uint64_t key = ar_graph_key(n_rows, n_blocks, n_dec, talker && n_prefill_rows > 0);
    run_graph(st, key, [&] { launch_ar_kernels(st, sd, n_rows, n_blocks, n_dec, talker && n_prefill_rows > 0); });
    OMNI_CUDA(cudaEventRecord(st->desc.in_use, s));  // staging read by the step's first kernel
    if (n_dec > 0) counters().d2h_bytes += n_dec * (sizeof(int32_t) + sizeof(float));
  } else if (dh->n > 0) {
    // no rows to run but pages were assigned: keep them pending for the next step
    for (int i = 0; i < dh->n; ++i) st->pending_deltas.push_back(dl[i]);
  }
  OMNI_CUDA(cudaEventRecord(st->ev_done, s));
  st->pending = true;
  st->pending_kind = 1;
  st->pending_dec_entries = std::move(dec_list);
  st->pending_entries = ne;
  st->user_tok = tok_out;
  st->user_margin = margin_out;
}

// ---------------------------------------------------------------------------
// DiT step
// ---------------------------------------------------------------------------
// Persistent grid of a fused DiT iteration of nt (padded) tokens. Beside AR
// stages the DiT holds `dit_ctas` SMs (its share) for small batches and grows
// with the batch -- one CTA per kDitTokPerCta tokens, up to every SM --
// because a big iteration on a small share lands late on every request's tail.
// A function of nt alone: graphs stay keyed by nt, and outputs do not depend
// on the grid. Pipeline req/s (profiles/r02_dit_sm_share.txt), fixed share 48
// vs tokens per CTA 4 / 3 / 2 / 1: c16 216 / 219 / 224-229 / 228 / 207,
// c64 279 / 346 / 348 / 341 / 314.
constexpr int kDitTokPerCta = 3;
int dit_ctas_for(const omni_stage* st, int64_t nt) {
  if (st->dit_ctas >= st->dit_sms_all) return st->dit_ctas;
  return (int)std::min<int64_t>(st->dit_sms_all, std::max<int64_t>(st->dit_ctas, nt / kDitTokPerCta));
}

bool dit_fused_enabled() {  // OMNI_DIT_FUSED=0: one kernel per op (A/B only)
  static const bool on = [] {
    const char* e = std::getenv("OMNI_DIT_FUSED");
    return !(e && e[0] == '0');
  }();
  return on;
}

// The whole iteration as one persistent dataflow kernel (dit_fused.cu): noise
// + counter reset, then T Euler steps x L layers in ONE launch.
void dit_chunk_fused(omni_stage* st, const DitTokDesc* toks_dev, int n_tok, int32_t* samples_dev) {
  const auto& m = st->m;
  const int d = m.d_model, L = m.n_layers, C = m.dit_channels, S = kDitSamples;
  const int ctas = dit_ctas_for(st, n_tok);
  const int tile_rows = dit_tile_rows(n_tok, ctas);
  const int n_rt = n_tok * S / tile_rows, nfd = d / kDitFeat;
  cudaStream_t s = st->stream;
  OMNI_KERNEL(dit_noise(toks_dev, n_tok, S, C, st->seed ^ kNoiseSeedSalt, st->dx, st->dxin, s, st->dctl,
                        n_rt + 6 * n_rt * nfd + 1));
  DitFusedParams p{};
  p.maps = st->dmaps;
  p.toks = toks_dev;
  p.pos_emb = st->pos_emb.p;
  p.mod_table = st->mod_table;
  p.x = st->dx;
  p.xb = st->dxin;
  p.h = st->dh;
  p.a = st->da;
  p.qkv = st->dqkv;
  p.o = st->dout;
  p.u = st->du;
  p.part = st->dpart;
  p.part2 = st->dpart + (size_t)2 * n_rt * nfd * tile_rows * kDitFeat;
  p.samples = samples_dev;
  p.progress = st->dctl;
  p.tile_cnt = st->dctl + n_rt;
  p.ready = st->dctl + n_rt + 2 * n_rt * nfd;
  p.tile_cnt2 = st->dctl + n_rt + 4 * n_rt * nfd;
  p.ready2 = st->dctl + n_rt + 5 * n_rt * nfd;
  p.next_item = st->dctl + n_rt + 6 * n_rt * nfd;
  p.n_rt = n_rt;
  p.tile_rows = tile_rows;
  p.d = d;
  p.C = C;
  p.H = m.n_heads;
  p.ff = m.d_ff;
  p.L = L;
  p.T = m.dit_steps;
  p.vocab = m.vocab;
  p.down_split = st->down_split;
  p.dt = 1.f / m.dit_steps;
  p.sample_scale = kSampleScale;
  p.trace = st->dit_trace;
  OMNI_KERNEL(dit_fused_run(p, st->dit_stages, ctas, s));
}

void dit_chunk(omni_stage* st, const DitTokDesc* toks_dev, int n_tok, int32_t* samples_dev) {
  const auto& m = st->m;
  if (dit_fused_enabled() && dit_fused_supported(m.d_model, m.dit_channels, m.n_heads, m.d_ff, m.n_layers, m.dit_steps))
    return dit_chunk_fused(st, toks_dev, n_tok, samples_dev);
  const int d = m.d_model, L = m.n_layers, C = m.dit_channels, S = kDitSamples, T = m.dit_steps;
  const int rows = n_tok * S;
  const int ld_mod = L * 6 * d;
  cudaStream_t s = st->stream;
  OMNI_KERNEL(dit_noise(toks_dev, n_tok, S, C, st->seed ^ kNoiseSeedSalt, st->dx, st->dxin, s));
  for (int t = 0; t < T; ++t) {
    // adaLN rows of this Euler step: table[t][id] (no per-step gather)
    const float* mod_t = st->mod_table + (size_t)t * m.vocab * ld_mod;
    const int32_t* tok_ids = &toks_dev[0].id;
    constexpr int kIdStride = sizeof(DitTokDesc) / sizeof(int32_t);
    GemmEpilogue e;
    e.out = st->dh;
    e.ldo = d;
    e.row_bias = st->pos_emb.p;  // h = W_in x + pos_emb[sample] (fused)
    e.bias_period = S;
    OMNI_KERNEL(gemm_run(st->g_in, st->din_x, rows, EPI_F32, e, s));
    for (int l = 0; l < L; ++l) {
      const auto& ly = st->dlayers[l];
      const int base = l * 6 * d;
      OMNI_KERNEL(dit_ln_mod(st->dh, rows, d, mod_t, toks_dev, ld_mod, base + 0, base + d, S, st->da, s));
      e = GemmEpilogue{};
      e.out = st->dqkv;
      e.ldo = 3 * d;
      OMNI_KERNEL(gemm_run(ly.gqkv, st->din_a, rows, EPI_BF16, e, s));
      OMNI_KERNEL(dit_attn(st->dqkv, n_tok, d, m.n_heads, st->dout, s));
      e = GemmEpilogue{};
      e.out = st->dh;
      e.ldo = d;
      e.gate = mod_t;
      e.ldg = ld_mod;
      e.gate_off = base + 2 * d;
      e.rows_per_group = S;
      e.gate_index = tok_ids;
      e.gate_index_stride = kIdStride;
      OMNI_KERNEL(gemm_run(ly.go, st->din_o, rows, EPI_GATED_RESID, e, s));
      OMNI_KERNEL(dit_ln_mod(st->dh, rows, d, mod_t, toks_dev, ld_mod, base + 3 * d, base + 4 * d, S, st->da, s));
      GemmEpilogue e1;
      e1.out = st->du;
      e1.ldo = m.d_ff;
      OMNI_KERNEL(gemm_run(ly.g1, st->din_a, rows, EPI_GELU, e1, s));
      e.gate_off = base + 5 * d;
      OMNI_KERNEL(gemm_run(ly.g2, st->din_u, rows, EPI_GATED_RESID, e, s));
    }
    OMNI_KERNEL(dit_ln_mod(st->dh, rows, d, nullptr, toks_dev, 0, 0, 0, S, st->da, s));
    // output projection with the Euler update fused: x += dt * v, next
    // step's bf16 input, and on the last step the int32 samples
    GemmEpilogue eo;
    eo.out = st->dx;
    eo.ldo = C;
    eo.xb = st->dxin;
    eo.dt = 1.f / T;
    eo.sample_scale = kSampleScale;
    eo.samples = t == T - 1 ? samples_dev : nullptr;
    OMNI_KERNEL(gemm_run(st->g_out, st->din_a, rows, EPI_EULER, eo, s));
  }
}

constexpr int kDitPadTok = kDitTileTok;  // DiT batches are padded to whole 128-row tiles (8 tokens)
// ... and to whole 256-row tiles once dit_tile_rows picks them
int64_t dit_pad_tokens(const omni_stage* st, int64_t n) {
  if (n == 0) return 0;
  const int64_t p8 = (n + kDitPadTok - 1) / kDitPadTok * kDitPadTok;
  return p8 >= dit_ctas_for(st, p8) ? (n + 15) / 16 * 16 : p8;
}
uint64_t dit_graph_key(int nt, int64_t t0) { return (uint64_t)nt << 20 | (uint64_t)t0; }

// Capture the DiT step graph of every padded batch size up front
// (OMNI_PREWARM caps the token count too; 0 = off).
void prewarm_dit_graphs(omni_stage* st) {
  if (!graphs_enabled()) return;
  static const int cap_env = [] {
    const char* e = std::getenv("OMNI_PREWARM");
    return e ? std::atoi(e) * kDitPadTok : -1;
  }();
  int upto = st->tok_cap;
  if (cap_env >= 0) upto = std::min(upto, cap_env);
  if (upto < kDitPadTok) return;
  if (staging_reserve(st->desc, align16((size_t)st->tok_cap * sizeof(DitTokDesc)))) drop_graphs(st);
  const auto* toks_dev = reinterpret_cast<const DitTokDesc*>(st->desc.dev);
  for (int nt = kDitPadTok; nt <= upto; nt += kDitPadTok) {
    if (dit_pad_tokens(st, nt) != nt) continue;  // not a padded size
    const uint64_t key = dit_graph_key(nt, 0);
    if (!st->graphs.count(key))
      capture_graph(st, key, [&] {
        OMNI_KERNEL(launch_desc_copy(st->desc.dev, st->desc.host, (size_t)nt * sizeof(DitTokDesc), nullptr, nullptr,
                                     st->stream));
        dit_chunk(st, toks_dev, nt, st->dsamples);
      });
  }
}

void dit_step(omni_stage* st, const omni_dit_batch* b, int32_t* samples_out) {
  ensure_idle(st);
  OMNI_REQUIRE(st->m.kind == OMNI_MODEL_DIT, OMNI_E_BADARG, "not a DiT stage");
  int64_t n_tok = 0;
  for (int j = 0; j < b->n_jobs; ++j) {
    OMNI_REQUIRE(b->n_tokens[j] >= 0 && b->token_offset[j] >= 0, OMNI_E_BADARG, "bad DiT job");
    n_tok += b->n_tokens[j];
  }
  // Pad the batch to a multiple of kDitPadTok tokens (= 128 rows, a whole
  // GEMM token tile: no extra MMA work) with dummy tokens whose rows are
  // computed and dropped. Rows never interact (token-local DiT), so real
  // outputs are unchanged, and the step-graph geometries shrink 8x (all
  // prewarmed at stage creation).
  const int64_t n_pad = dit_pad_tokens(st, n_tok);
  const size_t bytes = align16((size_t)n_pad * sizeof(DitTokDesc));
  if (staging_reserve(st->desc, std::max(bytes, align16((size_t)st->tok_cap * sizeof(DitTokDesc)))))
    drop_graphs(st);
  auto* toks = reinterpret_cast<DitTokDesc*>(st->desc.host);
  int64_t k = 0;
  for (int j = 0; j < b->n_jobs; ++j)
    for (int i = 0; i < b->n_tokens[j]; ++i, ++k) {
      const int id = b->tokens[k];
      OMNI_REQUIRE(id >= 0 && id < st->m.vocab, OMNI_E_BADARG,
                   "DiT conditioning id out of range (the reference demands I32 codec tokens, "
                   "diffusion_engine.hpp:29-30)");
      toks[k] = DitTokDesc{b->request_id[j], b->token_offset[j] + i, id};
    }
  for (; k < n_pad; ++k) toks[k] = DitTokDesc{0, 0, 0};
  cudaStream_t s = st->stream;
  OMNI_CUDA(cudaEventRecord(st->ev_start, s));
  if (n_tok > 0) {
    // descriptors: copied from pinned staging by the chunk graph's first kernel
    counters().h2d_bytes += bytes;
    const auto* toks_dev = reinterpret_cast<const DitTokDesc*>(st->desc.dev);
    for (int64_t t0 = 0; t0 < n_tok; t0 += st->tok_cap) {
      const int nt = (int)std::min<int64_t>(st->tok_cap, n_pad - t0);
      run_graph(st, dit_graph_key(nt, t0), [&] {
        OMNI_KERNEL(launch_desc_copy(st->desc.dev + t0 * sizeof(DitTokDesc), st->desc.host + t0 * sizeof(DitTokDesc),
                                     (size_t)nt * sizeof(DitTokDesc), nullptr, nullptr, s));
        dit_chunk(st, toks_dev + t0, nt, st->dsamples);
      });
      if (t0 + st->tok_cap >= n_tok) OMNI_CUDA(cudaEventRecord(st->desc.in_use, s));
      const int64_t nsamp = std::min<int64_t>(nt, n_tok - t0) * kDitSamples;  // real tokens only
      if (st->dsamples != st->h_samples)
        OMNI_CUDA(cudaMemcpyAsync(st->h_samples, st->dsamples, nsamp * sizeof(int32_t),
                                  cudaMemcpyDeviceToHost, s));
      counters().d2h_bytes += nsamp * sizeof(int32_t);
      if (n_tok > st->tok_cap) {  // multi-chunk: land each chunk before reusing h_samples
        OMNI_CUDA(cudaStreamSynchronize(s));
        std::memcpy(samples_out + t0 * kDitSamples, st->h_samples, nsamp * sizeof(int32_t));
      }
    }
  }
  OMNI_CUDA(cudaEventRecord(st->ev_done, s));
  st->pending = true;
  st->pending_kind = 2;
  st->user_samples = (n_tok > st->tok_cap) ? nullptr : samples_out;
  st->pending_samples = n_tok * kDitSamples;
}

void finish_pending(omni_stage* st) {
  if (!st->pending) return;
  st->pending = false;
  if (st->pending_kind == 1) {
    if (st->user_tok || st->user_margin) {
      for (int e = 0; e < st->pending_entries; ++e) {
        if (st->user_tok) st->user_tok[e] = -1;
        if (st->user_margin) st->user_margin[e] = 0.f;
      }
      for (size_t i = 0; i < st->pending_dec_entries.size(); ++i) {
        const int e = st->pending_dec_entries[i];
        if (st->user_tok) st->user_tok[e] = st->h_tok[i];
        if (st->user_margin) st->user_margin[e] = reinterpret_cast<const float*>(st->h_tok)[st->pending_dec_entries.size() + i];
      }
    }
  } else if (st->pending_kind == 2 && st->user_samples) {
    std::memcpy(st->user_samples, st->h_samples, st->pending_samples * sizeof(int32_t));
  }
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, st->ev_start, st->ev_done) == cudaSuccess) st->last_step_us = ms * 1e3f;
}

std::mutex g_init_mu;

}  // namespace

struct omni_arena {
  int dev = 0;
  uint8_t* base = nullptr;
  uint64_t bytes = 0;
  bool imported = false;  // mapped from another process (cudaIpcOpenMemHandle)
};

struct omni_ipc_event {
  int dev = 0;
  cudaEvent_t ev = nullptr;
};

extern "C" {

omni_status omni_init(int32_t n_dev, const int32_t* dev_ids) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_init_mu);
    require_device();
    std::vector<int> ids;
    if (n_dev <= 0) ids.push_back(0);
    for (int i = 0; i < n_dev; ++i) ids.push_back(dev_ids[i]);
    for (int a : ids) {
      OMNI_CUDA(cudaSetDevice(a));
      int major = 0;
      OMNI_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, a));
      OMNI_REQUIRE(major == 10, OMNI_E_NOGPU, "libomni_dev is built for sm_100a only");
      for (int b : ids) {
        if (a == b) continue;
        int can = 0;
        OMNI_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
        if (can) {
          cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else OMNI_CUDA(e);
        }
      }
    }
    OMNI_CUDA(cudaSetDevice(ids[0]));
  });
}

omni_status omni_model_default(int32_t kind, omni_model_desc* out) {
  return guarded([&] {
    omni_model_desc m{};
    m.kind = kind;
    m.head_dim = 128;
    if (kind == OMNI_MODEL_THINKER || kind == OMNI_MODEL_TALKER) {
      m.d_model = 2048;
      m.n_layers = kind == OMNI_MODEL_THINKER ? 8 : 4;
      m.n_heads = 16;
      m.n_kv_heads = 4;
      m.d_ff = 8192;
      m.vocab = kind == OMNI_MODEL_THINKER ? 256 : 64;
      m.cond_dim = kind == OMNI_MODEL_TALKER ? 2048 : 0;
    } else if (kind == OMNI_MODEL_DIT) {
      m.d_model = 1024;
      m.n_layers = 4;
      m.n_heads = 8;
      m.n_kv_heads = 8;
      m.d_ff = 4096;
      m.vocab = 256;
      m.dit_channels = 64;
      m.dit_samples = 16;
      m.dit_steps = 4;
    } else {
      throw DevError(OMNI_E_BADARG, "unknown model kind");
    }
    *out = m;
  });
}

omni_status omni_stage_create(const omni_model_desc* model, const omni_stage_limits* limits,
                              int32_t dev, uint64_t weight_seed, omni_stage** out) {
  omni_stage* st = nullptr;
  omni_status rc = guarded([&] {
    require_device();
    OMNI_REQUIRE(model && limits && out, OMNI_E_BADARG, "null argument");
    st = new omni_stage();
    st->m = *model;
    st->lim = *limits;
    st->dev = dev;
    st->seed = weight_seed;
    if (st->lim.max_batch_tokens <= 0) st->lim.max_batch_tokens = 256;
    if (st->lim.max_resident <= 0) st->lim.max_resident = 64;
    if (st->lim.max_seq_len <= 0) st->lim.max_seq_len = 512;
    if (st->lim.dit_max_tokens <= 0) st->lim.dit_max_tokens = 512;
    OMNI_CUDA(cudaSetDevice(dev));
    // Stream priority by stage kind when stages share a GPU. OMNI_PRIO = three
    // digits, the urgency rank (0 = most urgent) of thinker / talker / DiT.
    // Default "001": both AR chains above the DiT. With the fused DiT on a
    // batch-sized share, Thinker and Talker at equal rank beat Talker-first
    // ("101", round 1's winner) by ~4 % at c16 and ~11 % at c64
    // (profiles/r02_stream_priority.txt).
    int lo = 0, hi = 0;
    OMNI_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));  // hi = numerically lowest = most urgent
    const char* pe = std::getenv("OMNI_PRIO");
    const char* ranks = (pe && std::strlen(pe) == 3) ? pe : "001";
    const int kind_ix = model->kind == OMNI_MODEL_THINKER ? 0 : model->kind == OMNI_MODEL_TALKER ? 1 : 2;
    const int rank = std::clamp(ranks[kind_ix] - '0', 0, 2);
    const int prio = hi + (lo - hi) * rank / 2;
    OMNI_CUDA(cudaStreamCreateWithPriority(&st->stream, cudaStreamNonBlocking, prio));
    OMNI_CUDA(cudaEventCreate(&st->ev_start));
    OMNI_CUDA(cudaEventCreate(&st->ev_done));
    OMNI_CUDA(cudaEventCreateWithFlags(&st->ev_link, cudaEventDisableTiming));
    OMNI_CUDA(cudaEventCreateWithFlags(&st->ev_pack, cudaEventDisableTiming));
    if (model->kind == OMNI_MODEL_DIT) {
      build_dit(st);
      prewarm_dit_graphs(st);
    }
    else if (model->kind == OMNI_MODEL_THINKER || model->kind == OMNI_MODEL_TALKER) {
      build_ar(st);
      prewarm_decode_graphs(st);
    }
    else throw DevError(OMNI_E_BADARG, "unknown model kind");
    *out = st;
  });
  if (rc != OMNI_OK && st) destroy_stage(st);
  return rc;
}

omni_status omni_stage_destroy(omni_stage* st) {
  return guarded([&] { destroy_stage(st); });
}

omni_status omni_stage_weight_bytes(const omni_stage* st, uint64_t* bytes) {
  return guarded([&] { *bytes = st->weight_bytes; });
}

omni_status omni_stage_tensor(const omni_stage* st, const char* name, uint64_t* dev_ptr, int64_t* rows,
                              int64_t* cols) {
  return guarded([&] {
    const std::string n(name ? name : "");
    auto it = st->named.find(n);
    if (it != st->named.end()) {
      *dev_ptr = reinterpret_cast<uint64_t>(it->second.p);
      if (rows) *rows = it->second.rows_pad;
      if (cols) *cols = it->second.cols;
      return;
    }
    if (n == "buf.logits") {
      *dev_ptr = reinterpret_cast<uint64_t>(st->logits);
      if (rows) *rows = st->rows_cap;
      if (cols) *cols = st->vocab_pad;
      return;
    }
    if (n == "buf.dit_x") {
      *dev_ptr = reinterpret_cast<uint64_t>(st->dx);
      if (rows) *rows = st->drows_cap;
      if (cols) *cols = st->m.dit_channels;
      return;
    }
    if (n == "buf.hproj" && st->hproj) {
      *dev_ptr = reinterpret_cast<uint64_t>(st->hproj);
      if (rows) *rows = st->rows_cap;
      if (cols) *cols = st->m.d_model;
      return;
    }
    if (n == "buf.dit_trace" && st->dit_trace) {  // OMNI_DIT_TRACE=1: [item][5] u64 of the last DiT chunk
      *dev_ptr = reinterpret_cast<uint64_t>(st->dit_trace);
      if (rows) *rows = st->dit_trace_items;
      if (cols) *cols = 8;
      return;
    }
    if (n == "buf.step_trace" && st->step_trace) {  // OMNI_STEP_TRACE=1: [launch][cta][8] u64
      *dev_ptr = reinterpret_cast<uint64_t>(st->step_trace);
      if (rows) *rows = kStepTraceLaunches * kStepTraceCtas;
      if (cols) *cols = 8;
      return;
    }
    if (n == "buf.x") {
      *dev_ptr = reinterpret_cast<uint64_t>(st->x);
      if (rows) *rows = st->rows_cap;
      if (cols) *cols = st->m.d_model;
      return;
    }
    // bf16 activations of the last step (debug / tests): name -> (ptr, cols)
    const std::pair<const char*, std::pair<const void*, int64_t>> bf[] = {
        {"buf.xn", {st->xn, st->m.d_model}},
        {"buf.q", {st->q, (int64_t)st->m.n_heads * kHeadDim}},
        {"buf.attn", {st->attn, (int64_t)st->m.n_heads * kHeadDim}},
        {"buf.act", {st->act, st->m.d_ff}},
        {"buf.hbuf", {st->hbuf, st->m.d_model}},
        {"buf.ss", {st->ss, st->m.d_model / 128}}};
    for (const auto& [nm, pc] : bf)
      if (n == nm && pc.first) {
        *dev_ptr = reinterpret_cast<uint64_t>(pc.first);
        if (rows) *rows = st->rows_cap;
        if (cols) *cols = pc.second;
        return;
      }
    throw DevError(OMNI_E_BADARG, "unknown tensor " + n);
  });
}

omni_status omni_ar_step(omni_stage* st, const omni_ar_batch* batch, int32_t* token_out,
                         float* margin_out) {
  return guarded([&] {
    OMNI_REQUIRE(st && batch, OMNI_E_BADARG, "null argument");
    OMNI_REQUIRE(st->m.kind != OMNI_MODEL_DIT, OMNI_E_BADARG, "omni_ar_step on a DiT stage");
    OMNI_CUDA(cudaSetDevice(st->dev));
    ar_step(st, batch, token_out, margin_out);
  });
}

omni_status omni_seq_release(omni_stage* st, uint64_t seq_id) {
  return guarded([&] {
    auto it = st->seqs.find(seq_id);
    if (it == st->seqs.end()) return;
    // Pages may still be read by an in-flight step on this stage's stream;
    // stream order makes reuse by a later step safe.
    for (int p : it->second.pages) page_unref(st, p);
    st->free_slots.push_back(it->second.slot);
    st->seqs.erase(it);
  });
}

omni_status omni_seq_hidden_row(omni_stage* st, uint64_t seq_id, int32_t index, uint64_t* dev_ptr) {
  return guarded([&] {
    OMNI_REQUIRE(st->ring != nullptr, OMNI_E_BADARG, "stage has no hidden ring (not a thinker)");
    auto it = st->seqs.find(seq_id);
    OMNI_REQUIRE(it != st->seqs.end(), OMNI_E_BADARG, "unknown sequence");
    OMNI_REQUIRE(index >= 0 && index < st->ring_rows, OMNI_E_BADARG, "hidden row index");
    *dev_ptr = reinterpret_cast<uint64_t>(
        st->ring + ((size_t)it->second.slot * st->ring_rows + index) * st->m.d_model);
  });
}

omni_status omni_dit_step(omni_stage* st, const omni_dit_batch* batch, int32_t* samples_out) {
  return guarded([&] {
    OMNI_REQUIRE(st && batch, OMNI_E_BADARG, "null argument");
    OMNI_CUDA(cudaSetDevice(st->dev));
    dit_step(st, batch, samples_out);
  });
}

omni_status omni_stage_query(omni_stage* st) {
  omni_status rc = OMNI_OK;
  omni_status g = guarded([&] {
    if (!st->pending) return;
    cudaError_t e = cudaEventQuery(st->ev_done);
    if (e == cudaErrorNotReady) {
      rc = OMNI_EAGAIN;
      return;
    }
    OMNI_CUDA(e);
    finish_pending(st);
  });
  return g != OMNI_OK ? g : rc;
}

omni_status omni_stage_wait(omni_stage* st) {
  return guarded([&] {
    if (!st->pending) return;
    OMNI_CUDA(cudaEventSynchronize(st->ev_done));
    finish_pending(st);
  });
}

omni_status omni_stage_last_step_us(omni_stage* st, float* us) {
  return guarded([&] { *us = st->last_step_us; });
}

omni_status omni_arena_create(int32_t dev, uint64_t bytes, omni_arena** out) {
  return guarded([&] {
    require_device();
    auto* a = new omni_arena();
    a->dev = dev;
    a->bytes = bytes;
    OMNI_CUDA(cudaSetDevice(dev));
    cudaError_t e = cudaMalloc(&a->base, bytes);
    if (e != cudaSuccess) {
      delete a;
      throw DevError(OMNI_E_OOM, "arena allocation failed");
    }
    *out = a;
  });
}

omni_status omni_arena_destroy(omni_arena* a) {
  return guarded([&] {
    if (!a) return;
    cudaSetDevice(a->dev);
    cudaDeviceSynchronize();
    if (a->imported)
      cudaIpcCloseMemHandle(a->base);
    else
      cudaFree(a->base);
    delete a;
  });
}

omni_status omni_arena_base(const omni_arena* a, uint64_t* dev_ptr, uint64_t* bytes) {
  return guarded([&] {
    *dev_ptr = reinterpret_cast<uint64_t>(a->base);
    if (bytes) *bytes = a->bytes;
  });
}

uint64_t omni_pack_bytes(int32_t rows, int32_t d) { return pack_blob_bytes(rows, d); }

omni_status omni_pack_hidden(omni_stage* src, int32_t n_chunks, const uint64_t* seq_id,
                             const int32_t* begin, const int32_t* end, const int32_t* tokens,
                             uint64_t dst_base, const uint64_t* dst_offset) {
  return guarded([&] {
    OMNI_REQUIRE(src->ring != nullptr, OMNI_E_BADARG, "pack source is not a thinker stage");
    if (n_chunks <= 0) return;
    OMNI_CUDA(cudaSetDevice(src->dev));
    int total_rows = 0, max_rows = 0;
    for (int c = 0; c < n_chunks; ++c) {
      OMNI_REQUIRE(begin[c] >= 0 && end[c] >= begin[c] && end[c] <= src->ring_rows, OMNI_E_BADARG,
                   "pack row range");
      OMNI_REQUIRE(dst_offset[c] % 16 == 0, OMNI_E_BADARG, "pack destination must be 16-B aligned");
      total_rows += end[c] - begin[c];
      max_rows = std::max(max_rows, end[c] - begin[c]);
    }
    const size_t off_tok = align16((size_t)n_chunks * sizeof(PackChunkDesc));
    const size_t total = off_tok + align16((size_t)std::max(1, total_rows) * sizeof(int32_t));
    if (src->pack.in_use) OMNI_CUDA(cudaEventSynchronize(src->pack.in_use));
    staging_reserve(src->pack, total);
    auto* cd = reinterpret_cast<PackChunkDesc*>(src->pack.host);
    auto* tk = reinterpret_cast<int32_t*>(src->pack.host + off_tok);
    // Production-size packs (a few rows) read their descriptors straight from
    // the pinned staging buffer (UVA): no copy-engine H2D ahead of them on the
    // Thinker stream, where the next step queues behind. Large packs copy
    // them to the device first: small PCIe reads are throughput-limited
    // (profiles/r02_pack_large.txt).
    const bool copy_first = total_rows > kPackUvaRows;
    const uint8_t* desc_base = copy_first ? src->pack.dev : src->pack.host;
    const auto* tk_dev = reinterpret_cast<const int32_t*>(desc_base + off_tok);
    int at = 0;
    for (int c = 0; c < n_chunks; ++c) {
      auto it = src->seqs.find(seq_id[c]);
      OMNI_REQUIRE(it != src->seqs.end(), OMNI_E_BADARG, "pack of unknown sequence");
      cd[c] = PackChunkDesc{it->second.slot, begin[c], end[c], 0, dst_offset[c], tk_dev + at};
      for (int r = begin[c]; r < end[c]; ++r, ++at) tk[at] = tokens[at];
    }
    cudaStream_t s = src->stream;
    counters().h2d_bytes += total;
    if (copy_first) OMNI_CUDA(cudaMemcpyAsync(src->pack.dev, src->pack.host, total, cudaMemcpyHostToDevice, s));
    OMNI_KERNEL(launch_pack_hidden(reinterpret_cast<const PackChunkDesc*>(desc_base), n_chunks, max_rows,
                                 src->ring, src->m.d_model, src->ring_rows, reinterpret_cast<uint8_t*>(dst_base),
                                 copy_first, s));
    OMNI_CUDA(cudaEventRecord(src->pack.in_use, s));  // staging read by the kernel
    // consumers wait for exactly this pack (omni_stage_after_pack), not for
    // whatever the producer enqueues after it (its next step)
    OMNI_CUDA(cudaEventRecord(src->ev_pack, s));
    src->pack_recorded = true;
  });
}

omni_status omni_stage_after_pack(omni_stage* dst, omni_stage* src) {
  return guarded([&] {
    OMNI_REQUIRE(dst && src, OMNI_E_BADARG, "null stage");
    if (!src->pack_recorded) return;
    OMNI_CUDA(cudaSetDevice(dst->dev));
    OMNI_CUDA(cudaStreamWaitEvent(dst->stream, src->ev_pack, 0));  // cross-device waits are legal
  });
}

omni_status omni_seq_reserve(omni_stage* st, uint64_t seq_id, int32_t upto_tokens) {
  return guarded([&] {
    OMNI_REQUIRE(st && st->m.kind != OMNI_MODEL_DIT, OMNI_E_BADARG, "omni_seq_reserve needs an AR stage");
    OMNI_REQUIRE(upto_tokens >= 0, OMNI_E_BADARG, "negative token count");
    ensure_pages(st, seq_for(st, seq_id), upto_tokens);
  });
}

omni_status omni_seq_reserve_prompt(omni_stage* st, uint64_t seq_id, int32_t pos0, int32_t span,
                                    const int32_t* tokens) {
  return guarded([&] {
    OMNI_REQUIRE(st && st->m.kind != OMNI_MODEL_DIT, OMNI_E_BADARG, "omni_seq_reserve_prompt needs an AR stage");
    OMNI_REQUIRE(pos0 >= 0 && span >= 0 && (span == 0 || tokens), OMNI_E_BADARG, "bad prompt span");
    SeqSlot& s = seq_for(st, seq_id);
    if (st->prefix.enabled && span > 0) prefix_lookup(st, s, pos0, span, tokens);
    ensure_pages(st, s, pos0 + span);
  });
}

omni_status omni_stage_set_sm_share(omni_stage* st, int32_t sms) {
  return guarded([&] {
    OMNI_REQUIRE(st && st->m.kind == OMNI_MODEL_DIT, OMNI_E_BADARG, "the SM share applies to DiT stages");
    ensure_idle(st);
    int n = 0;
    OMNI_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, st->dev));
    const int want = sms <= 0 ? n : std::min(sms, n);
    if (want != st->dit_ctas) drop_graphs(st);  // the grid size is baked into the step graphs
    st->dit_ctas = want;
    st->dit_sms_all = n;
    prewarm_dit_graphs(st);
  });
}

omni_status omni_stage_set_prefix_cache(omni_stage* st, int32_t enable) {
  return guarded([&] {
    OMNI_REQUIRE(st && st->m.kind == OMNI_MODEL_THINKER, OMNI_E_BADARG,
                 "the prefix cache applies to Thinker stages (KV a function of the prompt alone)");
    OMNI_REQUIRE(st->seqs.empty(), OMNI_E_BADARG, "toggle the prefix cache with no resident sequence");
    ensure_idle(st);
    if (!enable) prefix_evict(st);  // every cached page is held by the cache alone now
    st->prefix.enabled = enable != 0;
  });
}

omni_status omni_stage_prefix_stats(const omni_stage* st, uint64_t* hit_tokens, uint64_t* cached_pages,
                                    uint64_t* evicted_pages) {
  return guarded([&] {
    if (hit_tokens) *hit_tokens = st->prefix.hit_tokens;
    if (cached_pages) *cached_pages = st->prefix.key_of.size();
    if (evicted_pages) *evicted_pages = st->prefix.evicted_pages;
  });
}

omni_status omni_stage_set_sampling(omni_stage* st, int32_t top_k, uint64_t seed) {
  return guarded([&] {
    OMNI_REQUIRE(st && st->m.kind != OMNI_MODEL_DIT, OMNI_E_BADARG, "sampling applies to AR stages");
    OMNI_REQUIRE(top_k >= 0 && top_k <= 32, OMNI_E_BADARG, "top_k must be in [0, 32]");
    ensure_idle(st);
    if (st->top_k != top_k || st->sample_seed != seed) drop_graphs(st);  // both are baked into step graphs
    st->top_k = top_k;
    st->sample_seed = seed;
    if (top_k > 1) prewarm_decode_graphs(st);
  });
}

omni_status omni_arena_export(const omni_arena* a, omni_ipc_handle* out) {
  return guarded([&] {
    OMNI_REQUIRE(a && out && !a->imported, OMNI_E_BADARG, "only an arena this process allocated can be exported");
    static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(out->handle), "IPC handle size");
    cudaIpcMemHandle_t h;
    OMNI_CUDA(cudaSetDevice(a->dev));
    OMNI_CUDA(cudaIpcGetMemHandle(&h, a->base));
    std::memcpy(out->handle, &h, sizeof(h));
    out->bytes = a->bytes;
    out->dev = a->dev;
    out->reserved = 0;
  });
}

omni_status omni_arena_import(const omni_ipc_handle* h, omni_arena** out) {
  return guarded([&] {
    require_device();
    OMNI_REQUIRE(h && out, OMNI_E_BADARG, "null IPC handle");
    int n = 0;
    OMNI_CUDA(cudaGetDeviceCount(&n));
    OMNI_REQUIRE(h->dev >= 0 && h->dev < n, OMNI_E_BADARG, "IPC arena on a device this process cannot see");
    cudaIpcMemHandle_t mh;
    std::memcpy(&mh, h->handle, sizeof(mh));
    OMNI_CUDA(cudaSetDevice(h->dev));
    void* base = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&base, mh, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw DevError(OMNI_E_TRANSPORT, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    }
    auto* a = new omni_arena();
    a->dev = h->dev;
    a->base = static_cast<uint8_t*>(base);
    a->bytes = h->bytes;
    a->imported = true;
    *out = a;
  });
}

omni_status omni_ipc_event_create(int32_t dev, omni_ipc_event** out, omni_ipc_event_handle* handle) {
  return guarded([&] {
    require_device();
    OMNI_REQUIRE(out && handle, OMNI_E_BADARG, "null output");
    static_assert(sizeof(cudaIpcEventHandle_t) == sizeof(handle->handle), "IPC event handle size");
    OMNI_CUDA(cudaSetDevice(dev));
    auto* e = new omni_ipc_event();
    e->dev = dev;
    OMNI_CUDA(cudaEventCreateWithFlags(&e->ev, cudaEventDisableTiming | cudaEventInterprocess));
    // an interprocess event must have been recorded once before a peer waits on it
    OMNI_CUDA(cudaEventRecord(e->ev, 0));
    OMNI_CUDA(cudaEventSynchronize(e->ev));
    cudaIpcEventHandle_t h;
    OMNI_CUDA(cudaIpcGetEventHandle(&h, e->ev));
    std::memcpy(handle->handle, &h, sizeof(h));
    *out = e;
  });
}

omni_status omni_ipc_event_open(int32_t dev, const omni_ipc_event_handle* handle, omni_ipc_event** out) {
  return guarded([&] {
    require_device();
    OMNI_REQUIRE(out && handle, OMNI_E_BADARG, "null IPC event handle");
    cudaIpcEventHandle_t h;
    std::memcpy(&h, handle->handle, sizeof(h));
    OMNI_CUDA(cudaSetDevice(dev));
    auto* e = new omni_ipc_event();
    e->dev = dev;
    const cudaError_t r = cudaIpcOpenEventHandle(&e->ev, h);
    if (r != cudaSuccess) {
      cudaGetLastError();
      delete e;
      throw DevError(OMNI_E_TRANSPORT, std::string("cudaIpcOpenEventHandle: ") + cudaGetErrorString(r));
    }
    *out = e;
  });
}

omni_status omni_ipc_event_destroy(omni_ipc_event* e) {
  return guarded([&] {
    if (!e) return;
    cudaSetDevice(e->dev);
    cudaEventDestroy(e->ev);
    delete e;
  });
}

omni_status omni_stage_record_pack(omni_stage* src, omni_ipc_event* e) {
  return guarded([&] {
    OMNI_REQUIRE(src && e, OMNI_E_BADARG, "null stage / event");
    OMNI_CUDA(cudaSetDevice(src->dev));
    // ordered after the stage's most recent pack (recorded on the same stream
    // right behind it); later steps on the stream are not included only if
    // this is called before they are enqueued -- the connector calls it right
    // after omni_pack_hidden
    OMNI_CUDA(cudaEventRecord(e->ev, src->stream));
  });
}

omni_status omni_stage_wait_event(omni_stage* dst, omni_ipc_event* e) {
  return guarded([&] {
    OMNI_REQUIRE(dst && e, OMNI_E_BADARG, "null stage / event");
    OMNI_CUDA(cudaSetDevice(dst->dev));
    OMNI_CUDA(cudaStreamWaitEvent(dst->stream, e->ev, 0));
  });
}

omni_status omni_ipc_event_sync(omni_ipc_event* e) {
  return guarded([&] {
    OMNI_REQUIRE(e, OMNI_E_BADARG, "null event");
    OMNI_CUDA(cudaEventSynchronize(e->ev));
  });
}

omni_status omni_stage_after(omni_stage* dst, omni_stage* src) {
  return guarded([&] {
    OMNI_CUDA(cudaSetDevice(src->dev));
    OMNI_CUDA(cudaEventRecord(src->ev_link, src->stream));
    OMNI_CUDA(cudaSetDevice(dst->dev));
    OMNI_CUDA(cudaStreamWaitEvent(dst->stream, src->ev_link, 0));
  });
}

}  // extern "C"
