/*
 * ORACLE / TEST INFRASTRUCTURE — CPU fp32 restatement of the B200 stage
 * models. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs load this (oracle/_build/liboracle_models.so); the
 * product never links it.
 *
 * PARITY NOTE: the reference (/root/reference/proj) has NO floating-point
 * model: its Thinker/Talker/vocoder are integer mocks (reference_pipeline.hpp:
 * 20-45) and its denoiser is closed form (diffusion_engine.hpp:28-43). The
 * float path is therefore "parity unpinned" by the reference;
 * this file DEFINES it, keeping the reference's integer semantics around it:
 *   - Thinker: prompt -> L = target_length(fold_prompt) tokens (lengths stay on
 *     the host, reference_pipeline.hpp:24-32), one token per DECODE entry, no
 *     token from prefill (ar_engine.hpp:313-331), alphabet [1,255] (id 0 =
 *     start token, masked; reference_pipeline.hpp:34).
 *   - Talker: 4 codec tokens per text row j = m/4 (reference_pipeline.hpp:
 *     43-45, 133-148), alphabet [0,63], conditioned on (t_j, h_j).
 *   - DiT: 16 samples per codec token, int32 in [-64,63] (diffusion_engine.hpp
 *     :36-41), token-local so output is chunking-invariant (:25-27).
 * Weights come from the counter stream of csrc/dev/rng.h, restated here in C;
 * bf16 rounding happens at the same tensor boundaries as the CUDA kernels and
 * every accumulation is fp32.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- counter RNG (csrc/dev/rng.h restated) ---------------- */
static uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static int32_t irwin4(uint64_t h) {
  return (int32_t)(h & 0xFFFF) + (int32_t)((h >> 16) & 0xFFFF) + (int32_t)((h >> 32) & 0xFFFF) +
         (int32_t)((h >> 48) & 0xFFFF) - 131070;
}
static uint64_t weight_hash(uint64_t seed, uint32_t tid, uint64_t idx) {
  return mix64(seed ^ mix64(((uint64_t)tid << 40) ^ idx));
}
static uint64_t noise_hash(uint64_t seed, uint64_t rid, uint32_t pos, uint32_t s, uint32_t ch) {
  return mix64(seed ^ mix64(rid * 0x100000001B3ull ^ mix64(((uint64_t)pos << 24) ^ ((uint64_t)s << 12) ^ ch)));
}
static float weight_mult(float scale) { return (float)((double)scale * 1.7320508075688772 / 65536.0); }
static const float kNoiseMult = 2.6429027e-05f;
static const uint64_t kNoiseSeedSalt = 0x6e6f697365ull;

/* bf16 round-to-nearest-even, returned as float */
static float bf16r(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return f;
  u += 0x7FFFu + ((u >> 16) & 1u);
  u &= 0xFFFF0000u;
  memcpy(&f, &u, 4);
  return f;
}
static uint16_t bf16bits(float f) {
  float r = bf16r(f);
  uint32_t u;
  memcpy(&u, &r, 4);
  return (uint16_t)(u >> 16);
}
static float from_bits(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

typedef struct {
  int rows, cols;
  uint16_t* w; /* bf16 bits, [rows][cols] */
} Mat;

static Mat mat_gen(int rows, int cols, uint64_t seed, uint32_t tid, float scale) {
  Mat m;
  m.rows = rows;
  m.cols = cols;
  m.w = (uint16_t*)malloc((size_t)rows * cols * 2);
  float mult = weight_mult(scale);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c)
      m.w[r * cols + c] = bf16bits((float)irwin4(weight_hash(seed, tid, (uint64_t)(r * cols + c))) * mult);
  return m;
}
static void mat_free(Mat* m) {
  free(m->w);
  m->w = NULL;
}

/* y[M][N] = x[M][K] . W[N][K]^T  (fp32 accumulate, fixed 16-lane order) */
static void gemm(const float* x, int M, const Mat* W, float* y) {
  const int K = W->cols, N = W->rows;
#pragma omp parallel
  {
    float* wr = (float*)malloc((size_t)K * sizeof(float));
#pragma omp for schedule(static)
    for (int n = 0; n < N; ++n) {
      const uint16_t* src = W->w + (size_t)n * K;
      for (int k = 0; k < K; ++k) wr[k] = from_bits(src[k]);
      for (int m = 0; m < M; ++m) {
        const float* xr = x + (size_t)m * K;
        float acc[16] = {0};
        int k = 0;
        for (; k + 16 <= K; k += 16)
          for (int t = 0; t < 16; ++t) acc[t] += xr[k + t] * wr[k + t];
        float s = 0.f;
        for (int t = 0; t < 16; ++t) s += acc[t];
        for (; k < K; ++k) s += xr[k] * wr[k];
        y[(size_t)m * N + n] = s;
      }
    }
    free(wr);
  }
}

static float silu(float v) { return v / (1.f + expf(-v)); }
static float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.f + tanhf(k0 * (x + k1 * x * x * x)));
}

/* ====================================================================== */
/*  AR models (Thinker / Talker)                                            */
/* ====================================================================== */
enum { OM_THINKER = 0, OM_TALKER = 1, OM_DIT = 2 };

typedef struct {
  int kind, d, L, H, KVH, hd, ff, V, cond_dim, C, S, T;
} om_desc;

typedef struct {
  Mat wqkv, wo, wg, wu, wd;
} ArLayer;
typedef struct {
  Mat wqkv, wo, w1, w2;
} DitLayer;

typedef struct {
  om_desc m;
  uint64_t seed;
  Mat emb, emb2, lm, whid;
  ArLayer* layers;
  Mat w_in, pos_emb, tok_emb, t_emb, w_out, w_mod;
  DitLayer* dlayers;
} om_model;

typedef struct {
  int len, cap;
  float* k; /* [L][cap][KVH*hd] bf16-rounded */
  float* v;
  float* cond; /* talker [64][d] */
} om_seq;

om_model* om_create(const om_desc* desc, uint64_t seed) {
  om_model* mo = (om_model*)calloc(1, sizeof(om_model));
  mo->m = *desc;
  mo->seed = seed;
  const om_desc* m = desc;
  if (m->kind == OM_DIT) {
    const int d = m->d, L = m->L, C = m->C;
    const float s_d = 1.f / sqrtf((float)d);
    mo->w_in = mat_gen(d, C, seed, 1, 1.f / sqrtf((float)C));
    mo->pos_emb = mat_gen(m->S, d, seed, 2, 0.5f);
    mo->tok_emb = mat_gen(m->V, d, seed, 3, 1.0f);
    mo->t_emb = mat_gen(m->T, d, seed, 4, 1.0f);
    mo->w_out = mat_gen(C, d, seed, 5, s_d);
    mo->w_mod = mat_gen(L * 6 * d, d, seed, 6, 0.5f * s_d);
    mo->dlayers = (DitLayer*)calloc(L, sizeof(DitLayer));
    for (int l = 0; l < L; ++l) {
      uint32_t b = 16u * (l + 1);
      mo->dlayers[l].wqkv = mat_gen(3 * d, d, seed, b + 1, s_d);
      mo->dlayers[l].wo = mat_gen(d, d, seed, b + 2, s_d);
      mo->dlayers[l].w1 = mat_gen(m->ff, d, seed, b + 3, s_d);
      mo->dlayers[l].w2 = mat_gen(d, m->ff, seed, b + 4, 1.f / sqrtf((float)m->ff));
    }
    return mo;
  }
  const int d = m->d;
  const float s_d = 1.f / sqrtf((float)d);
  mo->emb = mat_gen(256, d, seed, 1, 1.0f);
  mo->lm = mat_gen(m->V, d, seed, 2, 4.0f * s_d);
  if (m->kind == OM_TALKER) {
    mo->emb2 = mat_gen(m->V + 1, d, seed, 3, 1.0f);
    mo->whid = mat_gen(d, m->cond_dim, seed, 4, 1.f / sqrtf((float)m->cond_dim));
  }
  const int qkv_rows = (m->H + 2 * m->KVH) * m->hd;
  mo->layers = (ArLayer*)calloc(m->L, sizeof(ArLayer));
  for (int l = 0; l < m->L; ++l) {
    uint32_t b = 16u * (l + 1);
    ArLayer* ly = &mo->layers[l];
    ly->wqkv = mat_gen(qkv_rows, d, seed, b + 0, s_d);
    ly->wo = mat_gen(d, m->H * m->hd, seed, b + 1, 1.f / sqrtf((float)(m->H * m->hd)));
    ly->wg = mat_gen(m->ff, d, seed, b + 2, s_d);
    ly->wu = mat_gen(m->ff, d, seed, b + 3, s_d);
    ly->wd = mat_gen(d, m->ff, seed, b + 4, 1.f / sqrtf((float)m->ff));
  }
  return mo;
}

void om_destroy(om_model* mo) {
  if (!mo) return;
  Mat* all[] = {&mo->emb, &mo->emb2, &mo->lm, &mo->whid, &mo->w_in, &mo->pos_emb,
                &mo->tok_emb, &mo->t_emb, &mo->w_out, &mo->w_mod};
  for (size_t i = 0; i < sizeof(all) / sizeof(all[0]); ++i) mat_free(all[i]);
  if (mo->layers)
    for (int l = 0; l < mo->m.L; ++l) {
      mat_free(&mo->layers[l].wqkv);
      mat_free(&mo->layers[l].wo);
      mat_free(&mo->layers[l].wg);
      mat_free(&mo->layers[l].wu);
      mat_free(&mo->layers[l].wd);
    }
  if (mo->dlayers)
    for (int l = 0; l < mo->m.L; ++l) {
      mat_free(&mo->dlayers[l].wqkv);
      mat_free(&mo->dlayers[l].wo);
      mat_free(&mo->dlayers[l].w1);
      mat_free(&mo->dlayers[l].w2);
    }
  free(mo->layers);
  free(mo->dlayers);
  free(mo);
}

/* bf16 bits of one weight element (tests compare device weights). */
uint16_t om_weight_bits(const om_model* mo, const char* name, int64_t row, int64_t col) {
  const Mat* m = NULL;
  if (!strcmp(name, "embed")) m = &mo->emb;
  else if (!strcmp(name, "lm_head")) m = &mo->lm;
  else if (!strcmp(name, "embed_codec")) m = &mo->emb2;
  else if (!strcmp(name, "w_hid")) m = &mo->whid;
  else if (!strcmp(name, "L0.wqkv")) m = mo->layers ? &mo->layers[0].wqkv : &mo->dlayers[0].wqkv;
  else if (!strcmp(name, "w_mod")) m = &mo->w_mod;
  else if (!strcmp(name, "w_in")) m = &mo->w_in;
  if (!m || !m->w) return 0xFFFF;
  return m->w[row * m->cols + col];
}

om_seq* om_seq_new(const om_model* mo, int cap) {
  const om_desc* m = &mo->m;
  om_seq* s = (om_seq*)calloc(1, sizeof(om_seq));
  s->cap = cap;
  size_t n = (size_t)m->L * cap * m->KVH * m->hd;
  s->k = (float*)calloc(n, sizeof(float));
  s->v = (float*)calloc(n, sizeof(float));
  if (m->kind == OM_TALKER) s->cond = (float*)calloc((size_t)64 * m->d, sizeof(float));
  return s;
}
void om_seq_free(om_seq* s) {
  if (!s) return;
  free(s->k);
  free(s->v);
  free(s->cond);
  free(s);
}
int om_seq_len(const om_seq* s) { return s->len; }

/* Fused RMSNorm as the B200 kernels compute it (gemm_tc.cu EPI_RESID_NORM /
 * GemmEpilogue::ss_in): the GEMM consumes bf16(x) un-normalised and its
 * output row is scaled by inv = rsqrt(sum_tiles(sum_{i in tile} x_i^2)/d + eps),
 * tiles of 128 features summed in tile order. */
static float rms_inv_tiled(const float* x, int d) {
  float ss = 0.f;
  for (int t = 0; t < d; t += 128) {
    float p = 0.f;
    for (int i = t; i < t + 128 && i < d; ++i) p += x[i] * x[i];
    ss += p;
  }
  return 1.f / sqrtf(ss / d + 1e-6f);
}

static void rmsnorm_bf16(const float* x, int d, float* y) {
  float ss = 0.f;
  for (int i = 0; i < d; ++i) ss += x[i] * x[i];
  const float inv = 1.f / sqrtf(ss / d + 1e-6f);
  for (int i = 0; i < d; ++i) y[i] = bf16r(x[i] * inv);
}

/*
 * Feeds n tokens at positions [len, len+n) (prefill span, or one decode token).
 *   tokens[i]     : input id, -1 = stage start id (thinker 0, talker V)
 *   cond_rows[i]  : talker conditioning row j
 *   hid_rows      : talker prefill: n x cond_dim bf16 bits of the upstream
 *                   hidden row of each token (NULL for decode)
 *   is_decode     : 1 -> also run the final norm + LM head on the last row
 *   logits_out    : [V] fp32 (decode), hidden_out: [d] bf16 bits (decode)
 * Returns the greedy id (decode) or -1.
 */
int om_ar_feed(const om_model* mo, om_seq* s, int n, const int* tokens, const int* cond_rows,
               const uint16_t* hid_rows, int is_decode, float* logits_out, uint16_t* hidden_out,
               float* margin_out) {
  const om_desc* m = &mo->m;
  const int d = m->d, H = m->H, KVH = m->KVH, hd = m->hd, L = m->L, ff = m->ff;
  const int qkv_w = (H + 2 * KVH) * hd;
  const int talker = m->kind == OM_TALKER;
  const int start_id = talker ? m->V : 0;
  if (s->len + n > s->cap) return -2;
  float* x = (float*)calloc((size_t)n * d, sizeof(float));
  float* xn = (float*)malloc((size_t)n * d * sizeof(float));
  float* qkv = (float*)malloc((size_t)n * qkv_w * sizeof(float));
  float* q = (float*)malloc((size_t)n * H * hd * sizeof(float));
  float* at = (float*)malloc((size_t)n * H * hd * sizeof(float));
  float* tmp = (float*)malloc((size_t)n * (ff > d ? ff : d) * sizeof(float));
  float* g = (float*)malloc((size_t)n * ff * sizeof(float));
  float* u = (float*)malloc((size_t)n * ff * sizeof(float));

  /* embedding */
  if (!talker) {
    for (int i = 0; i < n; ++i) {
      int t = tokens[i] < 0 ? start_id : tokens[i];
      for (int c = 0; c < d; ++c) x[(size_t)i * d + c] = from_bits(mo->emb.w[(size_t)t * d + c]);
    }
  } else if (!is_decode) {
    float* hin = (float*)malloc((size_t)n * m->cond_dim * sizeof(float));
    float* hp = (float*)malloc((size_t)n * d * sizeof(float));
    for (size_t i = 0; i < (size_t)n * m->cond_dim; ++i) hin[i] = from_bits(hid_rows[i]);
    gemm(hin, n, &mo->whid, hp);
    for (int i = 0; i < n; ++i) {
      int t = tokens[i] < 0 ? start_id : tokens[i];
      float* cr = s->cond + (size_t)cond_rows[i] * d;
      for (int c = 0; c < d; ++c) {
        float v = from_bits(mo->emb.w[(size_t)t * d + c]) + hp[(size_t)i * d + c];
        cr[c] = v;
        x[(size_t)i * d + c] = v;
      }
    }
    free(hin);
    free(hp);
  } else {
    for (int i = 0; i < n; ++i) {
      int t = tokens[i] < 0 ? start_id : tokens[i];
      const float* cr = s->cond + (size_t)cond_rows[i] * d;
      for (int c = 0; c < d; ++c)
        x[(size_t)i * d + c] = from_bits(mo->emb2.w[(size_t)t * d + c]) + cr[c];
    }
  }

  const float scale = 1.0f / sqrtf((float)hd);
  const int half = hd / 2, group = H / KVH;
  for (int l = 0; l < L; ++l) {
    const ArLayer* ly = &mo->layers[l];
    for (size_t i = 0; i < (size_t)n * d; ++i) xn[i] = bf16r(x[i]);
    gemm(xn, n, &ly->wqkv, qkv);
    for (int i = 0; i < n; ++i) {
      const int pos = s->len + i;
      float* row = qkv + (size_t)i * qkv_w;
      const float inv = rms_inv_tiled(x + (size_t)i * d, d);
      for (int c = 0; c < qkv_w; ++c) row[c] *= inv;
      for (int h = 0; h < H + 2 * KVH; ++h)
        for (int j = 0; j < half; ++j) {
          float a = row[h * hd + j], b = row[h * hd + j + half], o0 = a, o1 = b;
          if (h < H + KVH) {
            const double inv = pow(10000.0, -(double)j / half);
            const double ang = pos * inv;
            const float cs = (float)cos(ang), sn = (float)sin(ang);
            o0 = a * cs - b * sn;
            o1 = b * cs + a * sn;
          }
          if (h < H) {
            q[(size_t)i * H * hd + h * hd + j] = bf16r(o0);
            q[(size_t)i * H * hd + h * hd + j + half] = bf16r(o1);
          } else {
            const int isv = h >= H + KVH;
            const int kh = isv ? h - H - KVH : h - H;
            float* dst = (isv ? s->v : s->k) + (((size_t)l * s->cap + pos) * KVH + kh) * hd;
            dst[j] = bf16r(o0);
            dst[j + half] = bf16r(o1);
          }
        }
    }
    /* attention, online softmax in key order like the kernel */
#pragma omp parallel for collapse(2) schedule(static)
    for (int i = 0; i < n; ++i)
      for (int h = 0; h < H; ++h) {
        const int qpos = s->len + i, kh = h / group;
        float qv[256];
        for (int c = 0; c < hd; ++c) qv[c] = q[(size_t)i * H * hd + h * hd + c] * scale;
        float mx = -INFINITY, lsum = 0.f, acc[256];
        for (int c = 0; c < hd; ++c) acc[c] = 0.f;
        for (int kp = 0; kp <= qpos; ++kp) {
          const float* kr = s->k + (((size_t)l * s->cap + kp) * KVH + kh) * hd;
          const float* vr = s->v + (((size_t)l * s->cap + kp) * KVH + kh) * hd;
          float dot = 0.f;
          for (int c = 0; c < hd; ++c) dot += qv[c] * kr[c];
          const float mn = fmaxf(mx, dot);
          const float corr = expf(mx - mn), p = expf(dot - mn);
          lsum = lsum * corr + p;
          for (int c = 0; c < hd; ++c) acc[c] = acc[c] * corr + p * vr[c];
          mx = mn;
        }
        const float inv = 1.f / lsum;
        for (int c = 0; c < hd; ++c) at[(size_t)i * H * hd + h * hd + c] = bf16r(acc[c] * inv);
      }
    gemm(at, n, &ly->wo, tmp);
    for (size_t i = 0; i < (size_t)n * d; ++i) x[i] += tmp[i];
    for (size_t i = 0; i < (size_t)n * d; ++i) xn[i] = bf16r(x[i]);
    gemm(xn, n, &ly->wg, g);
    gemm(xn, n, &ly->wu, u);
    for (int i = 0; i < n; ++i) {
      const float inv = rms_inv_tiled(x + (size_t)i * d, d);
      for (int c = 0; c < ff; ++c) {
        const size_t k = (size_t)i * ff + c;
        g[k] = bf16r(silu(g[k] * inv) * (u[k] * inv));
      }
    }
    gemm(g, n, &ly->wd, tmp);
    for (size_t i = 0; i < (size_t)n * d; ++i) x[i] += tmp[i];
  }
  s->len += n;

  int tok = -1;
  if (is_decode) {
    float* h = xn;
    rmsnorm_bf16(x + (size_t)(n - 1) * d, d, h);
    float* lg = (float*)malloc((size_t)m->V * sizeof(float));
    gemm(h, 1, &mo->lm, lg);
    const int lo = talker ? 0 : 1;
    float b1 = -INFINITY, b2 = -INFINITY;
    for (int i = lo; i < m->V; ++i) {
      if (lg[i] > b1) {
        b2 = b1;
        b1 = lg[i];
        tok = i;
      } else if (lg[i] > b2) {
        b2 = lg[i];
      }
    }
    if (logits_out) memcpy(logits_out, lg, (size_t)m->V * sizeof(float));
    if (hidden_out)
      for (int c = 0; c < d; ++c) hidden_out[c] = bf16bits(h[c]);
    if (margin_out) *margin_out = b1 - b2;
    free(lg);
  }
  free(x);
  free(xn);
  free(qkv);
  free(q);
  free(at);
  free(tmp);
  free(g);
  free(u);
  return tok;
}

/* ====================================================================== */
/*  DiT                                                                     */
/* ====================================================================== */
static void layer_norm_mod(const float* h, int d, const float* shift, const float* scl, float* a) {
  float s = 0.f;
  for (int i = 0; i < d; ++i) s += h[i];
  const float mean = s / d;
  float v = 0.f;
  for (int i = 0; i < d; ++i) {
    float t = h[i] - mean;
    v += t * t;
  }
  const float inv = 1.f / sqrtf(v / d + 1e-6f);
  for (int i = 0; i < d; ++i) {
    float y = (h[i] - mean) * inv;
    if (scl) y = y * (1.f + scl[i]) + shift[i];
    a[i] = bf16r(y);
  }
}

/*
 * Denoises n tokens: (rid[i], pos[i], id[i]) -> samples[i*S + s] (int32), and
 * the final fp32 latents if latents != NULL ([n][S][C]).
 */
void om_dit_denoise(const om_model* mo, int n, const uint64_t* rid, const int* pos, const int* ids,
                    int32_t* samples, float* latents) {
  const om_desc* m = &mo->m;
  const int d = m->d, L = m->L, C = m->C, S = m->S, T = m->T, ff = m->ff, H = m->H, hd = m->hd;
  const int ldm = L * 6 * d;
  const uint64_t seed = mo->seed ^ kNoiseSeedSalt;
  float* x = (float*)malloc((size_t)S * C * sizeof(float));
  float* xin = (float*)malloc((size_t)S * C * sizeof(float));
  float* h = (float*)malloc((size_t)S * d * sizeof(float));
  float* a = (float*)malloc((size_t)S * d * sizeof(float));
  float* qkv = (float*)malloc((size_t)S * 3 * d * sizeof(float));
  float* o = (float*)malloc((size_t)S * d * sizeof(float));
  float* tmp = (float*)malloc((size_t)S * (ff > d ? ff : d) * sizeof(float));
  float* uu = (float*)malloc((size_t)S * ff * sizeof(float));
  float* v = (float*)malloc((size_t)S * C * sizeof(float));
  float* cv = (float*)malloc((size_t)d * sizeof(float));
  float* mod = (float*)malloc((size_t)ldm * sizeof(float));
  for (int p = 0; p < n; ++p) {
    for (int s = 0; s < S; ++s)
      for (int ch = 0; ch < C; ++ch)
        x[s * C + ch] = (float)irwin4(noise_hash(seed, rid[p], (uint32_t)pos[p], (uint32_t)s, (uint32_t)ch)) * kNoiseMult;
    for (int t = 0; t < T; ++t) {
      for (int i = 0; i < d; ++i) {
        float e = from_bits(mo->tok_emb.w[(size_t)ids[p] * d + i]) + from_bits(mo->t_emb.w[(size_t)t * d + i]);
        cv[i] = bf16r(silu(e));
      }
      gemm(cv, 1, &mo->w_mod, mod);
      for (int i = 0; i < S * C; ++i) xin[i] = bf16r(x[i]);
      gemm(xin, S, &mo->w_in, h);
      for (int s = 0; s < S; ++s)
        for (int i = 0; i < d; ++i) h[(size_t)s * d + i] += from_bits(mo->pos_emb.w[(size_t)s * d + i]);
      for (int l = 0; l < L; ++l) {
        const DitLayer* ly = &mo->dlayers[l];
        const float* md = mod + (size_t)l * 6 * d;
        for (int s = 0; s < S; ++s) layer_norm_mod(h + (size_t)s * d, d, md, md + d, a + (size_t)s * d);
        gemm(a, S, &ly->wqkv, qkv);
        for (int i = 0; i < S * 3 * d; ++i) qkv[i] = bf16r(qkv[i]);
        const float scale = 1.0f / sqrtf((float)hd);
        for (int hh = 0; hh < H; ++hh) {
          float sp[16][16];
          for (int i = 0; i < S; ++i)
            for (int j = 0; j < S; ++j) {
              float acc = 0.f;
              for (int c = 0; c < hd; ++c)
                acc += qkv[(size_t)i * 3 * d + hh * hd + c] * qkv[(size_t)j * 3 * d + d + hh * hd + c];
              sp[i][j] = acc * scale;
            }
          for (int i = 0; i < S; ++i) {
            float mx = -INFINITY, l2 = 0.f;
            for (int j = 0; j < S; ++j) mx = fmaxf(mx, sp[i][j]);
            for (int j = 0; j < S; ++j) {
              sp[i][j] = expf(sp[i][j] - mx);
              l2 += sp[i][j];
            }
            const float inv = 1.f / l2;
            for (int j = 0; j < S; ++j) sp[i][j] *= inv;
          }
          for (int i = 0; i < S; ++i)
            for (int c = 0; c < hd; ++c) {
              float acc = 0.f;
              for (int j = 0; j < S; ++j) acc += sp[i][j] * qkv[(size_t)j * 3 * d + 2 * d + hh * hd + c];
              o[(size_t)i * d + hh * hd + c] = bf16r(acc);
            }
        }
        gemm(o, S, &ly->wo, tmp);
        for (int s = 0; s < S; ++s)
          for (int i = 0; i < d; ++i) h[(size_t)s * d + i] += md[2 * d + i] * tmp[(size_t)s * d + i];
        for (int s = 0; s < S; ++s)
          layer_norm_mod(h + (size_t)s * d, d, md + 3 * d, md + 4 * d, a + (size_t)s * d);
        gemm(a, S, &ly->w1, uu);
        for (int i = 0; i < S * ff; ++i) uu[i] = bf16r(gelu_tanh(uu[i]));
        gemm(uu, S, &ly->w2, tmp);
        for (int s = 0; s < S; ++s)
          for (int i = 0; i < d; ++i) h[(size_t)s * d + i] += md[5 * d + i] * tmp[(size_t)s * d + i];
      }
      for (int s = 0; s < S; ++s) layer_norm_mod(h + (size_t)s * d, d, NULL, NULL, a + (size_t)s * d);
      gemm(a, S, &mo->w_out, v);
      const float dt = 1.f / T;
      for (int i = 0; i < S * C; ++i) x[i] = x[i] + dt * v[i];
    }
    for (int s = 0; s < S; ++s) {
      float qv = rintf(24.f * x[s * C]);
      qv = fminf(fmaxf(qv, -64.f), 63.f);
      samples[(size_t)p * S + s] = (int32_t)qv;
    }
    if (latents) memcpy(latents + (size_t)p * S * C, x, (size_t)S * C * sizeof(float));
  }
  free(x);
  free(xin);
  free(h);
  free(a);
  free(qkv);
  free(o);
  free(tmp);
  free(uu);
  free(v);
  free(cv);
  free(mod);
}

int om_threads(void) { return omp_get_max_threads(); }
