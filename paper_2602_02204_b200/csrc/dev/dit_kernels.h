// DiT (K6) kernel launchers and constants. Internal to libomni_dev.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace omni_dev {

constexpr int kDitSamples = 16;       // S: samples per codec token (reference_pipeline.hpp:218-223)
constexpr float kSampleScale = 24.f;  // latent channel 0 -> int32 sample, clamped to [-64, 63]
// irwin4() -> N(0,1): sqrt(3) / 65536, rounded once to fp32
constexpr float kNoiseMult = 2.6429027e-05f;
constexpr uint64_t kNoiseSeedSalt = 0x6e6f697365ull;  // "noise"

struct DitTokDesc {  // one conditioning token of the batch
  uint64_t rid;      // request id (noise key)
  int32_t pos;       // global token position in the request's stream (noise key)
  int32_t id;        // conditioning id (codec / text token)
};

cudaError_t dit_noise(const DitTokDesc* toks, int n_tok, int S, int C, uint64_t seed, float* x,
                      __nv_bfloat16* xb, cudaStream_t st, int* zero = nullptr, int n_zero = 0);
cudaError_t dit_cond(const DitTokDesc* toks, int n_tok, const __nv_bfloat16* tok_emb,
                     const __nv_bfloat16* t_emb, int step, int d, __nv_bfloat16* cvec, cudaStream_t st);
// mod_base: adaLN table rows of this Euler step ([vocab][ld_mod]); the row of
// token p is mod_base + toks[p].id * ld_mod. nullptr -> plain LayerNorm.
cudaError_t dit_ln_mod(const float* h, int rows, int d, const float* mod_base, const DitTokDesc* toks,
                       int ld_mod, int shift_off, int scale_off, int S, __nv_bfloat16* a, cudaStream_t st);
cudaError_t dit_attn(const __nv_bfloat16* qkv, int n_tok, int d, int n_heads, __nv_bfloat16* out,
                     cudaStream_t st);

}  // namespace omni_dev
