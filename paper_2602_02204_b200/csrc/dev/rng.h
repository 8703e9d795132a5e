// Counter-based weight / noise generator shared (by construction, not by
// linkage) with the CPU oracle (oracle/models_cpu.c): every value is a pure
// function of (seed, tensor id, index) computed with integer arithmetic and a
// single fp32 multiply, so host and device produce identical bits without any
// weight files.  Irwin-Hall(4) approximates N(0, 1).
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define OMNI_HD __host__ __device__ __forceinline__
#else
#define OMNI_HD inline
#endif

namespace omni_dev {

OMNI_HD uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Sum of four 16-bit uniforms, centred: integer in [-131070, 131070].
OMNI_HD int32_t irwin4(uint64_t h) {
  return static_cast<int32_t>(h & 0xFFFF) + static_cast<int32_t>((h >> 16) & 0xFFFF) +
         static_cast<int32_t>((h >> 32) & 0xFFFF) + static_cast<int32_t>((h >> 48) & 0xFFFF) -
         131070;
}

OMNI_HD uint64_t weight_hash(uint64_t seed, uint32_t tensor_id, uint64_t idx) {
  return mix64(seed ^ mix64((static_cast<uint64_t>(tensor_id) << 40) ^ idx));
}

// Multiplier turning irwin4() into N(0, scale^2); computed in double, rounded once.
inline float weight_mult(float scale) {
  return static_cast<float>(static_cast<double>(scale) * 1.7320508075688772 / 65536.0);
}

// DiT initial noise key: (request, global token position, sample, channel).
OMNI_HD uint64_t noise_hash(uint64_t seed, uint64_t rid, uint32_t pos, uint32_t s, uint32_t ch) {
  return mix64(seed ^ mix64(rid * 0x100000001B3ull ^ mix64((static_cast<uint64_t>(pos) << 24) ^
                                                           (static_cast<uint64_t>(s) << 12) ^ ch)));
}

// Top-k sampler draw: (stage sampling seed, request key, emitted index).
OMNI_HD uint64_t sample_hash(uint64_t seed, uint32_t key, uint32_t index) {
  return mix64(seed ^ mix64((static_cast<uint64_t>(key) << 32) ^ index ^ 0x73616d706c650000ull));
}

}  // namespace omni_dev
