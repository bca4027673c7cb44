/* Counter-hash KV value generator -- the generator's OWN header, included only by
 * its two twins (msgen_host.c, msgen_dev.cu). Holds no MemShare arithmetic.
 *
 * value(seq, pos, token, layer, head, kv, x) =
 *     bf16_rne( base(token, layer, head, kv, x) + eta * noise(seq, pos, layer, head, kv, x) )
 *
 * base, noise ~ approx N(0,1): Irwin-Hall sum of four 16-bit uniforms taken from one
 * splitmix64 output, centred and scaled by sqrt(3)/65536 (SURVEY.md §8(d) "KV values").
 * Every step is integer arithmetic or a single IEEE round-to-nearest fp32 operation
 * (int->float of a value < 2^24 is exact; one multiply; one multiply + one add, no
 * contraction), so the host and CUDA twins agree bit for bit.
 */
#ifndef MSGEN_HASH_H
#define MSGEN_HASH_H
#include <stdint.h>

#if defined(__CUDACC__)
#define MSGEN_FN static __host__ __device__ __forceinline__
#else
#define MSGEN_FN static inline
#endif

#define MSGEN_GOLDEN 0x9E3779B97F4A7C15ULL
#define MSGEN_SEED_BASE 0xB45EB45EB45EB45EULL
#define MSGEN_SEED_NOISE 0x0015E0015E0015E0ULL
/* fp32 nearest to sqrt(3)/65536 */
#define MSGEN_SCALE_BITS 0x37DDB3D7u

MSGEN_FN uint64_t msgen_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* per-(token, layer, head, kv) row key of the base term */
MSGEN_FN uint64_t msgen_base_row(uint64_t seed, int32_t token, int32_t layer, int32_t head, int32_t kv) {
  uint64_t k = msgen_mix64(seed ^ MSGEN_SEED_BASE);
  k = msgen_mix64(k ^ (uint64_t)(uint32_t)token);
  return msgen_mix64(k + (((uint64_t)(uint32_t)layer << 20) | ((uint64_t)(uint32_t)head << 1) | (uint64_t)kv));
}

/* per-(seq, pos, layer, head, kv) row key of the noise term */
MSGEN_FN uint64_t msgen_noise_row(uint64_t seed, int32_t seq, int64_t pos, int32_t layer, int32_t head, int32_t kv) {
  uint64_t k = msgen_mix64(seed ^ MSGEN_SEED_NOISE);
  k = msgen_mix64(k ^ (uint64_t)(uint32_t)seq);
  k = msgen_mix64(k + (uint64_t)pos);
  return msgen_mix64(k + (((uint64_t)(uint32_t)layer << 20) | ((uint64_t)(uint32_t)head << 1) | (uint64_t)kv));
}

/* centred Irwin-Hall integer in [-131070, 131070]: exact in fp32 */
MSGEN_FN int32_t msgen_ih(uint64_t row, int32_t x) {
  uint64_t h = msgen_mix64(row + (uint64_t)(uint32_t)x * MSGEN_GOLDEN);
  int32_t s = (int32_t)(h & 0xFFFFu) + (int32_t)((h >> 16) & 0xFFFFu) +
              (int32_t)((h >> 32) & 0xFFFFu) + (int32_t)((h >> 48) & 0xFFFFu);
  return s - 131070;
}

/* fp32 -> bf16 bits, round to nearest even (finite inputs only) */
MSGEN_FN uint16_t msgen_bf16_rne(uint32_t u) {
  uint32_t bias = 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)((u + bias) >> 16);
}

#endif
