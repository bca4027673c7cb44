/* Host twin of the counter-hash KV generator (see msgen_hash.h). Input generation
 * only -- no MemShare arithmetic. Build: gcc -O2 -fopenmp -ffp-contract=off -shared. */
#include <string.h>
#include "msgen_hash.h"

static float msgen_scale(void) {
  union { uint32_t u; float f; } c;
  c.u = MSGEN_SCALE_BITS;
  return c.f;
}

/* one element from its two row keys; compile with -ffp-contract=off (no FMA) */
static uint16_t msgen_value(uint64_t brow, uint64_t nrow, int32_t x, float eta) {
  const float sc = msgen_scale();
  const float b = (float)msgen_ih(brow, x) * sc;
  const float n = (float)msgen_ih(nrow, x) * sc;
  const float t = eta * n;
  union { float f; uint32_t u; } r;
  r.f = b + t;
  return msgen_bf16_rne(r.u);
}

/* For i < nb: fill block (blk_seq[i], blk_logical[i]) into physical block blk_dst[i]
 * of the pool K/V (bf16 bits, element strides; slice [d][h_local][d_h] contiguous).
 * Token slots past the sequence end are zero. head_offset = global index of local head 0. */
void msgen_fill_blocks_host(uint16_t* k, uint16_t* v, int64_t layer_stride, int64_t block_stride,
                            int32_t num_layers, int32_t h_local, int32_t head_offset, int32_t head_dim,
                            int32_t block_size, const int32_t* tokens, const int64_t* seq_tok_off,
                            const int32_t* blk_seq, const int32_t* blk_logical, const int32_t* blk_dst,
                            int64_t nb, uint64_t seed, float eta) {
  const int64_t slice = (int64_t)block_size * h_local * head_dim;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < nb; ++i) {
    const int32_t s = blk_seq[i];
    const int64_t n = seq_tok_off[s + 1] - seq_tok_off[s];
    for (int32_t l = 0; l < num_layers; ++l) {
      for (int32_t kv = 0; kv < 2; ++kv) {
        uint16_t* dst = (kv ? v : k) + (int64_t)l * layer_stride + (int64_t)blk_dst[i] * block_stride;
        memset(dst, 0, (size_t)slice * 2);
        for (int32_t tau = 0; tau < block_size; ++tau) {
          const int64_t pos = (int64_t)blk_logical[i] * block_size + tau;
          if (pos >= n) break;
          const int32_t tok = tokens[seq_tok_off[s] + pos];
          for (int32_t hh = 0; hh < h_local; ++hh) {
            const uint64_t brow = msgen_base_row(seed, tok, l, head_offset + hh, kv);
            const uint64_t nrow = msgen_noise_row(seed, s, pos, l, head_offset + hh, kv);
            uint16_t* o = dst + ((int64_t)tau * h_local + hh) * head_dim;
            for (int32_t x = 0; x < head_dim; ++x) o[x] = msgen_value(brow, nrow, x, eta);
          }
        }
      }
    }
  }
}
