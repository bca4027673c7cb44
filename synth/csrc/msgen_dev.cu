// CUDA twin of the counter-hash KV generator (see msgen_hash.h). Input generation only --
// no MemShare arithmetic. Bit-identical to msgen_host.c: integer hash, then
// __int2float_rn / __fmul_rn / __fadd_rn (no contraction), then integer bf16 RNE.
#include <cstdint>
#include <cuda_runtime.h>
#include "msgen_hash.h"

namespace {

__device__ __forceinline__ uint16_t msgen_value_dev(uint64_t brow, uint64_t nrow, int32_t x, float eta) {
  const float sc = __uint_as_float(MSGEN_SCALE_BITS);
  const float b = __fmul_rn(__int2float_rn(msgen_ih(brow, x)), sc);
  const float n = __fmul_rn(__int2float_rn(msgen_ih(nrow, x)), sc);
  const float v = __fadd_rn(b, __fmul_rn(eta, n));
  return msgen_bf16_rne(__float_as_uint(v));
}

__global__ void msgen_fill_blocks_kernel(uint16_t* __restrict__ k, uint16_t* __restrict__ v,
                                         int64_t layer_stride, int64_t block_stride, int32_t num_layers,
                                         int32_t h_local, int32_t head_offset, int32_t head_dim,
                                         int32_t block_size, const int32_t* __restrict__ tokens,
                                         const int64_t* __restrict__ seq_tok_off,
                                         const int32_t* __restrict__ blk_seq,
                                         const int32_t* __restrict__ blk_logical,
                                         const int32_t* __restrict__ blk_dst, uint64_t seed, float eta) {
  const int64_t i = blockIdx.x;
  const int32_t l = blockIdx.y >> 1, kv = blockIdx.y & 1;
  const int32_t s = blk_seq[i];
  const int64_t n = seq_tok_off[s + 1] - seq_tok_off[s];
  uint16_t* dst = (kv ? v : k) + (int64_t)l * layer_stride + (int64_t)blk_dst[i] * block_stride;
  const int32_t chunks = block_size * h_local * head_dim / 8;
  for (int32_t c = threadIdx.x; c < chunks; c += blockDim.x) {
    const int32_t e = c * 8;
    const int32_t tau = e / (h_local * head_dim);
    const int32_t hh = (e / head_dim) % h_local;
    const int32_t x0 = e % head_dim;
    const int64_t pos = (int64_t)blk_logical[i] * block_size + tau;
    uint16_t out[8];
    if (pos < n) {
      const int32_t tok = tokens[seq_tok_off[s] + pos];
      const uint64_t brow = msgen_base_row(seed, tok, l, head_offset + hh, kv);
      const uint64_t nrow = msgen_noise_row(seed, s, pos, l, head_offset + hh, kv);
#pragma unroll
      for (int j = 0; j < 8; ++j) out[j] = msgen_value_dev(brow, nrow, x0 + j, eta);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) out[j] = 0;
    }
    uint4 pk;
    pk.x = (uint32_t)out[0] | ((uint32_t)out[1] << 16);
    pk.y = (uint32_t)out[2] | ((uint32_t)out[3] << 16);
    pk.z = (uint32_t)out[4] | ((uint32_t)out[5] << 16);
    pk.w = (uint32_t)out[6] | ((uint32_t)out[7] << 16);
    *reinterpret_cast<uint4*>(dst + e) = pk;
  }
}

}  // namespace

// Same contract as msgen_fill_blocks_host, device pointers, enqueued on `stream`.
// Returns 0 on success, else the cudaError_t of the launch.
extern "C" int msgen_fill_blocks_dev(uint16_t* k, uint16_t* v, int64_t layer_stride, int64_t block_stride,
                                     int32_t num_layers, int32_t h_local, int32_t head_offset,
                                     int32_t head_dim, int32_t block_size, const int32_t* tokens,
                                     const int64_t* seq_tok_off, const int32_t* blk_seq,
                                     const int32_t* blk_logical, const int32_t* blk_dst, int64_t nb,
                                     uint64_t seed, float eta, void* stream) {
  if (nb <= 0) return 0;
  if (head_dim % 8 != 0) return (int)cudaErrorInvalidValue;
  for (int64_t first = 0; first < nb; first += 65535 * 16) {
    const int64_t cnt = (nb - first < 65535 * 16) ? nb - first : 65535 * 16;
    dim3 grid((unsigned)cnt, (unsigned)(num_layers * 2));
    msgen_fill_blocks_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        k, v, layer_stride, block_stride, num_layers, h_local, head_offset, head_dim, block_size, tokens,
        seq_tok_off, blk_seq + first, blk_logical + first, blk_dst + first, seed, eta);
  }
  return (int)cudaGetLastError();
}
