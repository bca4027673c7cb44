// a1 -- step segmentation (readings R1-R4).
//
// Two launches, integer and latency-bound:
//   seg_count: one CTA per sequence counts step ends in [gen_start, n); the last CTA to
//              finish scans the per-sequence counts into seq_step_off.
//   seg_fill : one CTA per sequence re-walks its tokens in 4096-token tiles, numbers the
//              step ends with a block scan and writes [start, end) and the content count.
#include "common.cuh"

namespace ms {
namespace {

constexpr int kCountThreads = 256;
constexpr int kFillThreads = 512;
constexpr int kFillItems = 8;

struct SegWs {
  int32_t* cnt;        // [num_seqs]
  unsigned int* done;  // 1
};

SegWs seg_layout(Ws& w, int32_t num_seqs) {
  SegWs s;
  s.cnt = w.take<int32_t>((size_t)num_seqs + 1);
  s.done = w.take<unsigned int>(1);
  return s;
}

__device__ __forceinline__ int64_t clamp_gs(int32_t g, int64_t n) {
  return g < 0 ? 0 : (g > n ? n : (int64_t)g);
}

__global__ void __launch_bounds__(kCountThreads) seg_count_kernel(
    const int32_t* __restrict__ tokens, const int64_t* __restrict__ seq_tok_off, const int32_t* __restrict__ gen_start,
    const uint8_t* __restrict__ seq_final, int32_t num_seqs, Delims dl, int64_t* __restrict__ seq_step_off,
    int64_t step_cap, SegWs ws, int32_t* status) {
  __shared__ int64_t sh[kCountThreads / 32 + 1];
  for (int32_t s = blockIdx.x; s < num_seqs; s += gridDim.x) {
    const int64_t off = seq_tok_off[s], n = seq_tok_off[s + 1] - off;
    const int32_t* t = tokens + off;
    const bool fin = seq_final[s] != 0;
    int64_t c = 0;
    for (int64_t i = clamp_gs(gen_start[s], n) + threadIdx.x; i < n; i += kCountThreads) {
      const bool e = (i + 1 < n) ? (is_delim(t[i], dl) && !is_delim(t[i + 1], dl)) : fin;
      c += e ? 1 : 0;
    }
    c = block_sum<kCountThreads>(c, sh);
    if (threadIdx.x == 0) ws.cnt[s] = (int32_t)c;
  }
  if (last_block_done(ws.done)) {
    cta_scan_counts<kCountThreads>(ws.cnt, seq_step_off, num_seqs, sh);
    __syncthreads();
    if (threadIdx.x == 0 && seq_step_off[num_seqs] > step_cap) set_status(status, MEMSHARE_ERR_CAPACITY);
  }
}

__global__ void __launch_bounds__(kFillThreads) seg_fill_kernel(
    const int32_t* __restrict__ tokens, const int64_t* __restrict__ seq_tok_off, const int32_t* __restrict__ gen_start,
    const uint8_t* __restrict__ seq_final, int32_t num_seqs, Delims dl, int32_t* __restrict__ step_start,
    int32_t* __restrict__ step_end, int32_t* __restrict__ step_nbag, const int64_t* __restrict__ seq_step_off,
    int64_t step_cap) {
  __shared__ int64_t sh[kFillThreads / 32 + 1];
  __shared__ int64_t sh_carry;
  constexpr int kTile = kFillThreads * kFillItems;
  for (int32_t s = blockIdx.x; s < num_seqs; s += gridDim.x) {
    const int64_t off = seq_tok_off[s], n = seq_tok_off[s + 1] - off;
    const int32_t* t = tokens + off;
    const bool fin = seq_final[s] != 0;
    const int64_t gbase = seq_step_off[s];
    const int64_t steps_s = seq_step_off[s + 1] - gbase;
    if (steps_s == 0) continue;
    const int64_t gs = clamp_gs(gen_start[s], n);
    if (threadIdx.x == 0 && gbase < step_cap) step_start[gbase] = (int32_t)gs;
    int64_t m_carry = 0, c_carry = 0;
    for (int64_t tile = gs; tile < n; tile += kTile) {
      const int64_t i0 = tile + (int64_t)threadIdx.x * kFillItems;
      uint32_t eflags = 0, cflags = 0;
      bool dnext = (i0 < n) ? is_delim(t[i0], dl) : false;
#pragma unroll
      for (int j = 0; j < kFillItems; ++j) {
        const int64_t i = i0 + j;
        if (i < n) {
          const bool d = dnext;
          dnext = (i + 1 < n) ? is_delim(t[i + 1], dl) : false;
          const bool e = (i + 1 < n) ? (d && !dnext) : fin;
          eflags |= (e ? 1u : 0u) << j;
          cflags |= (d ? 0u : 1u) << j;
        }
      }
      const int64_t packed = ((int64_t)__popc(eflags) << 32) | (int64_t)__popc(cflags);
      int64_t tot;
      const int64_t ex = block_excl_scan<kFillThreads>(packed, tot, sh);
      int64_t m_run = m_carry + (ex >> 32);
      int64_t c_run = c_carry + (ex & 0xffffffffll);
#pragma unroll
      for (int j = 0; j < kFillItems; ++j) {
        const int64_t i = i0 + j;
        c_run += (cflags >> j) & 1u;
        if ((eflags >> j) & 1u) {
          const int64_t g = gbase + m_run;
          if (g < step_cap) {
            step_end[g] = (int32_t)(i + 1);
            step_nbag[g] = (int32_t)c_run;   // cumulative for now
          }
          if (m_run + 1 < steps_s && g + 1 < step_cap) step_start[g + 1] = (int32_t)(i + 1);
          m_run += 1;
        }
      }
      m_carry += tot >> 32;
      c_carry += tot & 0xffffffffll;
    }
    __syncthreads();
    // cumulative content counts -> per-step counts
    int64_t prev = 0;
    for (int64_t mb = 0; mb < steps_s; mb += kFillThreads) {
      const int64_t m = mb + threadIdx.x;
      const int64_t g = gbase + m;
      const bool ok = m < steps_s && g < step_cap;
      const int64_t v = ok ? step_nbag[g] : 0;
      const int64_t pv = (m == mb) ? prev : (ok ? step_nbag[g - 1] : 0);
      const int64_t last_m = (steps_s - mb < kFillThreads ? steps_s - mb : kFillThreads) - 1;
      __syncthreads();
      if (ok) step_nbag[g] = (int32_t)(v - pv);
      if (threadIdx.x == last_m) sh_carry = v;
      __syncthreads();
      prev = sh_carry;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace ms

using namespace ms;

extern "C" size_t memshare_segment_steps_workspace_size(int32_t num_seqs) {
  if (num_seqs < 0) return 0;
  Ws w{nullptr, 0};
  seg_layout(w, num_seqs);
  return w.size();
}

extern "C" memshare_status memshare_segment_steps(const int32_t* tokens, const int64_t* seq_tok_off,
                                                  const int32_t* gen_start, const uint8_t* seq_final,
                                                  int32_t num_seqs, const int32_t* delim_ids_host, int32_t num_delims,
                                                  int32_t* step_start, int32_t* step_end, int32_t* step_nbag,
                                                  int64_t* seq_step_off, int64_t step_cap, void* workspace,
                                                  size_t workspace_bytes, int32_t* device_status, void* stream) {
  if (num_seqs < 0 || step_cap < 0 || num_delims < 1 || num_delims > MEMSHARE_MAX_DELIMS) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (!seq_tok_off || !seq_step_off || !delim_ids_host || !workspace || !device_status) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (num_seqs > 0 && (!tokens || !gen_start || !seq_final)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (step_cap > 0 && (!step_start || !step_end || !step_nbag)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < memshare_segment_steps_workspace_size(num_seqs)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  Delims dl{};
  dl.n = num_delims;
  for (int i = 0; i < num_delims; ++i) dl.id[i] = delim_ids_host[i];
  Ws w{static_cast<char*>(workspace), 0};
  SegWs ws = seg_layout(w, num_seqs);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(ws.done, 0, sizeof(unsigned int), st) != cudaSuccess) return MEMSHARE_ERR_CUDA;
  const int grid = num_seqs < 1 ? 1 : (num_seqs < 4 * sm_count() ? num_seqs : 4 * sm_count());
  seg_count_kernel<<<grid, kCountThreads, 0, st>>>(tokens, seq_tok_off, gen_start, seq_final, num_seqs, dl,
                                                   seq_step_off, step_cap, ws, device_status);
  if (num_seqs > 0)
    seg_fill_kernel<<<grid, kFillThreads, 0, st>>>(tokens, seq_tok_off, gen_start, seq_final, num_seqs, dl, step_start,
                                                   step_end, step_nbag, seq_step_off, step_cap);
  return launch_status();
}
