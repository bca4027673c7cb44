// f3 / f4 -- analysis calls built on the path.
//   memshare_similarity_ratio : PAPER.md:121-126 (Fig. 2) -- per sequence, the number of finished
//                               steps with at least one Stage-1 survivor at the caller's tau_s
//                               ("whose cosine similarity with any previous step exceeds a
//                               specified threshold"), counted from memshare_step_candidates'
//                               matches (rank 0 exists iff the best cosine exceeds tau_s).
//   memshare_all_pairs        : PAPER.md:142-145 (Observation 2, block-wise distance heatmaps;
//                               SPEC.md:271-279) -- every block pair (i < j) of a per-sequence
//                               logical-block range as a target-grouped pair list, to be scored by
//                               memshare_block_distance (the distance matrix is symmetric).
#include "common.cuh"

namespace ms {
namespace {

constexpr int kNT = 256;

__global__ void ratio_kernel(const memshare_step_match* __restrict__ m, const int64_t* __restrict__ num_matches,
                             int64_t match_cap, int32_t num_seqs, int64_t* __restrict__ redundant, int32_t* status) {
  int64_t M = __ldcg(num_matches);
  M = M < 0 ? 0 : (M < match_cap ? M : match_cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
    const memshare_step_match x = m[i];
    if (x.rank != 0) continue;
    if (x.seq < 0 || x.seq >= num_seqs) { set_status(status, MEMSHARE_ERR_CORRUPTION); continue; }
    atomicAdd(reinterpret_cast<unsigned long long*>(redundant + x.seq), 1ull);
  }
}

struct AllPairsWs {
  int32_t* tcnt;        // [num_seqs] targets per sequence
  int32_t* pcnt;        // [num_seqs] pairs per sequence
  int64_t* toff;        // [num_seqs + 1]
  int64_t* poff;        // [num_seqs + 1]
  unsigned int* done;
};

AllPairsWs ap_layout(Ws& w, int32_t num_seqs) {
  AllPairsWs a;
  a.tcnt = w.take<int32_t>((size_t)num_seqs + 1);
  a.pcnt = w.take<int32_t>((size_t)num_seqs + 1);
  a.toff = w.take<int64_t>((size_t)num_seqs + 2);
  a.poff = w.take<int64_t>((size_t)num_seqs + 2);
  a.done = w.take<unsigned int>(1);
  return a;
}

__device__ __forceinline__ void range_of(const int32_t* blk_begin, const int32_t* blk_end, const int64_t* seq_tok_off,
                                         int32_t s, int32_t d, int32_t& lo, int32_t& hi) {
  const int32_t full = (int32_t)((seq_tok_off[s + 1] - seq_tok_off[s]) / d);   // full blocks only
  lo = blk_begin[s] < 0 ? 0 : blk_begin[s];
  hi = blk_end[s] > full ? full : blk_end[s];
  if (hi < lo) hi = lo;
}

__global__ void __launch_bounds__(kNT) ap_count_kernel(const int64_t* seq_tok_off, int32_t num_seqs,
                                                       const int32_t* blk_begin, const int32_t* blk_end, int32_t d,
                                                       AllPairsWs ws, int64_t* num_pairs, int64_t* num_targets,
                                                       int64_t* target_off, int64_t pair_cap, int64_t target_cap,
                                                       int32_t* status) {
  __shared__ int64_t sh[kNT / 32 + 1];
  for (int32_t s = blockIdx.x * kNT + threadIdx.x; s < num_seqs; s += gridDim.x * kNT) {
    int32_t lo, hi;
    range_of(blk_begin, blk_end, seq_tok_off, s, d, lo, hi);
    const int64_t m = hi - lo;
    ws.tcnt[s] = m > 1 ? (int32_t)(m - 1) : 0;
    ws.pcnt[s] = (int32_t)(m * (m - 1) / 2);
  }
  if (last_block_done(ws.done)) {
    cta_scan_counts<kNT>(ws.tcnt, ws.toff, num_seqs, sh);
    cta_scan_counts<kNT>(ws.pcnt, ws.poff, num_seqs, sh);
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t T = ws.toff[num_seqs], P = ws.poff[num_seqs];
      *num_targets = T;
      *num_pairs = P;
      if (T > target_cap || P > pair_cap) set_status(status, MEMSHARE_ERR_CAPACITY);
      if (T <= target_cap) target_off[T] = P;
    }
  }
}

__global__ void __launch_bounds__(kNT) ap_fill_kernel(const int64_t* seq_tok_off, int32_t num_seqs,
                                                      const int32_t* blk_begin, const int32_t* blk_end, int32_t d,
                                                      const int32_t* table, int32_t table_stride, int32_t num_blocks,
                                                      AllPairsWs ws, memshare_block_pair* pairs, int64_t* target_off,
                                                      int64_t pair_cap, int64_t target_cap, int32_t* status) {
  // one warp per target
  const int lane = threadIdx.x & 31;
  const int64_t T = __ldcg(ws.toff + num_seqs);
  for (int64_t t = (blockIdx.x * (int64_t)kNT + threadIdx.x) >> 5; t < T; t += ((int64_t)gridDim.x * kNT) >> 5) {
    int32_t lo_s = 0, hi_s = num_seqs - 1;              // sequence of target t
    while (lo_s < hi_s) {
      const int32_t mid = (lo_s + hi_s + 1) >> 1;
      if (__ldcg(ws.toff + mid) <= t) lo_s = mid; else hi_s = mid - 1;
    }
    const int32_t s = lo_s;
    int32_t lo, hi;
    range_of(blk_begin, blk_end, seq_tok_off, s, d, lo, hi);
    const int32_t j = lo + 1 + (int32_t)(t - __ldcg(ws.toff + s));     // target logical block
    // pairs of targets lo+1 .. j-1 precede: sum_{q=1}^{j-lo-1} q
    const int64_t r = j - lo;
    const int64_t base = __ldcg(ws.poff + s) + (r - 1) * r / 2;
    const int32_t* trow = table + (int64_t)s * table_stride;
    const int32_t tp = trow[j];
    if (tp < 0 || tp >= num_blocks) set_status(status, MEMSHARE_ERR_CORRUPTION);
    if (lane == 0 && t < target_cap) target_off[t] = base;
    for (int32_t i = lo + lane; i < j; i += 32) {
      const int64_t pos = base + (i - lo);
      const int32_t sp = trow[i];
      if (sp < 0 || sp >= num_blocks) set_status(status, MEMSHARE_ERR_CORRUPTION);
      if (pos < pair_cap) {
        memshare_block_pair pr;
        pr.seq = s; pr.target_idx = (int32_t)t; pr.target_logical = j; pr.source_logical = i;
        pr.target_phys = tp; pr.source_phys = sp;
        pairs[pos] = pr;
      }
    }
  }
}

}  // namespace
}  // namespace ms

using namespace ms;

extern "C" memshare_status memshare_similarity_ratio(const memshare_step_match* matches, const int64_t* num_matches,
                                                     int64_t match_cap, int32_t num_seqs, int64_t* redundant_steps,
                                                     int32_t* device_status, void* stream) {
  MS_NVTX("memshare_similarity_ratio");
  if (!num_matches || !redundant_steps || !device_status || num_seqs < 0 || match_cap < 0 ||
      (match_cap > 0 && !matches))
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (num_seqs == 0) return MEMSHARE_OK;
  if (cudaMemsetAsync(redundant_steps, 0, sizeof(int64_t) * (size_t)num_seqs, st) != cudaSuccess)
    return MEMSHARE_ERR_CUDA;
  const int64_t mc = match_cap < 1 ? 1 : match_cap;
  const int grid = (int)((mc + kNT - 1) / kNT < 4 * sm_count() ? (mc + kNT - 1) / kNT : 4 * sm_count());
  ratio_kernel<<<grid, kNT, 0, st>>>(matches, num_matches, match_cap, num_seqs, redundant_steps, device_status);
  return launch_status();
}

extern "C" size_t memshare_all_pairs_workspace_size(int32_t num_seqs) {
  if (num_seqs < 0) return 0;
  Ws w{nullptr, 0};
  ap_layout(w, num_seqs);
  return w.size();
}

extern "C" memshare_status memshare_all_pairs(const int64_t* seq_tok_off, int32_t num_seqs, const int32_t* blk_begin,
                                              const int32_t* blk_end, const int32_t* block_table, int32_t table_stride,
                                              int32_t num_blocks, int32_t block_size, memshare_block_pair* pairs,
                                              int64_t pair_cap, int64_t* num_pairs, int64_t* target_off,
                                              int64_t target_cap, int64_t* num_targets, void* workspace,
                                              size_t workspace_bytes, int32_t* device_status, void* stream) {
  MS_NVTX("memshare_all_pairs");
  if (!seq_tok_off || !num_pairs || !target_off || !num_targets || !workspace || !device_status || num_seqs < 0 ||
      block_size < 1 || table_stride < 0 || num_blocks < 0 || pair_cap < 0 || target_cap < 0)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (num_seqs > 0 && (!blk_begin || !blk_end || !block_table)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (pair_cap > 0 && !pairs) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < memshare_all_pairs_workspace_size(num_seqs)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  Ws w{static_cast<char*>(workspace), 0};
  AllPairsWs ws = ap_layout(w, num_seqs);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(ws.done, 0, sizeof(unsigned int), st) != cudaSuccess) return MEMSHARE_ERR_CUDA;
  const int grid = num_seqs < 1 ? 1 : (int)((num_seqs + kNT - 1) / kNT < 4 * sm_count() ? (num_seqs + kNT - 1) / kNT
                                                                                          : 4 * sm_count());
  ap_count_kernel<<<grid, kNT, 0, st>>>(seq_tok_off, num_seqs, blk_begin, blk_end, block_size, ws, num_pairs,
                                        num_targets, target_off, pair_cap, target_cap, device_status);
  if (num_seqs > 0)
    ap_fill_kernel<<<4 * sm_count(), kNT, 0, st>>>(seq_tok_off, num_seqs, blk_begin, blk_end, block_size, block_table,
                                                  table_stride, num_blocks, ws, pairs, target_off, pair_cap, target_cap,
                                                  device_status);
  return launch_status();
}
