// a1 -- step segmentation (readings R1-R4).
//
// Tile-parallel over the FLAT token array (sequences are concatenated, so the global order of
// step ends is the global step order and a device-wide scan numbers them directly):
//   seg_count : one CTA per 4096-token tile counts step ends and in-generation content tokens;
//               the last CTA scans the tile counts into tile offsets (and writes the
//               seq_step_off entries of trailing empty sequences and the total).
//   seg_fill  : each tile re-derives its flags, block-scans them and writes, per step end,
//               step_end and the inclusive content prefix; the thread holding a sequence's
//               first token writes seq_step_off[s] and the content count before s.
//   seg_final : one thread per step: step_start = previous end in the sequence (or gen_start),
//               content count = prefix difference.
// A token i of sequence s (local position q, length n) ends a step iff q >= gen_start and
//   (q + 1 < n) ? (t[i] in D && t[i+1] not in D) : final[s]          (reading R3).
#include <climits>

#include "common.cuh"

namespace ms {
namespace {

constexpr int kNT = 1024;
constexpr int kItems = 4;
constexpr int kTile = kNT * kItems;

struct SegWs {
  int64_t* tile_cnt;    // [tiles] packed (ends << 32 | content)
  int64_t* tile_off;    // [tiles + 1] exclusive, packed
  int32_t* step_seq;    // [step_cap]
  int64_t* cum;         // [step_cap] inclusive content prefix at each step end
  int64_t* seq_cbase;   // [num_seqs + 1] content tokens before sequence s
  unsigned int* done;
};

SegWs seg_layout(Ws& w, int64_t num_tokens, int32_t num_seqs, int64_t step_cap) {
  const int64_t tiles = (num_tokens + kTile - 1) / kTile;
  SegWs s;
  s.tile_cnt = w.take<int64_t>(tiles + 1);
  s.tile_off = w.take<int64_t>(tiles + 2);
  s.step_seq = w.take<int32_t>(step_cap + 1);
  s.cum = w.take<int64_t>(step_cap + 1);
  s.seq_cbase = w.take<int64_t>((size_t)num_seqs + 1);
  s.done = w.take<unsigned int>(1);
  return s;
}

struct SegArgs {
  const int32_t* tokens;
  const int64_t* seq_tok_off;
  const int32_t* gen_start;
  const uint8_t* seq_final;
  int32_t num_seqs;
  int64_t num_tokens;
  Delims dl;
  int32_t* step_start;
  int32_t* step_end;
  int32_t* step_nbag;
  int64_t* seq_step_off;
  int64_t step_cap;
  int32_t* status;
  SegWs ws;
};

// last s with seq_tok_off[s] <= i (sequences of length 0 are skipped by taking the last)
__device__ __forceinline__ int32_t seq_of_token(const SegArgs& a, int64_t i) {
  int32_t lo = 0, hi = a.num_seqs - 1;
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (__ldg(a.seq_tok_off + mid) <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

struct TokFlags {
  uint32_t end, content;
  int32_t seq0;            // sequence of the thread's first token
};

// flags of the kItems tokens starting at global position i0
__device__ __forceinline__ TokFlags token_flags(const SegArgs& a, int64_t i0) {
  TokFlags f{0u, 0u, 0};
  if (i0 >= a.num_tokens) return f;
  int32_t s = seq_of_token(a, i0);
  f.seq0 = s;
  int64_t off = __ldg(a.seq_tok_off + s), nxt = __ldg(a.seq_tok_off + s + 1);
  int64_t gs = off + (int64_t)max(0, __ldg(a.gen_start + s));
  bool fin = __ldg(a.seq_final + s) != 0;
  bool dcur = is_delim(a.tokens[i0], a.dl);
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int64_t i = i0 + j;
    if (i >= a.num_tokens) break;
    while (i >= nxt) {                        // crossed into the next (non-empty) sequence
      ++s;
      off = nxt;
      nxt = __ldg(a.seq_tok_off + s + 1);
      gs = off + (int64_t)max(0, __ldg(a.gen_start + s));
      fin = __ldg(a.seq_final + s) != 0;
    }
    const bool dnext = (i + 1 < nxt) ? is_delim(a.tokens[i + 1], a.dl) : false;
    if (i >= gs) {
      const bool e = (i + 1 < nxt) ? (dcur && !dnext) : fin;
      f.end |= (e ? 1u : 0u) << j;
      f.content |= (dcur ? 0u : 1u) << j;
    }
    dcur = (i + 1 < a.num_tokens) ? ((i + 1 < nxt) ? dnext : is_delim(a.tokens[i + 1], a.dl)) : false;
  }
  return f;
}

__global__ void __launch_bounds__(kNT) seg_count_kernel(SegArgs a) {
  __shared__ int64_t sh[kNT / 32 + 1];
  const int64_t tiles = (a.num_tokens + kTile - 1) / kTile;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const TokFlags f = token_flags(a, tile * kTile + (int64_t)threadIdx.x * kItems);
    const int64_t packed = ((int64_t)__popc(f.end) << 32) | (int64_t)__popc(f.content);
    const int64_t tot = block_sum<kNT>(packed, sh);
    if (threadIdx.x == 0) a.ws.tile_cnt[tile] = tot;
  }
  if (last_block_done(a.ws.done)) {
    int64_t carry = 0;
    for (int64_t base = 0; base < tiles; base += kNT) {
      const int64_t i = base + threadIdx.x;
      const int64_t v = i < tiles ? __ldcg(a.ws.tile_cnt + i) : 0;
      int64_t tot;
      const int64_t ex = block_excl_scan<kNT>(v, tot, sh);
      if (i < tiles) a.ws.tile_off[i] = carry + ex;
      carry += tot;
    }
    if (threadIdx.x == 0) {
      a.ws.tile_off[tiles] = carry;
      const int64_t total = carry >> 32;
      if (total > a.step_cap) set_status(a.status, MEMSHARE_ERR_CAPACITY);
    }
    // sequences that start at the end of the token array (trailing empties) and the total
    for (int32_t s = threadIdx.x; s <= a.num_seqs; s += kNT) {
      if (__ldg(a.seq_tok_off + s) >= a.num_tokens) {
        a.seq_step_off[s] = carry >> 32;
        a.ws.seq_cbase[s] = carry & 0xffffffffll;
      }
    }
  }
}

__global__ void __launch_bounds__(kNT) seg_fill_kernel(SegArgs a) {
  __shared__ int64_t sh[kNT / 32 + 1];
  const int64_t tiles = (a.num_tokens + kTile - 1) / kTile;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t i0 = tile * kTile + (int64_t)threadIdx.x * kItems;
    const TokFlags f = token_flags(a, i0);
    const int64_t packed = ((int64_t)__popc(f.end) << 32) | (int64_t)__popc(f.content);
    int64_t tot;
    const int64_t ex = block_excl_scan<kNT>(packed, tot, sh) + __ldcg(a.ws.tile_off + tile);
    int64_t m = ex >> 32, c = ex & 0xffffffffll;
    int32_t s = f.seq0;
    for (int j = 0; j < kItems; ++j) {
      const int64_t i = i0 + j;
      if (i >= a.num_tokens) break;
      while (i >= __ldg(a.seq_tok_off + s + 1)) ++s;
      const int64_t off = __ldg(a.seq_tok_off + s);
      if (i == off) {
        // first token of s (and of the empty sequences just before it sharing this offset)
        int32_t s0 = s;
        while (s0 > 0 && __ldg(a.seq_tok_off + s0 - 1) == off) --s0;
        for (int32_t q = s0; q <= s; ++q) {
          a.seq_step_off[q] = m;
          a.ws.seq_cbase[q] = c;
        }
      }
      c += (f.content >> j) & 1u;
      if ((f.end >> j) & 1u) {
        if (m < a.step_cap) {
          a.step_end[m] = (int32_t)(i - off + 1);
          a.ws.step_seq[m] = s;
          a.ws.cum[m] = c;
        }
        ++m;
      }
    }
  }
}

__global__ void seg_final_kernel(SegArgs a) {
  int64_t G = __ldcg(a.seq_step_off + a.num_seqs);
  G = G < a.step_cap ? G : a.step_cap;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = a.ws.step_seq[g];
    const bool first = g == a.seq_step_off[s];
    const int64_t n = a.seq_tok_off[s + 1] - a.seq_tok_off[s];
    const int32_t gsv = a.gen_start[s];
    const int64_t gs = gsv < 0 ? 0 : (gsv > n ? n : gsv);
    a.step_start[g] = first ? (int32_t)gs : a.step_end[g - 1];
    a.step_nbag[g] = (int32_t)(a.ws.cum[g] - (first ? a.ws.seq_cbase[s] : a.ws.cum[g - 1]));
  }
}

}  // namespace
}  // namespace ms

using namespace ms;

extern "C" size_t memshare_segment_steps_workspace_size(int64_t num_tokens, int32_t num_seqs, int64_t step_cap) {
  if (num_tokens < 0 || num_seqs < 0 || step_cap < 0) return 0;
  Ws w{nullptr, 0};
  seg_layout(w, num_tokens, num_seqs, step_cap);
  return w.size();
}

extern "C" memshare_status memshare_segment_steps(const int32_t* tokens, int64_t num_tokens, const int64_t* seq_tok_off,
                                                  const int32_t* gen_start, const uint8_t* seq_final,
                                                  int32_t num_seqs, const int32_t* delim_ids_host, int32_t num_delims,
                                                  int32_t* step_start, int32_t* step_end, int32_t* step_nbag,
                                                  int64_t* seq_step_off, int64_t step_cap, void* workspace,
                                                  size_t workspace_bytes, int32_t* device_status, void* stream) {
  if (num_tokens < 0 || num_tokens > (int64_t)INT32_MAX || num_seqs < 0 || step_cap < 0 || num_delims < 1 ||
      num_delims > MEMSHARE_MAX_DELIMS)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (!seq_tok_off || !seq_step_off || !delim_ids_host || !workspace || !device_status) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (num_seqs > 0 && (!gen_start || !seq_final)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (num_tokens > 0 && (!tokens || num_seqs == 0)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (step_cap > 0 && (!step_start || !step_end || !step_nbag)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < memshare_segment_steps_workspace_size(num_tokens, num_seqs, step_cap))
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  SegArgs a{};
  a.tokens = tokens; a.seq_tok_off = seq_tok_off; a.gen_start = gen_start; a.seq_final = seq_final;
  a.num_seqs = num_seqs; a.num_tokens = num_tokens;
  a.dl.n = num_delims;
  for (int i = 0; i < num_delims; ++i) a.dl.id[i] = delim_ids_host[i];
  a.step_start = step_start; a.step_end = step_end; a.step_nbag = step_nbag; a.seq_step_off = seq_step_off;
  a.step_cap = step_cap; a.status = device_status;
  Ws w{static_cast<char*>(workspace), 0};
  a.ws = seg_layout(w, num_tokens, num_seqs, step_cap);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(a.ws.done, 0, sizeof(unsigned int), st) != cudaSuccess) return MEMSHARE_ERR_CUDA;
  const int64_t tiles = (num_tokens + kTile - 1) / kTile;
  const int grid = (int)(tiles < 1 ? 1 : (tiles < 4 * sm_count() ? tiles : 4 * sm_count()));
  seg_count_kernel<<<grid, kNT, 0, st>>>(a);
  seg_fill_kernel<<<grid, kNT, 0, st>>>(a);
  const int64_t sc = step_cap < 1 ? 1 : step_cap;
  const int fgrid = (int)((sc + 255) / 256 < 4 * sm_count() ? (sc + 255) / 256 : 4 * sm_count());
  seg_final_kernel<<<fgrid, 256, 0, st>>>(a);
  return launch_status();
}
