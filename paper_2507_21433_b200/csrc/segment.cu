// a1 -- step segmentation (readings R1-R4).
//
// ONE single-pass kernel over the FLAT token array (sequences are concatenated, so the global
// order of step ends is the global step order). Each CTA owns a kTile-token tile (1024 threads x 4
// tokens; larger per-thread runs were measured slower: their loads do not coalesce) and computes,
// per thread of kItems tokens, an aggregate (ends, content, last boundary): a "boundary" is the
// position where the next step starts -- a sequence's generation start, or the token after a
// step end -- together with the content-token prefix at that point. Aggregates combine with an
// associative operator (counts add; the later boundary wins), so a block scan gives each
// thread its prefix within the tile and a decoupled look-back over the preceding tiles' published
// aggregates / inclusive prefixes gives the tile's prefix. Every step end then knows its global
// step number (ends before it), its start (the last boundary) and its bag size (content since
// that boundary) without a second pass.
// A token i of sequence s (local position q, length n) ends a step iff q >= gen_start and
//   (q + 1 < n) ? (t[i] in D && t[i+1] not in D) : final[s]          (reading R3).
#include <climits>

#include "segment_impl.cuh"

namespace ms {
namespace {

#ifndef MS_SEG_NT
#define MS_SEG_NT 1024
#endif
#ifndef MS_SEG_ITEMS
#define MS_SEG_ITEMS 2
#endif
constexpr int kNT = MS_SEG_NT;           // threads per tile
constexpr int kItems = MS_SEG_ITEMS;     // tokens per thread (a 32-bit flag word each)
static_assert(kItems <= 32, "per-thread flags are 32-bit masks");
constexpr int kTile = kNT * kItems;

struct SegWs {
  int32_t* flag;   // [tiles] 0 = nothing, 1 = aggregate, 2 = inclusive prefix; [tiles] = tile ticket (zeroed per call)
  int4* agg;       // [tiles]
  int4* inc;       // [tiles]
};

SegWs seg_layout(Ws& w, int64_t num_tokens) {
  const int64_t tiles = (num_tokens + kTile - 1) / kTile;
  SegWs s;
  s.flag = w.take<int32_t>(tiles + 1);
  s.agg = w.take<int4>(tiles + 1);
  s.inc = w.take<int4>(tiles + 1);
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

// the sequence context of a flat position (advanced monotonically)
struct SeqCur {
  int32_t s;
  int64_t off, nxt, gs;
  bool fin;
};

__device__ __forceinline__ void seq_load(const SegArgs& a, SeqCur& q, int32_t s) {
  q.s = s;
  q.off = __ldg(a.seq_tok_off + s);
  q.nxt = __ldg(a.seq_tok_off + s + 1);
  const int64_t n = q.nxt - q.off;
  const int32_t g = __ldg(a.gen_start + s);
  q.gs = q.off + (g < 0 ? 0 : (g > n ? n : (int64_t)g));
  q.fin = __ldg(a.seq_final + s) != 0;
}

__device__ __forceinline__ void seq_advance(const SegArgs& a, SeqCur& q, int64_t i) {
  while (i >= q.nxt) seq_load(a, q, q.s + 1);   // crossed into the next (non-empty) sequence
}

struct Bits {
  uint32_t end, content, gstart;
};

// flags of the kItems tokens starting at i0 (i0 < num_tokens)
__device__ __forceinline__ Bits token_bits(const SegArgs& a, int64_t i0, SeqCur& q) {
  Bits b{0u, 0u, 0u};
  int32_t tk[kItems + 1];
#pragma unroll
  for (int j = 0; j <= kItems; ++j) tk[j] = (i0 + j < a.num_tokens) ? __ldg(a.tokens + i0 + j) : INT_MIN;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int64_t i = i0 + j;
    if (i >= a.num_tokens) break;
    seq_advance(a, q, i);
    if (i >= q.gs) {
      const bool dcur = is_delim(tk[j], a.dl);
      const bool e = (i + 1 < q.nxt) ? (dcur && !is_delim(tk[j + 1], a.dl)) : q.fin;
      b.end |= (e ? 1u : 0u) << j;
      b.content |= (dcur ? 0u : 1u) << j;
      b.gstart |= (i == q.gs ? 1u : 0u) << j;
    }
  }
  return b;
}

__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ Agg ld_agg(const int4* p) {
  const int4 v = __ldcg(p);
  return Agg{v.x, v.y, v.z, v.w};
}

__global__ void __launch_bounds__(kNT, 1) seg_kernel(SegArgs a) {
  pdl_trigger();
  TL_SCOPE(1);
  __shared__ Agg s_warp[kNT / 32];
  __shared__ Agg s_tile_prefix;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t tiles = (a.num_tokens + kTile - 1) / kTile;
  if (tiles == 0) {                                      // no tokens: every sequence has 0 steps
    for (int32_t s = threadIdx.x; s <= a.num_seqs; s += kNT) a.seq_step_off[s] = 0;
    return;
  }
  // the tile comes from an atomic ticket (flag[tiles], zeroed with the flags), not blockIdx: a
  // tile's look-back waits only on tiles already claimed by running CTAs, so the scan completes
  // however many CTAs are co-resident
  __shared__ int32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(a.ws.flag + tiles, 1);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t i0 = tile * kTile + (int64_t)threadIdx.x * kItems;
  const bool live = i0 < a.num_tokens;
  SeqCur q{};
  Bits b{0u, 0u, 0u};
  if (live) {
    seq_load(a, q, seq_of_token(a, i0));
    b = token_bits(a, i0, q);
  }
  // thread aggregate
  Agg mine = agg_identity();
  mine.e = __popc(b.end);
  mine.c = __popc(b.content);
  {
    int32_t c = 0;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      if ((b.gstart >> j) & 1u) { mine.bpos = (int32_t)(i0 + j); mine.bcb = c; }
      c += (b.content >> j) & 1u;
      if ((b.end >> j) & 1u) { mine.bpos = (int32_t)(i0 + j + 1); mine.bcb = c; }
    }
  }
  // block-wide exclusive scan of the thread aggregates
  Agg x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Agg y = shfl_agg_up(x, o);
    if (lane >= o) x = combine(y, x);
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    Agg v = lane < kNT / 32 ? s_warp[lane] : agg_identity();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const Agg y = shfl_agg_up(v, o);
      if (lane >= o) v = combine(y, v);
    }
    if (lane < kNT / 32) s_warp[lane] = v;               // inclusive warp totals
  }
  __syncthreads();
  Agg excl = shfl_agg_up(x, 1);
  if (lane == 0) excl = agg_identity();
  if (w > 0) excl = combine(s_warp[w - 1], excl);
  const Agg tile_agg = s_warp[kNT / 32 - 1];
  // decoupled look-back for the tile prefix
  if (w == 0) {
    if (tile == 0) {
      if (lane == 0) {
        a.ws.inc[0] = make_int4(tile_agg.e, tile_agg.c, tile_agg.bpos, tile_agg.bcb);
        __threadfence();
        st_release(a.ws.flag, 2);
        s_tile_prefix = agg_identity();
      }
    } else {
      if (lane == 0) {
        a.ws.agg[tile] = make_int4(tile_agg.e, tile_agg.c, tile_agg.bpos, tile_agg.bcb);
        __threadfence();
        st_release(a.ws.flag + tile, 1);
      }
      Agg run = agg_identity();                          // combination of tiles (p, tile)
      int64_t p = tile - 1;
      for (;;) {
        const int64_t qi = p - lane;
        int32_t f = 2;
        if (qi >= 0) {
          SpinGuard sg;
          while ((f = ld_acquire(a.ws.flag + qi)) == 0) {
            if (sg.expired()) {                          // never published: report, do not hang
              set_status(a.status, MEMSHARE_ERR_CORRUPTION);
              f = 2;
              break;
            }
          }
        }
        const unsigned inc_mask = __ballot_sync(0xffffffffu, f == 2);
        const int stop = inc_mask ? __ffs(inc_mask) - 1 : 32;   // lowest lane (latest tile) with a prefix
        Agg v = agg_identity();
        if (lane < stop && qi >= 0) v = ld_agg(a.ws.agg + qi);
        else if (lane == stop && qi >= 0) v = ld_agg(a.ws.inc + qi);
        // ordered reduction: higher lane = earlier tile
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const Agg y = shfl_agg_down(v, o);
          if (lane + o < 32) v = combine(y, v);
        }
        v.e = __shfl_sync(0xffffffffu, v.e, 0);
        v.c = __shfl_sync(0xffffffffu, v.c, 0);
        v.bpos = __shfl_sync(0xffffffffu, v.bpos, 0);
        v.bcb = __shfl_sync(0xffffffffu, v.bcb, 0);
        run = combine(v, run);
        if (stop < 32) break;
        p -= 32;
      }
      if (lane == 0) {
        const Agg incl = combine(run, tile_agg);
        a.ws.inc[tile] = make_int4(incl.e, incl.c, incl.bpos, incl.bcb);
        __threadfence();
        st_release(a.ws.flag + tile, 2);
        s_tile_prefix = run;
      }
    }
  }
  __syncthreads();
  const Agg tp = s_tile_prefix;
  if (live) {
    const Agg pre = combine(tp, excl);                   // everything before this thread's tokens
    int64_t m = pre.e;
    int32_t c = pre.c;
    int64_t bpos = pre.bpos;
    int32_t bcb = pre.bcb;
    seq_load(a, q, seq_of_token(a, i0));
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int64_t i = i0 + j;
      if (i >= a.num_tokens) break;
      seq_advance(a, q, i);
      if (i == q.off) {
        // first token of s (and of the empty sequences just before it sharing this offset)
        int32_t s0 = q.s;
        while (s0 > 0 && __ldg(a.seq_tok_off + s0 - 1) == q.off) --s0;
        for (int32_t r = s0; r <= q.s; ++r) a.seq_step_off[r] = m;
      }
      if ((b.gstart >> j) & 1u) { bpos = i; bcb = c; }
      c += (b.content >> j) & 1u;
      if ((b.end >> j) & 1u) {
        if (m < a.step_cap) {
          a.step_end[m] = (int32_t)(i - q.off + 1);
          a.step_start[m] = (int32_t)(bpos - q.off);
          a.step_nbag[m] = c - bcb;
        }
        ++m;
        bpos = i + 1;
        bcb = c;
      }
    }
  }
  if (tile == tiles - 1) {
    const int64_t total = (int64_t)tp.e + tile_agg.e;
    if (threadIdx.x == 0 && total > a.step_cap) set_status(a.status, MEMSHARE_ERR_CAPACITY);
    // sequences that start at the end of the token array (trailing empties) and the total
    for (int32_t s = threadIdx.x; s <= a.num_seqs; s += kNT)
      if (__ldg(a.seq_tok_off + s) >= a.num_tokens) a.seq_step_off[s] = total;
  }
}

// zeroes the look-back flags (a kernel, not a memset node: keeps the launch chain programmatic)
__global__ void flag_reset_kernel(int32_t* flag, int64_t n) {
  pdl_trigger();
  TL_SCOPE(0);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) flag[i] = 0;
}

}  // namespace
}  // namespace ms

using namespace ms;

TL_EXPORT(segment)


extern "C" size_t memshare_segment_steps_workspace_size(int64_t num_tokens, int32_t num_seqs, int64_t step_cap) {
  if (num_tokens < 0 || num_seqs < 0 || step_cap < 0) return 0;
  Ws w{nullptr, 0};
  seg_layout(w, num_tokens);
  return w.size();
}

extern "C" memshare_status memshare_segment_steps(const int32_t* tokens, int64_t num_tokens, const int64_t* seq_tok_off,
                                                  const int32_t* gen_start, const uint8_t* seq_final,
                                                  int32_t num_seqs, const int32_t* delim_ids_host, int32_t num_delims,
                                                  int32_t* step_start, int32_t* step_end, int32_t* step_nbag,
                                                  int64_t* seq_step_off, int64_t step_cap, void* workspace,
                                                  size_t workspace_bytes, int32_t* device_status, void* stream) {
  MS_NVTX("memshare_segment_steps");
  if (num_tokens < 0 || num_tokens > (int64_t)INT32_MAX - kTile || num_seqs < 0 || step_cap < 0 || num_delims < 1 ||
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
  a.ws = seg_layout(w, num_tokens);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t tiles = (num_tokens + kTile - 1) / kTile;
  // the look-back flags are zeroed by a small kernel, not a memset node: it keeps the launch chain
  // programmatic (seg_kernel's CTAs wait for it to complete before they publish)
  if (tiles > 0) launch_pdl(flag_reset_kernel, dim3(1), dim3(256), 0, st, a.ws.flag, tiles + 1);   // + the ticket
  launch_pdl(seg_kernel, dim3((unsigned)(tiles < 1 ? 1 : tiles)), dim3(kNT), 0, st, a);
  return launch_status();
}
