// a2-a4 -- bag-of-words encoding, Stage-1 cosine filter and candidate block pairs.
// PAPER.md:224-234 (Alg. 1 Stage 1), :254 (bag of words), :318 ('exceeding' -> strict >),
// :267 / :319-320 (corresponding / pairwise blocks); readings R5-R14, R25.
//
// Design (B200): the bag of words of step k is never densified. The dot product with an
// earlier step j is  <c_k, c_j> = sum over content tokens p of j of c_k[t_p],  so only the
// CURRENT step needs a count table: an open-addressing hash table in shared memory (global
// workspace for steps > 2048 content tokens). Because steps tile the sequence, the whole
// history of k is one contiguous token range; the CTA stages it in shared memory with coalesced
// loads, each thread walks a contiguous run, probes k's table and adds its partial dot once per
// history step it touches (32-bit smem atomics with carry; step boundaries staged in smem).
// Integer dot and norms are exact; the cosine is one IEEE expression (__ddiv_rn / __dsqrt_rn / __dmul_rn), bit-identical to the C oracle.
//
// Launches:
//   encode  : n2 = sum count^2 per step (history norms) -- one CTA per step for a single CoT,
//             one warp per step for large batches
//   stage1  : per current step: table, streamed history dots, strict threshold, (cos desc, j asc)
//             sort (by rank for <= 256 survivors, else bitonic), top-K, count targets/pairs.
//             Shapes: one 1024-thread CTA per step (single CoT); 512-thread CTAs two per SM (large
//             batches); a thread-block cluster of up to 8 CTAs per step sharing its history scan
//             over DSMEM (online LAST rounds).
//             Offline single-CoT launches and online rounds FUSE the fill: each work item
//             (step / sequence) gets its output offsets by summing the published counts of all
//             preceding items (one warp, one memory latency) and writes its matches and pairs.
//             The 512-thread batch shape stashes the survivors and its last CTA scans the counts.
//   fill    : (when not fused) one CTA per current step: write matches, targets, target_off, pairs
#include <cfloat>
#include <climits>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"

namespace ms {
namespace {

constexpr int kNT = 256;          // encode / fill
constexpr int kNW = kNT / 32;
constexpr int kSmemSlots = 8192;       // smem hash table (steps with <= 2048 content tokens, load <= 0.25)
constexpr int kCandCap = 1024;         // survivors held per current step
constexpr int kChunk = kCandCap / 2;   // history steps per selection chunk
constexpr int kMaxTgt = 4096;          // full blocks per step handled by the fill kernel
constexpr int kHistTok = 16384;        // history tokens staged in smem per pass (64 KiB)
constexpr int32_t kEmpty = -1;

struct CandWs {
  unsigned int* done;
  unsigned long long* stash_alloc;
  unsigned long long* ticket;   // stage1 work-item ticket (zeroed by encode)
  int32_t* step_seq;     // [step_cap]
  int64_t* n2;           // [step_cap]
  int32_t* cnt_m;        // [step_cap]
  int32_t* cnt_t;
  int32_t* cnt_p;
  int64_t* stash_base;   // [step_cap]
  int64_t* off_m;        // [step_cap+1]
  int64_t* off_t;
  int64_t* off_p;
  double* stash_cos;     // [match_cap]
  int32_t* stash_j;
  int2* gtab;            // [4*num_tokens] {key, count} global tables of oversize steps
  int4* lb_agg;          // [step_cap] fused fill: {matches+1, targets+1, pairs+1, 1} of the step, 0 = not yet
                         // published (zeroed by encode)
  int64_t* cur_off;      // [num_seqs+1] RANGE work items: exclusive prefix of the current-step counts (encode)
};

CandWs cand_layout(Ws& w, int64_t num_tokens, int64_t step_cap, int64_t match_cap, int32_t num_seqs) {
  CandWs c;
  c.done = w.take<unsigned int>(1);
  c.stash_alloc = w.take<unsigned long long>(1);
  c.ticket = w.take<unsigned long long>(1);
  c.step_seq = w.take<int32_t>(step_cap + 1);
  c.n2 = w.take<int64_t>(step_cap + 1);
  c.cnt_m = w.take<int32_t>(step_cap + 1);
  c.cnt_t = w.take<int32_t>(step_cap + 1);
  c.cnt_p = w.take<int32_t>(step_cap + 1);
  c.stash_base = w.take<int64_t>(step_cap + 1);
  c.off_m = w.take<int64_t>(step_cap + 1);
  c.off_t = w.take<int64_t>(step_cap + 1);
  c.off_p = w.take<int64_t>(step_cap + 1);
  c.stash_cos = w.take<double>(match_cap + 1);
  c.stash_j = w.take<int32_t>(match_cap + 1);
  c.gtab = w.take<int2>(4 * num_tokens + 1);
  c.lb_agg = w.take<int4>(step_cap + 1);
  c.cur_off = w.take<int64_t>((size_t)(num_seqs > 0 ? num_seqs : 0) + 1);
  return c;
}

struct CandArgs {
  const int32_t* tokens;
  const int64_t* seq_tok_off;
  int32_t num_seqs;
  const int64_t* seq_step_off;
  const int32_t* step_start;
  const int32_t* step_end;
  const int32_t* step_nbag;
  int64_t step_cap;
  Delims dl;
  int32_t cur_mode;
  const int32_t* cur_begin;
  const int32_t* cur_end;
  const int32_t* table;
  int32_t table_stride;
  int32_t num_blocks;
  int32_t block_size;
  double tau_s;
  int32_t top_k;
  int32_t pairing;
  memshare_step_match* matches;
  int64_t match_cap;
  int64_t* num_matches;
  memshare_block_pair* pairs;
  int64_t pair_cap;
  int64_t* num_pairs;
  int64_t* target_off;
  int64_t target_cap;
  int64_t* num_targets;
  int32_t* status;
  int32_t fused;        // offline single-CoT launch: stage1 writes matches / pairs itself (no fill kernel)
  int32_t range_items;  // RANGE with the fused fill: work items are the current steps only (a dense list)
  int32_t dbg_skip;     // tuning only (env MEMSHARE_DEBUG_SKIP): bit3 phase stamps; in -DMEMSHARE_TUNING builds also
                        // bit0 skip history stream, bit1 pair count, bit2 last-CTA scan, bit4 table probes
  CandWs ws;
};

__device__ __forceinline__ int64_t total_steps(const CandArgs& a) {
  const int64_t g = __ldcg(a.seq_step_off + a.num_seqs);
  return g < a.step_cap ? g : a.step_cap;
}

// multiplicative hash, top bits (the well-mixed ones); `shift` = 32 - log2(capacity)
__device__ __forceinline__ uint32_t hash_slot(int32_t tok, uint32_t shift) {
  return ((uint32_t)tok * 0x9E3779B1u) >> shift;
}

__device__ __forceinline__ uint32_t pow2_ceil(uint32_t x) { return x <= 1 ? 1u : 1u << (32 - __clz(x - 1)); }
__device__ __forceinline__ uint32_t pow2_floor(uint32_t x) { return 1u << (31 - __clz(x)); }

// Count table of one step, {key, count} pairs with open addressing: in smem (steps with <= 2048
// content tokens, load factor <= 0.25) or in the step's private region of the global workspace
// (4 slots per token of the step, load factor <= 0.5).
struct Table {
  int2* slots;
  uint32_t mask;
  uint32_t shift;
  bool global;
};

// Presence filter of a step's tokens for the history stream: 2^16 bits indexed by the top 16 bits
// of the same multiplicative hash; a clear bit is a definite miss, so the stream skips the table
// probe (and its divergent probe loop) for the history tokens the step does not contain.
constexpr int kBmWords = 2048;
static_assert(kBmWords == 2 * kCandCap, "the filter overlays jasc + flo");
__device__ __forceinline__ uint32_t bm_bit(int32_t tok) { return ((uint32_t)tok * 0x9E3779B1u) >> 16; }

// `own_global`: whether this CTA fills a GLOBAL table. The ranks of a Stage-1 cluster all work on
// the same step; a global table (a step of > smem_slots/4 content tokens) lives in the step's one
// workspace region, so only rank 0 clears and fills it and the caller makes the other ranks wait
// on a cluster barrier before they probe it. Every rank builds its own presence filter.
__device__ Table build_table(const CandArgs& a, int2* s_tab, const int32_t* t, int64_t tok_base, int32_t start,
                             int32_t end, int32_t nbag, int32_t smem_slots = kSmemSlots, uint32_t* bm = nullptr,
                             bool own_global = true) {
  Table tb;
  uint32_t cap;
  if (nbag <= smem_slots / 4) {
    cap = pow2_ceil(4u * (uint32_t)(nbag > 32 ? nbag : 32));
    tb.slots = s_tab;
    tb.global = false;
  } else {
    cap = pow2_floor(4u * (uint32_t)(end - start));
    tb.slots = a.ws.gtab + 4 * (tok_base + start);
    tb.global = true;
  }
  tb.mask = cap - 1;
  tb.shift = 32u - (31u - __clz(cap));
  const bool fill = !tb.global || own_global;
  if (fill)
    for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x) tb.slots[i] = make_int2(kEmpty, 0);
  if (bm != nullptr)
    for (int i = threadIdx.x; i < kBmWords; i += blockDim.x) bm[i] = 0u;
  __syncthreads();
  for (int32_t p = start + threadIdx.x; p < end; p += blockDim.x) {
    const int32_t tok = t[p];
    if (is_delim(tok, a.dl)) continue;
    if (bm != nullptr) {
      const uint32_t hb = bm_bit(tok);
      atomicOr(bm + (hb >> 5), 1u << (hb & 31));
    }
    if (!fill) continue;
    uint32_t slot = hash_slot(tok, tb.shift);
    for (uint32_t probe = 0; probe <= tb.mask; ++probe) {
      int* key = &tb.slots[slot].x;
      const int32_t prev = atomicCAS(key, kEmpty, tok);
      if (prev == kEmpty || prev == tok) {
        atomicAdd(&tb.slots[slot].y, 1);
        break;
      }
      slot = (slot + 1) & tb.mask;
    }
  }
  __syncthreads();
  return tb;
}

__device__ __forceinline__ int32_t seq_of_step(const CandArgs& a, int64_t g) {
  int32_t lo = 0, hi = a.num_seqs - 1;   // last s with seq_step_off[s] <= g
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (__ldg(a.seq_step_off + mid) <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// RANGE: the current local steps [b, e) of sequence s, clamped to its steps below the capacity
__device__ __forceinline__ void cur_range(const CandArgs& a, int32_t s, int64_t G, int64_t& b, int64_t& e) {
  const int64_t g0 = a.seq_step_off[s];
  int64_t g1 = a.seq_step_off[s + 1];
  if (g1 > G) g1 = G;
  const int64_t S = g1 > g0 ? g1 - g0 : 0;
  b = a.cur_begin[s];
  e = a.cur_end[s];
  b = b < 0 ? 0 : (b > S ? S : b);
  e = e < b ? b : (e > S ? S : e);
}

// RANGE work items (range_items): one block of the encode kernel writes cur_off, the exclusive
// prefix over the sequences of their current-step counts (all NT threads of that block)
template <int NT>
__device__ void range_item_offsets(const CandArgs& a, int64_t G, int64_t* sh) {
  int64_t carry = 0;
  for (int64_t base = 0; base < a.num_seqs; base += NT) {
    const int64_t s = base + threadIdx.x;
    int64_t n = 0;
    if (s < a.num_seqs) {
      int64_t b, e;
      cur_range(a, (int32_t)s, G, b, e);
      n = e - b;
    }
    int64_t tot;
    const int64_t ex = block_excl_scan<NT>(n, tot, sh);
    if (s < a.num_seqs) a.ws.cur_off[s] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) a.ws.cur_off[a.num_seqs] = carry;
}

// RANGE work item i -> its step g (global)
__device__ __forceinline__ int64_t range_item_step(const CandArgs& a, int64_t i, int64_t G, int32_t& s_out) {
  int32_t lo = 0, hi = a.num_seqs - 1;                  // last s with cur_off[s] <= i
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (__ldcg(a.ws.cur_off + mid) <= i) lo = mid; else hi = mid - 1;
  }
  int64_t b, e;
  cur_range(a, lo, G, b, e);
  s_out = lo;
  return a.seq_step_off[lo] + b + (i - __ldcg(a.ws.cur_off + lo));
}

// publication keys of the fused fill: steps (offline) or sequences (online LAST rounds)
__device__ __forceinline__ int64_t fill_keys(const CandArgs& a, int64_t G) {
  const int64_t z = a.cur_mode == MEMSHARE_CUR_LAST ? (int64_t)a.num_seqs : G;
  return z < a.step_cap + 1 ? z : a.step_cap + 1;
}

// One CTA per step (latency-optimal when the steps fit in one wave: a single CoT).
__global__ void __launch_bounds__(kNT) encode_kernel(CandArgs a) {
  pdl_trigger();
  TL_SCOPE(2);
  extern __shared__ int2 s_tab[];                         // [kSmemSlots]
  __shared__ int64_t sh[kNW + 1];
  const int64_t G = total_steps(a);
  const int64_t Z = fill_keys(a, G);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < Z; g += (int64_t)gridDim.x * blockDim.x)
    a.ws.lb_agg[g] = make_int4(0, 0, 0, 0);               // stage1's published counts (fused fill)
  if (blockIdx.x == 0 && threadIdx.x == 0) {            // stage1's done counter + stash allocator
    *a.ws.done = 0u;
    *a.ws.stash_alloc = 0ull;
    *a.ws.ticket = 0ull;
  }
  if (a.range_items && blockIdx.x == gridDim.x - 1) range_item_offsets<kNT>(a, G, sh);
  for (int64_t g = blockIdx.x; g < G; g += gridDim.x) {
    const int32_t s = seq_of_step(a, g);
    const int64_t tok_base = a.seq_tok_off[s];
    const int32_t nbag = a.step_nbag[g];
    int64_t n2 = 0;
    if (nbag > 0) {
      const Table tb = build_table(a, s_tab, a.tokens + tok_base, tok_base, a.step_start[g], a.step_end[g], nbag);
      for (uint32_t i = threadIdx.x; i <= tb.mask; i += kNT) {
        const int64_t c = tb.global ? __ldcg(tb.slots + i).y : tb.slots[i].y;
        n2 += c * c;
      }
    }
    n2 = block_sum<kNT>(n2, sh);
    if (threadIdx.x == 0) {
      a.ws.n2[g] = n2;
      a.ws.step_seq[g] = s;
    }
    __syncthreads();
  }
}

// One WARP per step (8 steps per CTA in flight): the step's {key, count} table lives in the
// warp's 1024-slot slice of shared memory (steps of <= 256 content tokens: load <= 0.25) or in the
// step's private region of the global workspace; n2 = sum of count^2 (int64, exact).
constexpr int kEncSlots = kSmemSlots / kNW;                // 1024 slots per warp

template <int kSlotsW = kEncSlots>
__device__ int64_t warp_step_n2(const CandArgs& a, int2* s_tab, const int32_t* t, int64_t tok_base, int32_t start,
                                int32_t end, int32_t nbag) {
  const int lane = threadIdx.x & 31;
  int2* slots;
  uint32_t cap;
  bool global;
  if (nbag <= kSlotsW / 2) {                          // load factor <= 0.5 (<= 0.25 when the slots allow)
    cap = pow2_ceil(4u * (uint32_t)(nbag > 32 ? nbag : 32));
    if (cap > (uint32_t)kSlotsW) cap = (uint32_t)kSlotsW;
    slots = s_tab;
    global = false;
  } else {
    cap = pow2_floor(4u * (uint32_t)(end - start));
    slots = a.ws.gtab + 4 * (tok_base + start);
    global = true;
  }
  const uint32_t mask = cap - 1, shift = 32u - (31u - __clz(cap));
  for (uint32_t i = lane; i < cap; i += 32) slots[i] = make_int2(kEmpty, 0);
  if (global) __threadfence_block();
  __syncwarp();
  for (int32_t p = start + lane; p < end; p += 32) {
    const int32_t tok = t[p];
    if (is_delim(tok, a.dl)) continue;
    uint32_t slot = hash_slot(tok, shift);
    for (uint32_t probe = 0; probe <= mask; ++probe) {
      const int32_t prev = atomicCAS(&slots[slot].x, kEmpty, tok);
      if (prev == kEmpty || prev == tok) {
        atomicAdd(&slots[slot].y, 1);
        break;
      }
      slot = (slot + 1) & mask;
    }
  }
  if (global) __threadfence_block();
  __syncwarp();
  int64_t n2 = 0;
  for (uint32_t i = lane; i < cap; i += 32) {
    const int64_t c = global ? __ldcg(slots + i).y : slots[i].y;
    n2 += c * c;
  }
  return warp_sum(n2);
}

__global__ void __launch_bounds__(kNT) encode_warp_kernel(CandArgs a) {
  pdl_trigger();
  TL_SCOPE(2);
  extern __shared__ int2 s_tab[];                         // [kSmemSlots] = kNW warps x kEncSlots
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t G = total_steps(a);
  const int64_t Z = fill_keys(a, G);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < Z; g += (int64_t)gridDim.x * blockDim.x)
    a.ws.lb_agg[g] = make_int4(0, 0, 0, 0);               // stage1's published counts (fused fill)
  if (blockIdx.x == 0 && threadIdx.x == 0) {            // stage1's done counter + stash allocator
    *a.ws.done = 0u;
    *a.ws.stash_alloc = 0ull;
    *a.ws.ticket = 0ull;
  }
  if (a.range_items && blockIdx.x == gridDim.x - 1) {
    __shared__ int64_t sh[kNW + 1];
    range_item_offsets<kNT>(a, G, sh);
  }
  for (int64_t g = (int64_t)blockIdx.x * kNW + w; g < G; g += (int64_t)gridDim.x * kNW) {
    const int32_t s = seq_of_step(a, g);
    const int64_t tok_base = a.seq_tok_off[s];
    const int32_t nbag = a.step_nbag[g];
    const int64_t n2 = nbag > 0 ? warp_step_n2(a, s_tab + w * kEncSlots, a.tokens + tok_base, tok_base,
                                               a.step_start[g], a.step_end[g], nbag)
                                : 0;
    if (lane == 0) {
      a.ws.n2[g] = n2;
      a.ws.step_seq[g] = s;
    }
    __syncwarp();
  }
}

// --------------------------------------------------------------------------------------------
// candidate list helpers
__device__ __forceinline__ bool cand_before(double ca, int32_t ja, double cb, int32_t jb) {
  return ca > cb || (ca == cb && ja < jb);
}

// Short lists (n <= kRankSort and <= blockDim) are sorted by rank: each thread ranks its own entry
// against all n (broadcast shared-memory reads) and scatters it -- two barriers, where the bitonic
// network costs one barrier per stage (log2(n)(log2(n)+1)/2 stages). Keys are distinct (j is unique
// among a step's candidates), so the ranks are a permutation.
constexpr int kRankSort = 256;

// sort of (cos desc, j asc) over n entries: by rank, else bitonic over n padded to a power of two
__device__ void sort_cands(double* cs, int32_t* js, int n) {
  if (n <= 1) return;
  if (n <= kRankSort && n <= (int)blockDim.x) {
    const int i = threadIdx.x;
    double c = 0.0;
    int32_t j = 0;
    int rank = 0;
    if (i < n) {
      c = cs[i];
      j = js[i];
      for (int k = 0; k < n; ++k) rank += cand_before(cs[k], js[k], c, j) ? 1 : 0;
    }
    __syncthreads();
    if (i < n) { cs[rank] = c; js[rank] = j; }
    __syncthreads();
    return;
  }
  const int np = (int)pow2_ceil((uint32_t)n);
  for (int i = n + threadIdx.x; i < np; i += blockDim.x) {
    cs[i] = -2.0;
    js[i] = INT_MAX;
  }
  __syncthreads();
  for (int k = 2; k <= np; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < np; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const bool swap = up ? cand_before(cs[ixj], js[ixj], cs[i], js[i]) : cand_before(cs[i], js[i], cs[ixj], js[ixj]);
          if (swap) {
            const double tc = cs[i]; cs[i] = cs[ixj]; cs[ixj] = tc;
            const int32_t tj = js[i]; js[i] = js[ixj]; js[ixj] = tj;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ void sort_ints(int32_t* v, int n) {   // distinct values
  if (n <= 1) return;
  if (n <= kRankSort && n <= (int)blockDim.x) {
    const int i = threadIdx.x;
    int32_t x = 0;
    int rank = 0;
    if (i < n) {
      x = v[i];
      for (int k = 0; k < n; ++k) rank += v[k] < x ? 1 : 0;
    }
    __syncthreads();
    if (i < n) v[rank] = x;
    __syncthreads();
    return;
  }
  const int np = (int)pow2_ceil((uint32_t)n);
  for (int i = n + threadIdx.x; i < np; i += blockDim.x) v[i] = INT_MAX;
  __syncthreads();
  for (int k = 2; k <= np; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < np; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          if (up ? v[ixj] < v[i] : v[i] < v[ixj]) {
            const int32_t t = v[i]; v[i] = v[ixj]; v[ixj] = t;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Candidate steps of one current step in ascending j, with their full-block ranges.
struct Cands {
  int m;
  int32_t* jasc;
  int32_t* flo;
  int32_t* flen;
  int32_t* cum;    // CROSS prefix of flen [m+1]
};

__device__ __forceinline__ int32_t ceil_div(int32_t a, int32_t b) { return (a + b - 1) / b; }

__device__ void prepare_cands(const CandArgs& a, Cands& c, int64_t gfirst) {
  sort_ints(c.jasc, c.m);
  for (int r = threadIdx.x; r < c.m; r += blockDim.x) {
    const int64_t gj = gfirst + c.jasc[r];
    const int32_t lo = ceil_div(a.step_start[gj], a.block_size), hi = a.step_end[gj] / a.block_size;
    c.flo[r] = lo;
    c.flen[r] = hi > lo ? hi - lo : 0;
  }
  __syncthreads();
  if (a.pairing == MEMSHARE_PAIR_ALIGNED) return;     // only CROSS slots index through cum
  if (threadIdx.x < 32) {                            // exclusive prefix of flen, one warp
    const int lane = threadIdx.x;
    int32_t carry = 0;
    for (int base = 0; base < c.m; base += 32) {
      const int r = base + lane;
      const int32_t f = r < c.m ? c.flen[r] : 0;
      int32_t v = f;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (r < c.m) c.cum[r] = carry + v - f;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) c.cum[c.m] = carry;
  }
  __syncthreads();
}

// Logical source block of slot e for target offset i (-1 = no block in this slot).
__device__ __forceinline__ int32_t slot_logical(const Cands& c, int pairing, int32_t i, int32_t e) {
  if (pairing == MEMSHARE_PAIR_ALIGNED) return i < c.flen[e] ? c.flo[e] + i : -1;
  int lo = 0, hi = c.m - 1;   // last r with cum[r] <= e
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (c.cum[mid] <= e) lo = mid; else hi = mid - 1;
  }
  return c.flo[lo] + (e - c.cum[lo]);
}

__device__ __forceinline__ int32_t phys_of(const CandArgs& a, const int32_t* trow, int32_t lg) {
  if (lg < 0 || lg >= a.table_stride) { set_status(a.status, MEMSHARE_ERR_CORRUPTION); return INT_MIN; }
  const int32_t p = trow[lg];
  if (p < 0 || p >= a.num_blocks) set_status(a.status, MEMSHARE_ERR_CORRUPTION);
  return p;
}

// Warp-cooperative: kept (deduplicated) sources of target offset i. If `out` is non-null the
// kept pairs are written from out[0]. Returns the kept count (all lanes).
__device__ int32_t target_sources(const CandArgs& a, const Cands& c, const int32_t* trow, int32_t s, int32_t i,
                                  int32_t tl, int32_t tphys, int32_t tidx, memshare_block_pair* out, int64_t out_pos,
                                  int64_t cap) {
  const int lane = threadIdx.x & 31;
  const int32_t nslots = a.pairing == MEMSHARE_PAIR_ALIGNED ? c.m : c.cum[c.m];
  int32_t kept_total = 0;
  // a slot is kept unless an earlier slot holds the same physical block: each lane's block is
  // compared with the earlier slots' blocks broadcast from the lanes that loaded them (one table
  // load per lane per 32-slot window instead of a per-lane walk over all earlier slots)
  auto slot_phys = [&](int32_t e, bool& in_range) -> int32_t {
    const int32_t lg = e < nslots ? slot_logical(c, a.pairing, i, e) : -1;
    in_range = lg >= 0 && lg < a.table_stride;
    return in_range ? trow[lg] : 0;
  };
  for (int32_t eb = 0; eb < nslots; eb += 32) {
    const int32_t e = eb + lane;
    const int32_t lg = e < nslots ? slot_logical(c, a.pairing, i, e) : -1;
    const int32_t ph = lg >= 0 ? phys_of(a, trow, lg) : -1;
    bool dup = false;
    for (int32_t pb = 0; pb < eb; pb += 32) {
      bool r2;
      const int32_t p2 = slot_phys(pb + lane, r2);
#pragma unroll 8
      for (int t = 0; t < 32; ++t) {
        const int32_t x = __shfl_sync(0xffffffffu, p2, t);
        const bool rx = __shfl_sync(0xffffffffu, r2, t);
        dup |= rx && x == ph;
      }
    }
    bool r1;
    const int32_t p1 = slot_phys(e, r1);
    // within the window: lanes holding the same in-range block share a match mask (out-of-range
    // lanes get a key of their own); a lane whose slot is out of range (ph = INT_MIN, corrupt
    // table row) is compared lane by lane, as the earlier windows are
    const unsigned long long key = r1 ? (unsigned long long)(uint32_t)p1 : (1ull << 32) | (unsigned)lane;
    const unsigned same = __match_any_sync(0xffffffffu, key);
    dup |= (same & ((1u << lane) - 1u)) != 0u;
    if (__any_sync(0xffffffffu, lg >= 0 && !r1)) {
#pragma unroll 8
      for (int t = 0; t < 32; ++t) {
        const int32_t x = __shfl_sync(0xffffffffu, p1, t);
        const bool rx = __shfl_sync(0xffffffffu, r1, t);
        dup |= t < lane && rx && x == ph;
      }
    }
    const bool keep = lg >= 0 && !dup;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (out != nullptr && keep) {
      const int64_t pos = out_pos + kept_total + __popc(bal & ((1u << lane) - 1u));
      if (pos < cap) {
        memshare_block_pair pr;
        pr.seq = s; pr.target_idx = tidx; pr.target_logical = tl; pr.source_logical = lg;
        pr.target_phys = tphys; pr.source_phys = ph;
        out[pos] = pr;
      }
    }
    kept_total += __popc(bal);
  }
  return kept_total;
}

__device__ __forceinline__ bool is_current(const CandArgs& a, int32_t s, int64_t k, int64_t S) {
  if (a.cur_mode == MEMSHARE_CUR_ALL) return true;
  if (a.cur_mode == MEMSHARE_CUR_LAST) return k == S - 1;
  return k >= a.cur_begin[s] && k < a.cur_end[s];
}

// Tuning only (MEMSHARE_DEBUG_SKIP bit 3): per-CTA phase timestamps of stage1 (globaltimer ns).
constexpr int kDbgSlots = 16;
__device__ unsigned long long g_dbg_t[2048 * kDbgSlots];
__device__ long long g_dbg_tok[2048 * 32];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define DBG_T(slot)                                                                         \
  do {                                                                                      \
    if ((a.dbg_skip & 8) && threadIdx.x == 0 && blockIdx.x < 2048)                          \
      g_dbg_t[blockIdx.x * kDbgSlots + (slot)] = gtimer();                                  \
  } while (0)

// Stage-1 CTA shapes: 1024 threads, one CTA per SM (a single CoT / online rounds: the widest
// history stream per step), or 512 threads with half the table and staging, two CTAs per SM
// (large batches: two steps in flight per SM hide each other's latency-bound phases).
template <int NT>
struct S1Cfg {
  static constexpr int kSlots = NT == 1024 ? kSmemSlots : kSmemSlots / 2;
  static constexpr int kTok = NT == 1024 ? kHistTok : kHistTok / 2;
};

template <int NT>
struct SelSmem {
  int2 tab[S1Cfg<NT>::kSlots];
  double cs[kCandCap];
  int32_t js[kCandCap];
  union {                                     // the presence filter lives only during the history
    struct {                                  // stream; jasc / flo only after it
      int32_t jasc[kCandCap];
      int32_t flo[kCandCap];
    } l;
    uint32_t bm[kBmWords];
  } u;
  int32_t flen[kCandCap];
  int32_t cum[kCandCap + 1];
  int32_t hst[kChunk];
  int32_t hen[kChunk];
  alignas(16) int32_t tok[S1Cfg<NT>::kTok];   // staged history tokens (fused fill: reused, needs 8 B alignment)
  uint32_t dot_lo[kChunk];
  uint32_t dot_hi[kChunk];
  int64_t sh[NT / 32 + 1];
  int count;
  int overflow;
  uint32_t acc_t;
  uint32_t acc_p;
};

// Stream the history token range [clo, chi) (staged in shared memory at s_tok) through k's
// count table. Each thread takes a contiguous run, walks the step boundaries (hen, smem) and
// adds its partial dot once per step it touches. A rolled loop on purpose: this code runs once
// per launch, so instruction-fetch misses of an unrolled body cost more than the work.
template <bool kGlobal>
__device__ __forceinline__ void stream_history(const int2* tab, const uint32_t* bm, uint32_t mask, uint32_t shift,
                                               uint32_t* dot_lo,
                                               uint32_t* dot_hi, const int32_t* hen, int32_t nj, int32_t d0,
                                               int32_t dn, const Delims& dl, const int32_t* s_tok, int32_t clo,
                                               int32_t chi, bool dbg_noprobe) {
  const int32_t n = chi - clo;
  const int32_t per = (n + (int32_t)blockDim.x - 1) / (int32_t)blockDim.x;   // tokens per thread
  int32_t p = clo + (int32_t)threadIdx.x * per;
  const int32_t pe = (p + per < chi) ? p + per : chi;
  if (p >= pe) return;
  int32_t jl = 0, jh = nj - 1;                              // first step with hen > p
  while (jl < jh) {
    const int32_t mid = (jl + jh) >> 1;
    if (hen[mid] > p) jh = mid; else jl = mid + 1;
  }
  int32_t bound = hen[jl];
  uint32_t acc = 0u;
#pragma unroll 1
  for (; p < pe; ++p) {
    const int32_t tok = s_tok[p - clo];
    if (p >= bound) {
      if (acc) { const uint32_t old = atomicAdd(dot_lo + jl, acc); if (old + acc < old) atomicAdd(dot_hi + jl, 1u); }
      acc = 0u;
      do { ++jl; bound = hen[jl]; } while (p >= bound);
    }
    if (tok == d0 || (dn > 1 && is_delim(tok, dl))) continue;
    if (dbg_noprobe) { acc += (uint32_t)(tok & 1); continue; }
    const uint32_t hb = bm_bit(tok);
    if (!((bm[hb >> 5] >> (hb & 31)) & 1u)) continue;   // not in the step: no probe
    uint32_t slot = hash_slot(tok, shift);
    int32_t c = 0;
#pragma unroll 1
    for (uint32_t probe = 0; probe <= mask; ++probe) {
      const int2 e = kGlobal ? __ldcg(tab + slot) : tab[slot];
      if (e.x == tok) { c = e.y; break; }
      if (e.x == kEmpty) break;
      slot = (slot + 1) & mask;
    }
    acc += (uint32_t)c;
  }
  if (acc) { const uint32_t old = atomicAdd(dot_lo + jl, acc); if (old + acc < old) atomicAdd(dot_hi + jl, 1u); }
}

// One-CTA exclusive scans of the per-step match / target / pair counts (one pass, one set of
// barriers: the three int32 counts of a step travel packed as 3 x 21 bits when they fit).
template <int NT>
__device__ void scan_counts3(const CandArgs& a, int64_t G, int64_t* sh) {
  int64_t cm = 0, ct = 0, cp = 0;
  for (int64_t base = 0; base < G; base += NT) {
    const int64_t i = base + threadIdx.x;
    int64_t m = 0, t = 0, p = 0;
    if (i < G) { m = __ldcg(a.ws.cnt_m + i); t = __ldcg(a.ws.cnt_t + i); p = __ldcg(a.ws.cnt_p + i); }
    int64_t tot;
    // per-pass totals stay < 2^21 for each count when every step count is < 2^11 (1024 x 2047)
    const bool packed = m < 2048 && t < 2048 && p < 2048;
    const int all_packed = __syncthreads_and(packed);
    if (all_packed) {
      const int64_t ex = block_excl_scan<NT>(m | (t << 21) | (p << 42), tot, sh);
      if (i < G) {
        a.ws.off_m[i] = cm + (ex & 0x1FFFFF);
        a.ws.off_t[i] = ct + ((ex >> 21) & 0x1FFFFF);
        a.ws.off_p[i] = cp + (ex >> 42);
      }
      cm += tot & 0x1FFFFF; ct += (tot >> 21) & 0x1FFFFF; cp += tot >> 42;
    } else {
      const int64_t exm = block_excl_scan<NT>(m, tot, sh);
      if (i < G) a.ws.off_m[i] = cm + exm;
      cm += tot;
      const int64_t ext = block_excl_scan<NT>(t, tot, sh);
      if (i < G) a.ws.off_t[i] = ct + ext;
      ct += tot;
      const int64_t exp_ = block_excl_scan<NT>(p, tot, sh);
      if (i < G) a.ws.off_p[i] = cp + exp_;
      cp += tot;
    }
  }
  if (threadIdx.x == 0) { a.ws.off_m[G] = cm; a.ws.off_t[G] = ct; a.ws.off_p[G] = cp; }
}

__device__ __forceinline__ int4 s1_ld_relaxed(const int4* p) {
  int4 v;
  asm volatile("ld.relaxed.gpu.global.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void s1_st_relaxed(int4* p, int4 v) {
  asm volatile("st.relaxed.gpu.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Fused fill (offline, one CTA per step): step g publishes its {matches, targets, pairs} counts
// and obtains the exclusive prefix over steps < g by summing the published counts of ALL its
// predecessors -- independent loads, one memory latency, where a look-back walk through 32-step
// windows costs two dependent L2 round trips per window. Each count is stored +1, so every 32-bit
// word is its own "published" flag (zero: not yet; no separate flag, no fence ordering between two
// locations). One warp polls, 8 independent loads per lane in flight (against every thread
// polling one predecessor: -0.6 us per c2 step; with a __nanosleep back-off: +1.9 us). Every step
// publishes before it waits and steps are taken in ascending order by co-resident CTAs, so the
// waits always end. Returns the prefix to every thread of the CTA.
__device__ int4 s1_prefix(const CandArgs& a, int64_t g, int32_t m, int32_t t, int32_t p, int4* s_out) {
  constexpr int kU = 8;
  if (threadIdx.x == 0) s1_st_relaxed(a.ws.lb_agg + g, make_int4(m + 1, t + 1, p + 1, 1));
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int rm = 0, rt = 0, rp = 0;
    for (int64_t q0 = lane; q0 < g; q0 += 32 * kU) {
      int4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        v[u] = (q0 + 32 * u < g) ? s1_ld_relaxed(a.ws.lb_agg + q0 + 32 * u) : make_int4(1, 1, 1, 1);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        SpinGuard sg;
        while (v[u].x == 0 || v[u].y == 0 || v[u].z == 0) {
          if (sg.expired()) {                          // a predecessor never published: report, do not hang
            set_status(a.status, MEMSHARE_ERR_CORRUPTION);
            v[u] = make_int4(1, 1, 1, 1);
            break;
          }
          v[u] = s1_ld_relaxed(a.ws.lb_agg + q0 + 32 * u);
        }
        rm += v[u].x - 1;
        rt += v[u].y - 1;
        rp += v[u].z - 1;
      }
    }
    rm = warp_sum(rm);
    rt = warp_sum(rt);
    rp = warp_sum(rp);
    if (lane == 0) *s_out = make_int4(rm, rt, rp, 0);
  }
  __syncthreads();
  return *s_out;
}

// the last step's CTA: totals and target_off[T]
__device__ void s1_totals(const CandArgs& a, int4 incl) {
  if (threadIdx.x == 0) {
    const int64_t M = incl.x, T = incl.y, P = incl.z;
    *a.num_matches = M;
    *a.num_targets = T;
    *a.num_pairs = P;
    if (M > a.match_cap || T > a.target_cap || P > a.pair_cap) set_status(a.status, MEMSHARE_ERR_CAPACITY);
    if (T <= a.target_cap) a.target_off[T] = P;
  }
}


// Publish "no outputs" for work item `key` of the fused fill (all CTA threads call it; the last key
// also writes the totals).
template <int NT>
__device__ void s1_publish_nothing(const CandArgs& a, int64_t key, int64_t nwork, int4* s_lb) {
  if (key == nwork - 1) {
    const int4 pre = s1_prefix(a, key, 0, 0, 0, s_lb);
    s1_totals(a, pre);
  } else if (threadIdx.x == 0) {
    s1_st_relaxed(a.ws.lb_agg + key, make_int4(1, 1, 1, 1));
  }
}

// Publish "no outputs" for the keys [k0, k1) (all CTA threads; the last key also the totals).
template <int NT>
__device__ void s1_publish_zero_range(const CandArgs& a, int64_t k0, int64_t k1, int64_t nwork,
                                                   int4* s_lb) {
  for (int64_t key = k0 + threadIdx.x; key < k1; key += NT)
    if (key != nwork - 1) s1_st_relaxed(a.ws.lb_agg + key, make_int4(1, 1, 1, 1));
  if (k0 <= nwork - 1 && nwork - 1 < k1) s1_publish_nothing<NT>(a, nwork - 1, nwork, s_lb);
}

// One Stage-1 work item: current step g (local k) of sequence s (steps [gfirst, gfirst + S)):
// table, history stream (this CTA's share of a cluster's), selection, pair counts and -- fused --
// the fill. All threads of the CTA (and of its cluster) call it.
template <int NT>
__device__ void s1_item(const CandArgs& a, SelSmem<NT>& sm, int64_t wi, int64_t g, int32_t s, int64_t gfirst,
                        int64_t S, bool fused, int64_t nwork, int4* s_lb_p) {
  constexpr int kNTs = NT, kNWs = NT / 32;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int csize = (int)cl.num_blocks(), crank = (int)cl.block_rank();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int4& s_lb = *s_lb_p;
  auto publish_nothing = [&](int64_t key) { s1_publish_nothing<NT>(a, key, nwork, s_lb_p); };
  const int64_t k = g - gfirst;
  // every per-step value the item needs, issued together before the first branch (one memory
  // latency instead of a chain: the branch on nbag kept the compiler from hoisting the others)
  const int32_t nbag = a.step_nbag[g];
  const int64_t tok_base = a.seq_tok_off[s];
  const int32_t st_start = a.step_start[g], st_end = a.step_end[g];
  const int64_t n2_raw = a.ws.n2[g];
  if (nbag == 0 || !is_current(a, s, k, S)) {
    if (crank == 0 && threadIdx.x == 0) { a.ws.cnt_m[g] = 0; a.ws.cnt_t[g] = 0; a.ws.cnt_p[g] = 0; a.ws.stash_base[g] = 0; }
    if (fused && crank == 0) publish_nothing(wi);
    return;
  }
  const int32_t* t = a.tokens + tok_base;
  const Table tb = build_table(a, sm.tab, t, tok_base, st_start, st_end, nbag, S1Cfg<NT>::kSlots,
                               sm.u.bm, crank == 0);
  if (tb.global && csize > 1) cl.sync();                 // rank 0 filled the shared global table
  DBG_T(1);
  const double n2k = (double)n2_raw;
  if (threadIdx.x == 0) { sm.count = 0; sm.overflow = 0; }
  __syncthreads();
  const bool compact = a.top_k > 0 && a.top_k <= kCandCap / 2;
  // The history of step k is the contiguous token range [start_0, end_{k-1}) of the sequence:
  // stream it with all threads (coalesced), look each content token up in k's table and add
  // the count to the dot product of the step that holds it (smem atomics, only for hits).
  for (int64_t jb = 0; jb < k; jb += kChunk) {
    const int64_t je = (jb + kChunk < k) ? jb + kChunk : k;
    const int nj = (int)(je - jb);
    for (int i = threadIdx.x; i < nj; i += kNTs) {
      sm.hst[i] = a.step_start[gfirst + jb + i];
      sm.hen[i] = a.step_end[gfirst + jb + i];
      sm.dot_lo[i] = 0u;
      sm.dot_hi[i] = 0u;
    }
    __syncthreads();
    if (jb == 0) DBG_T(10);
    if (jb == 0 && (a.dbg_skip & 8) && threadIdx.x == 0 && blockIdx.x < 2048)
      g_dbg_t[blockIdx.x * kDbgSlots + 12] = clock64();
    const int32_t lo0 = sm.hst[0], hi0 = sm.hen[nj - 1];
    const int32_t lo = lo0 + (int32_t)((int64_t)(hi0 - lo0) * crank / csize);      // this rank's share
    const int32_t hi = lo0 + (int32_t)((int64_t)(hi0 - lo0) * (crank + 1) / csize);
    for (int32_t clo = lo; clo < hi; clo += S1Cfg<NT>::kTok) {
      const int32_t chi = (hi - clo > S1Cfg<NT>::kTok) ? clo + S1Cfg<NT>::kTok : hi;
      // coalesced, independent loads: one memory latency for the whole pass
#pragma unroll 4
      for (int32_t i = threadIdx.x; i < chi - clo; i += kNTs) sm.tok[i] = __ldg(t + clo + i);
      __syncthreads();
      if (jb == 0 && clo == lo) DBG_T(14);
      if (!(a.dbg_skip & 1)) {
        if (tb.global)
          stream_history<true>(tb.slots, sm.u.bm, tb.mask, tb.shift, sm.dot_lo, sm.dot_hi, sm.hen, nj, a.dl.id[0], a.dl.n,
                               a.dl, sm.tok, clo, chi, (a.dbg_skip & 16) != 0);
        else
          stream_history<false>(sm.tab, sm.u.bm, tb.mask, tb.shift, sm.dot_lo, sm.dot_hi, sm.hen, nj, a.dl.id[0], a.dl.n,
                                a.dl, sm.tok, clo, chi, (a.dbg_skip & 16) != 0);
      }
      __syncthreads();
    }
    __syncthreads();
    if (csize > 1) {
      cl.sync();                                         // every rank's partial dots are final
      if (crank == 0) {
        // every remote load issued before any sum (one DSMEM latency, not csize - 1 of them)
        for (int i = threadIdx.x; i < nj; i += kNTs) {
          uint32_t lo_r[8], hi_r[8];
#pragma unroll
          for (int r = 1; r < 8; ++r) {
            lo_r[r] = r < csize ? cl.map_shared_rank(sm.dot_lo, r)[i] : 0u;
            hi_r[r] = r < csize ? cl.map_shared_rank(sm.dot_hi, r)[i] : 0u;
          }
          uint64_t d = ((uint64_t)sm.dot_hi[i] << 32) | sm.dot_lo[i];
#pragma unroll
          for (int r = 1; r < 8; ++r) d += ((uint64_t)hi_r[r] << 32) | lo_r[r];
          sm.dot_lo[i] = (uint32_t)d;
          sm.dot_hi[i] = (uint32_t)(d >> 32);
        }
      }
      cl.sync();                                         // remote reads done before ranks reuse them
      if (crank != 0) continue;                          // ranks > 0 only stream (uniform per CTA)
    }
    if (jb == 0) DBG_T(11);
    if (jb == 0 && (a.dbg_skip & 8) && threadIdx.x == 0 && blockIdx.x < 2048)
      g_dbg_t[blockIdx.x * kDbgSlots + 13] = clock64();
    for (int i = threadIdx.x; i < nj; i += kNTs) {
      const int64_t gj = gfirst + jb + i;
      if (a.step_nbag[gj] == 0) continue;                // void history step (reading R5)
      const int64_t dot = (int64_t)(((uint64_t)sm.dot_hi[i] << 32) | sm.dot_lo[i]);
      // sim = <v_curr, v_i> / (||v_curr|| ||v_i||), reading R12
      const double cs = __ddiv_rn(__ll2double_rn(dot), __dsqrt_rn(__dmul_rn(n2k, __ll2double_rn(a.ws.n2[gj]))));
      if (cs > a.tau_s) {                                // strict: "exceeding"
        const int idx = atomicAdd(&sm.count, 1);
        if (idx < kCandCap) { sm.cs[idx] = cs; sm.js[idx] = (int32_t)(jb + i); }
        else sm.overflow = 1;
      }
    }
    __syncthreads();
    if (compact && sm.count > kCandCap / 2) {
      sort_cands(sm.cs, sm.js, sm.count);
      __syncthreads();
      if (threadIdx.x == 0) sm.count = a.top_k;
      __syncthreads();
    }
  }
  if (crank != 0) return;
  DBG_T(2);
  if (sm.overflow) {
    if (threadIdx.x == 0) set_status(a.status, MEMSHARE_ERR_CAPACITY);
    __syncthreads();
  }
  int m = sm.count < kCandCap ? sm.count : kCandCap;
  sort_cands(sm.cs, sm.js, m);
  if (a.top_k > 0 && m > a.top_k) m = a.top_k;
  DBG_T(3);
  // stash the ranked survivors for the fill kernel
  __shared__ unsigned long long s_base;
  if (threadIdx.x == 0) {
    s_base = (m > 0 && !fused) ? atomicAdd(a.ws.stash_alloc, (unsigned long long)m) : 0ull;
    if (!fused && (int64_t)(s_base + m) > a.match_cap) set_status(a.status, MEMSHARE_ERR_CAPACITY);
  }
  __syncthreads();
  const int64_t base = (int64_t)s_base;
  for (int r = threadIdx.x; r < m; r += kNTs) {
    if (!fused && base + r < a.match_cap) { a.ws.stash_cos[base + r] = sm.cs[r]; a.ws.stash_j[base + r] = sm.js[r]; }
    sm.u.l.jasc[r] = sm.js[r];
  }
  if (threadIdx.x == 0) { sm.acc_t = 0u; sm.acc_p = 0u; }
  __syncthreads();
  // a4: count targets and deduplicated pairs of this step
  DBG_T(4);
  Cands c{m, sm.u.l.jasc, sm.u.l.flo, sm.flen, sm.cum};
  prepare_cands(a, c, gfirst);
  DBG_T(5);
  const int32_t fk_lo = ceil_div(a.step_start[g], a.block_size), fk_hi = a.step_end[g] / a.block_size;
  const int32_t nt = (m > 0 && fk_hi > fk_lo) ? fk_hi - fk_lo : 0;
  if (nt > kMaxTgt && threadIdx.x == 0) set_status(a.status, MEMSHARE_ERR_CAPACITY);
  const int32_t* trow = a.table + (int64_t)s * a.table_stride;
  int64_t my_t = 0, my_p = 0;
  // fused fill: the history staging area is free now; it holds the per-target kept counts,
  // pair offsets and target numbers of the step (kMaxTgt x 16 B = 64 KiB)
  int32_t* f_tc = reinterpret_cast<int32_t*>(sm.tok);
  int64_t* f_tpos = reinterpret_cast<int64_t*>(f_tc + kMaxTgt);
  int32_t* f_tnum = reinterpret_cast<int32_t*>(f_tpos + kMaxTgt);
  for (int32_t i = w; i < nt && !(a.dbg_skip & 2); i += kNWs) {
    const int32_t kept = target_sources(a, c, trow, s, i, fk_lo + i, 0, 0, nullptr, 0, 0);
    my_t += kept > 0 ? 1 : 0;
    my_p += kept;
    if (fused && lane == 0 && i < kMaxTgt) f_tc[i] = kept;
  }
  if (lane == 0) { atomicAdd(&sm.acc_t, (uint32_t)my_t); atomicAdd(&sm.acc_p, (uint32_t)my_p); }
  __syncthreads();
  DBG_T(6);
  if (threadIdx.x == 0) {
    a.ws.cnt_m[g] = m;
    a.ws.cnt_t[g] = (int32_t)sm.acc_t;
    a.ws.cnt_p[g] = (int32_t)sm.acc_p;
    a.ws.stash_base[g] = base;
  }
  __syncthreads();
  if (fused) {
    // offsets of this step's outputs, then the fill kernel's work done here
    const int4 pre = s1_prefix(a, wi, m, (int32_t)sm.acc_t, (int32_t)sm.acc_p, &s_lb);
    DBG_T(8);
    if (wi == nwork - 1) s1_totals(a, make_int4(pre.x + m, pre.y + (int32_t)sm.acc_t, pre.z + (int32_t)sm.acc_p, 0));
    const int64_t mo = pre.x, to = pre.y, po = pre.z;
    for (int r = threadIdx.x; r < m; r += kNTs) {
      if (mo + r < a.match_cap) {
        memshare_step_match mt;
        mt.seq = s; mt.step = (int32_t)k; mt.cand_step = sm.js[r]; mt.rank = r; mt.cosine = sm.cs[r];
        a.matches[mo + r] = mt;
      }
    }
    const int32_t ntf = nt < kMaxTgt ? nt : kMaxTgt;
    int64_t pcarry = 0, tcarry = 0;
    for (int32_t ib = 0; ib < ntf; ib += kNTs) {
      const int32_t i = ib + threadIdx.x;
      const int64_t v = i < ntf ? f_tc[i] : 0;
      int64_t tot;
      const int64_t ex = block_excl_scan<NT>(v, tot, sm.sh);
      int64_t tt;
      const int64_t tex = block_excl_scan<NT>(v > 0 ? 1 : 0, tt, sm.sh);
      if (i < ntf) { f_tpos[i] = pcarry + ex; f_tnum[i] = v > 0 ? (int32_t)(tcarry + tex) : -1; }
      pcarry += tot;
      tcarry += tt;
    }
    __syncthreads();
    DBG_T(9);
    for (int32_t i = w; i < ntf; i += kNWs) {
      if (f_tnum[i] < 0) continue;
      const int64_t tidx = to + f_tnum[i];
      const int32_t tl = fk_lo + i;
      const int32_t tphys = phys_of(a, trow, tl);
      target_sources(a, c, trow, s, i, tl, tphys, (int32_t)tidx, a.pairs, po + f_tpos[i], a.pair_cap);
      if (lane == 0 && tidx < a.target_cap) a.target_off[tidx] = po + f_tpos[i];
    }
    __syncthreads();
  }
}

// RI: the RANGE-work-item instantiation (a separate kernel keeps the ALL / LAST kernels' code --
// run once per launch, instruction-fetch sensitive -- as small as before)
template <int NT, bool RI = false>
__global__ void __launch_bounds__(NT, 1024 / NT) stage1_kernel(CandArgs a) {
  constexpr int kNTs = NT;
  static_assert(NT != 1024 || kMaxTgt * 16 <= S1Cfg<1024>::kTok * 4, "fused fill reuses the staging area");
  const bool fused = NT == 1024 && a.fused != 0;   // the 512-thread shape never fuses
  pdl_trigger();
  TL_SCOPE(3);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SelSmem<NT>& sm = *reinterpret_cast<SelSmem<NT>*>(smem_raw);
  // Thread-block cluster of csize CTAs per current step (online rounds: few current steps, long
  // histories): every rank builds the step's table, streams 1/csize of the history into its own
  // shared dot array, and rank 0 sums the ranks' arrays over DSMEM and does the selection.
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int csize = (int)cl.num_blocks(), crank = (int)cl.block_rank();
  DBG_T(0);
  const int64_t G = total_steps(a);
  __shared__ int4 s_lb;
  // LAST (online): the work list is one step per sequence, found directly; without the fused fill
  // the counts of every other step are zeroed up front by all threads (one parallel pass instead
  // of a chain of dependent loads per skipped step) for the last-CTA scan.
  const bool last_mode = a.cur_mode == MEMSHARE_CUR_LAST;
  const bool range_items = RI && fused && a.range_items != 0;
  // publication keys: sequences (LAST) or steps; work items: the keys, or -- RANGE with the fused
  // fill -- the current steps only, each publishing zeros for the non-current keys before it (the
  // last one also for those after it)
  const int64_t nwork = last_mode ? a.num_seqs : G;
  const int64_t nitems = range_items ? __ldcg(a.ws.cur_off + a.num_seqs) : nwork;
  // fused fill: work item wi publishes its counts at key wi (= g offline, = the sequence online);
  // the last key also writes the totals
  if (fused && (nwork == 0 || nitems == 0) && blockIdx.x == 0) s1_totals(a, make_int4(0, 0, 0, 0));
  auto publish_zero_range = [&](int64_t k0, int64_t k1) { s1_publish_zero_range<NT>(a, k0, k1, nwork, &s_lb); };
  auto publish_nothing = [&](int64_t key) {     // a work item without outputs (all CTA threads call it)
    if (key == nwork - 1) {
      const int4 pre = s1_prefix(a, key, 0, 0, 0, &s_lb);
      s1_totals(a, pre);
    } else if (threadIdx.x == 0) {
      s1_st_relaxed(a.ws.lb_agg + key, make_int4(1, 1, 1, 1));
    }
  };
  if (last_mode && !fused) {
    for (int64_t g = (int64_t)blockIdx.x * kNTs + threadIdx.x; g < G; g += (int64_t)gridDim.x * kNTs) {
      const int32_t s = a.ws.step_seq[g];
      if (g != a.seq_step_off[s + 1] - 1) { a.ws.cnt_m[g] = 0; a.ws.cnt_t[g] = 0; a.ws.cnt_p[g] = 0; a.ws.stash_base[g] = 0; }
    }
  }
  // Work items come from an atomic ticket (ascending), not a static CTA -> item map: an item's
  // fused-fill prefix waits only on items with smaller tickets, which running CTAs already hold
  // and which never wait on larger ones, so progress does not depend on how many CTAs (or
  // clusters) are co-resident (a static map deadlocks when fewer fit than were launched).
  __shared__ unsigned long long s_ticket;
  for (bool first = true;; first = false) {
    int64_t wi;
    if (csize == 1) {
      __syncthreads();                                     // everyone has read the previous ticket
      if (threadIdx.x == 0) s_ticket = atomicAdd(a.ws.ticket, 1ull);
      __syncthreads();
      wi = (int64_t)s_ticket;
    } else {
      // every rank has read rank 0's previous ticket (none before the first: the barrier below
      // alone orders rank 0's write before the remote reads)
      if (!first) cl.sync();
      if (crank == 0 && threadIdx.x == 0) s_ticket = atomicAdd(a.ws.ticket, 1ull);
      cl.sync();
      wi = (int64_t)*cl.map_shared_rank(&s_ticket, 0);
    }
    if (wi >= nitems) {
      // rank 0 may not exit while another rank still reads its s_ticket over DSMEM
      if (csize > 1) cl.sync();
      break;
    }
    // one s1_item call site (a second inlined copy costs instruction-cache misses: this code runs
    // once per launch)
    int64_t key, g;
    int32_t s;
    if (range_items) {
      g = range_item_step(a, wi, G, s);
      int32_t sp;
      const int64_t gprev = wi > 0 ? range_item_step(a, wi - 1, G, sp) : -1;
      if (crank == 0) publish_zero_range(gprev + 1, g);          // the non-current keys before g
      key = g;
    } else {
      g = last_mode ? a.seq_step_off[wi + 1] - 1 : wi;
      if (last_mode && (g < a.seq_step_off[wi] || g >= G)) {            // sequence without steps
        if (fused && crank == 0) publish_nothing(wi);
        continue;
      }
      s = last_mode ? (int32_t)wi : a.ws.step_seq[g];       // LAST: the item is the sequence
      key = wi;
    }
    const int64_t gfirst = a.seq_step_off[s];
    const int64_t S = a.seq_step_off[s + 1] - gfirst;
    s1_item<NT>(a, sm, key, g, s, gfirst, S, fused, nwork, &s_lb);
    // Every cluster takes exactly one ticket first, so with no more items than clusters every item
    // is already held: leave without the second ticket round trip (s1_item's last cluster barrier
    // follows the last DSMEM access, so no rank reads another's shared memory after this point).
    if (range_items && wi == nitems - 1 && crank == 0) publish_zero_range(g + 1, nwork);   // and after the last
    if (nitems <= (int64_t)(gridDim.x / csize)) break;
  }
  DBG_T(7);
  if (!fused && !(a.dbg_skip & 4) && last_block_done(a.ws.done)) {
    DBG_T(8);
    scan_counts3<NT>(a, G, sm.sh);
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t M = a.ws.off_m[G], T = a.ws.off_t[G], P = a.ws.off_p[G];
      *a.num_matches = M;
      *a.num_targets = T;
      *a.num_pairs = P;
      if (M > a.match_cap || T > a.target_cap || P > a.pair_cap) set_status(a.status, MEMSHARE_ERR_CAPACITY);
      if (T <= a.target_cap) a.target_off[T] = P;
    }
    DBG_T(9);
  }
}

struct FillSmem {
  double cs[kCandCap];
  int32_t js[kCandCap];
  union {                                     // the presence filter lives only during the history
    struct {                                  // stream; jasc / flo only after it
      int32_t jasc[kCandCap];
      int32_t flo[kCandCap];
    } l;
    uint32_t bm[kBmWords];
  } u;
  int32_t flen[kCandCap];
  int32_t cum[kCandCap + 1];
  int32_t tc[kMaxTgt];
  int64_t tpos[kMaxTgt];   // pair offset (within the step) of each target offset i
  int32_t tnum[kMaxTgt];   // target number (within the step), -1 if no pair
  int64_t sh[kNW + 1];
};

__global__ void __launch_bounds__(kNT) fill_kernel(CandArgs a) {
  pdl_trigger();
  TL_SCOPE(4);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FillSmem& sm = *reinterpret_cast<FillSmem*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t G = total_steps(a);
  for (int64_t g = blockIdx.x; g < G; g += gridDim.x) {
    const int m = a.ws.cnt_m[g];
    if (m == 0) continue;
    const int32_t s = a.ws.step_seq[g];
    const int64_t gfirst = a.seq_step_off[s];
    const int64_t k = g - gfirst;
    const int64_t sbase = a.ws.stash_base[g];
    if (sbase + m > a.match_cap) continue;              // stash overflowed: CAPACITY already set
    const int64_t mo = a.ws.off_m[g];
    for (int r = threadIdx.x; r < m; r += kNT) {
      const double cs = a.ws.stash_cos[sbase + r];
      const int32_t j = a.ws.stash_j[sbase + r];
      sm.u.l.jasc[r] = j;
      if (mo + r < a.match_cap) {
        memshare_step_match mt;
        mt.seq = s; mt.step = (int32_t)k; mt.cand_step = j; mt.rank = r; mt.cosine = cs;
        a.matches[mo + r] = mt;
      }
    }
    __syncthreads();
    Cands c{m, sm.u.l.jasc, sm.u.l.flo, sm.flen, sm.cum};
    prepare_cands(a, c, gfirst);
    const int32_t fk_lo = ceil_div(a.step_start[g], a.block_size), fk_hi = a.step_end[g] / a.block_size;
    int32_t nt = fk_hi > fk_lo ? fk_hi - fk_lo : 0;
    if (nt > kMaxTgt) continue;                          // CAPACITY already set by stage1
    const int32_t* trow = a.table + (int64_t)s * a.table_stride;
    for (int32_t i = w; i < nt; i += kNW) {
      const int32_t kept = target_sources(a, c, trow, s, i, fk_lo + i, 0, 0, nullptr, 0, 0);
      if (lane == 0) sm.tc[i] = kept;
    }
    __syncthreads();
    // per-target pair offsets and target numbers within the step (block scans)
    int64_t pcarry = 0, tcarry = 0;
    for (int32_t ib = 0; ib < nt; ib += kNT) {
      const int32_t i = ib + threadIdx.x;
      const int64_t v = i < nt ? sm.tc[i] : 0;
      int64_t tot;
      const int64_t ex = block_excl_scan<kNT>(v, tot, sm.sh);
      int64_t tt;
      const int64_t tex = block_excl_scan<kNT>(v > 0 ? 1 : 0, tt, sm.sh);
      if (i < nt) { sm.tpos[i] = pcarry + ex; sm.tnum[i] = v > 0 ? (int32_t)(tcarry + tex) : -1; }
      pcarry += tot;
      tcarry += tt;
    }
    __syncthreads();
    const int64_t po = a.ws.off_p[g], to = a.ws.off_t[g];
    for (int32_t i = w; i < nt; i += kNW) {
      if (sm.tnum[i] < 0) continue;
      const int64_t tidx = to + sm.tnum[i];
      const int32_t tl = fk_lo + i;
      const int32_t tphys = phys_of(a, trow, tl);
      target_sources(a, c, trow, s, i, tl, tphys, (int32_t)tidx, a.pairs, po + sm.tpos[i], a.pair_cap);
      if (lane == 0 && tidx < a.target_cap) a.target_off[tidx] = po + sm.tpos[i];
    }
    __syncthreads();
  }
}


}  // namespace
}  // namespace ms

using namespace ms;

TL_EXPORT(candidates)

extern "C" int memshare_debug_stage1_tok(long long* host, int n) {
  if (n > 2048 * 32) n = 2048 * 32;
  return (int)cudaMemcpyFromSymbol(host, g_dbg_tok, (size_t)n * sizeof(long long));
}

// Tuning only, not part of the public ABI: copy the stage1 phase timestamps to the host.
extern "C" int memshare_debug_stage1_times(unsigned long long* host, int n) {
  if (n > 2048 * kDbgSlots) n = 2048 * kDbgSlots;
  return (int)cudaMemcpyFromSymbol(host, g_dbg_t, (size_t)n * sizeof(unsigned long long));
}

extern "C" size_t memshare_step_candidates_workspace_size(int64_t num_tokens, int32_t num_seqs, int64_t step_cap,
                                                          int64_t match_cap) {
  if (num_tokens < 0 || num_seqs < 0 || step_cap < 0 || match_cap < 0) return 0;
  Ws w{nullptr, 0};
  cand_layout(w, num_tokens, step_cap, match_cap, num_seqs);
  return w.size();
}

static bool fused_env() {            // MEMSHARE_FUSED_FILL=0: separate fill kernel (A/B)
  static int on = -1;
  if (on < 0) { const char* e = getenv("MEMSHARE_FUSED_FILL"); on = (e && e[0] == '0') ? 0 : 1; }
  return on == 1;
}

extern "C" memshare_status memshare_step_candidates(
    const int32_t* tokens, int64_t num_tokens, const int64_t* seq_tok_off, int32_t num_seqs,
    const int64_t* seq_step_off, const int32_t* step_start, const int32_t* step_end, const int32_t* step_nbag,
    int64_t step_cap, const int32_t* delim_ids_host, int32_t num_delims, int32_t cur_mode, const int32_t* cur_begin,
    const int32_t* cur_end, const int32_t* block_table, int32_t table_stride, int32_t num_blocks, int32_t block_size,
    double tau_s, int32_t top_k, int32_t pairing, memshare_step_match* matches, int64_t match_cap,
    int64_t* num_matches, memshare_block_pair* pairs, int64_t pair_cap, int64_t* num_pairs, int64_t* target_off,
    int64_t target_cap, int64_t* num_targets, void* workspace, size_t workspace_bytes, int32_t* device_status,
    void* stream) {
  MS_NVTX("memshare_step_candidates");
  if (num_tokens < 0 || num_seqs < 0 || step_cap < 0 || match_cap < 0 || pair_cap < 0 || target_cap < 0)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (num_delims < 1 || num_delims > MEMSHARE_MAX_DELIMS || !delim_ids_host) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (cur_mode < MEMSHARE_CUR_ALL || cur_mode > MEMSHARE_CUR_RANGE) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (cur_mode == MEMSHARE_CUR_RANGE && num_seqs > 0 && (!cur_begin || !cur_end)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (pairing != MEMSHARE_PAIR_ALIGNED && pairing != MEMSHARE_PAIR_CROSS) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (!(tau_s >= -1.0 && tau_s <= 1.0) || top_k < 0 || block_size < 1 || table_stride < 0 || num_blocks < 0)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (num_tokens > (int64_t)INT32_MAX / 4) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (!seq_tok_off || !seq_step_off || !num_matches || !num_pairs || !num_targets || !target_off || !workspace ||
      !device_status)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (num_seqs > 0 && (!tokens || !block_table)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (step_cap > 0 && (!step_start || !step_end || !step_nbag)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if ((match_cap > 0 && !matches) || (pair_cap > 0 && !pairs)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < memshare_step_candidates_workspace_size(num_tokens, num_seqs, step_cap, match_cap))
    return MEMSHARE_ERR_INVALID_ARGUMENT;

  CandArgs a{};
  a.tokens = tokens; a.seq_tok_off = seq_tok_off; a.num_seqs = num_seqs; a.seq_step_off = seq_step_off;
  a.step_start = step_start; a.step_end = step_end; a.step_nbag = step_nbag; a.step_cap = step_cap;
  a.dl.n = num_delims;
  for (int i = 0; i < num_delims; ++i) a.dl.id[i] = delim_ids_host[i];
  a.cur_mode = cur_mode; a.cur_begin = cur_begin; a.cur_end = cur_end;
  a.table = block_table; a.table_stride = table_stride; a.num_blocks = num_blocks; a.block_size = block_size;
  a.tau_s = tau_s; a.top_k = top_k; a.pairing = pairing;
  a.matches = matches; a.match_cap = match_cap; a.num_matches = num_matches;
  a.pairs = pairs; a.pair_cap = pair_cap; a.num_pairs = num_pairs;
  a.target_off = target_off; a.target_cap = target_cap; a.num_targets = num_targets;
  a.status = device_status;
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* e = getenv("MEMSHARE_DEBUG_SKIP");
      dbg = e ? atoi(e) : 0;
#ifndef MEMSHARE_TUNING
      dbg &= 8;   // shipped library: only the (harmless) phase stamps; work-skipping masks need -DMEMSHARE_TUNING
#endif
    }
    a.dbg_skip = dbg;
  }
  Ws w{static_cast<char*>(workspace), 0};
  a.ws = cand_layout(w, num_tokens, step_cap, match_cap, num_seqs);

  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static bool attr_set_dev[kMaxDevices] = {};
  bool& attr_set = attr_set_dev[current_device()];
  if (!attr_set) {
    cudaFuncSetAttribute(stage1_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SelSmem<1024>));
    cudaFuncSetAttribute(stage1_kernel<1024, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(SelSmem<1024>));
    cudaFuncSetAttribute(stage1_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SelSmem<512>));
    cudaFuncSetAttribute(encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSmemSlots * sizeof(int2)));
    cudaFuncSetAttribute(encode_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(kSmemSlots * sizeof(int2)));
    cudaFuncSetAttribute(fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FillSmem));
    attr_set = true;
  }
  const int sms = sm_count();
  const int64_t gcap = step_cap < 1 ? 1 : step_cap;
  // a2 encode: one CTA per step while the steps (~1 per 100 tokens) fit in 8 waves of CTAs,
  // one warp per step beyond (large batches: 8 steps in flight per CTA)
  const bool enc_warp = num_tokens > (int64_t)100 * 8 * sms;
  const int64_t enc_ctas = enc_warp ? (gcap + kNW - 1) / kNW : gcap;
  const int grid_enc = (int)(enc_ctas < 8 * sms ? enc_ctas : 8 * sms);
  const int grid_sel = (int)(gcap < 2 * sms ? gcap : 2 * sms);
  // Stage-1 shape (decided first: the encode kernel prepares RANGE work items for it). Cluster
  // size per current step: online rounds (LAST: one current step per sequence; RANGE: work items
  // are the current steps, sized for a few per sequence) split each step's history over up to 8
  // CTAs while the clusters still fit in one wave; offline (ALL) keeps one CTA per step.
  // MEMSHARE_S1_CLUSTER overrides the online size (tuning / regression tests).
  static int env_cs = -1;
  if (env_cs < 0) { const char* e = getenv("MEMSHARE_S1_CLUSTER"); env_cs = e ? atoi(e) : 0; }
  int cs = 1;
  if (env_cs > 0 && cur_mode != MEMSHARE_CUR_ALL) cs = env_cs;    // forced (tuning / regression tests)
  else if (cur_mode != MEMSHARE_CUR_ALL)
    for (int c = 8; c > 1; c >>= 1)
      if ((int64_t)num_seqs * c <= sms) { cs = c; break; }
  if (cs != 1 && cs != 2 && cs != 4 && cs != 8) cs = 1;
  // large batches without clusters: 512-thread CTAs, two per SM (MEMSHARE_S1_NT overrides)
  static int env_nt = -1;
  if (env_nt < 0) { const char* e = getenv("MEMSHARE_S1_NT"); env_nt = e ? atoi(e) : 0; }
  const bool half = cs == 1 && (env_nt == 512 || (env_nt == 0 && enc_warp));
  // the fused fill: stage1 also writes the matches and pairs (offsets from the predecessors'
  // published counts), so no fill kernel and no last-CTA scan -- offline with the steps as keys,
  // LAST with the sequences as keys, RANGE with the steps as keys and the current steps as items
  a.fused = (!half && fused_env() && (cur_mode != MEMSHARE_CUR_LAST || (int64_t)num_seqs <= step_cap + 1)) ? 1 : 0;
  a.range_items = (cur_mode == MEMSHARE_CUR_RANGE && a.fused) ? 1 : 0;
  if (enc_warp)
    launch_pdl(encode_warp_kernel, dim3(grid_enc), dim3(kNT), kSmemSlots * sizeof(int2), st, a);
  else
    launch_pdl(encode_kernel, dim3(grid_enc), dim3(kNT), kSmemSlots * sizeof(int2), st, a);
  {
    const int per_sm = half ? 2 : 1;
    const int ncl = (int)((gcap < (int64_t)per_sm * sms / cs) ? gcap : (int64_t)per_sm * sms / cs);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(ncl * cs));
    cfg.blockDim = dim3(half ? 512 : 1024);
    cfg.dynamicSmemBytes = half ? sizeof(SelSmem<512>) : sizeof(SelSmem<1024>);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = (unsigned)cs;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, half ? stage1_kernel<512> : (a.range_items ? stage1_kernel<1024, true>
                                                                            : stage1_kernel<1024>), a) != cudaSuccess)
      return MEMSHARE_ERR_CUDA;
  }
  if (!a.fused) launch_pdl(fill_kernel, dim3(grid_sel), dim3(kNT), sizeof(FillSmem), st, a);
  return launch_status();
}
