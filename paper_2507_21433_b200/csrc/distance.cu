// a5-a6 -- Stage 2 block distance + threshold + per-target selection.
// PAPER.md:237-248 (Alg. 1 Stage 2):  D = (1/N) sum_l (||K_l[Bt]-K_l[Bs]||_F + ||V_l[Bt]-V_l[Bs]||_F)/(2dh)
// PAPER.md:268 ("small Euclidean distance are flagged as reusable"), :319-320 (minimal distance).
//
// B200 design. The op is a bf16 reduction bound by HBM, not a contraction: no
// tensor cores. Three launches:
//  plan_kernel -- one CTA: targets sorted by (first source block, index) in shared memory
//   (bitonic); runs of <= kAnchors targets with the same first source become ITEMS (<= 64 pairs).
//   Near-copies of one earlier step (redundant thinking) pair with the same
//   source blocks, so the targets of an item share most of their sources.
//  distance_kernel -- one persistent CTA per SM, warp-specialised:
//   * warp 16 (producer) takes (item, layer chunk) units from a global ticket, layer-chunk-major
//     so that all SMs work on the same layers at a time (the per-layer working set stays in
//     L2); for every (layer, K|V, sub-slice) it issues one 1-D TMA bulk copy (cp.async.bulk,
//     SASS UBLKCP) per ANCHOR (the item's targets) and then one per DISTINCT source of the item
//     into a 6-stage 32 KiB shared-memory ring, completed through mbarrier transaction counts;
//     each stage carries the list of pairs to evaluate against it;
//   * warps 0-15 (consumers) copy each stage into registers and release it at once; anchors stay
//     in registers (bf16, 4 x 16 regs); every other stage is evaluated against the anchors its
//     pairs name: d = t - s (FFMA2, exactly rounded), acc += d*d (FFMA2, fp32, 32 terms per
//     thread), warp-shuffle sum, one fp32 partial per warp (fixed order, no fp atomics).
//   A source shared by several targets of an item crosses HBM->SMEM once per item.
//  finalize_kernel -- one CTA per target: fixed-order fp32 sums of the warp partials, fp64 sqrt,
//   /(2dh), layer mean, fp32 distance, the strict tau_b test and the argmin with the
//   smaller-source-logical tie break.
#include <cfloat>
#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace ms {
namespace {

// Tuning knobs (compile-time; defaults are the shipped configuration).
#ifndef MS_CONSUMER_WARPS
#define MS_CONSUMER_WARPS 8
#endif
#ifndef MS_STAGE_BYTES
#define MS_STAGE_BYTES 32768
#endif
#ifndef MS_STAGES
#define MS_STAGES 6
#endif
#ifndef MS_DIAG_NO_COMPUTE
#define MS_DIAG_NO_COMPUTE 0      // 1 = consumers release stages without reading them (bandwidth probe)
#endif
#ifndef MS_ANCHORS
#define MS_ANCHORS 1
#endif
#ifndef MS_ANCHOR_FP32
#define MS_ANCHOR_FP32 1          // 1: anchors cached as fp32 (2x registers, no per-pair unpack)
#endif
#ifndef MS_PIPE
#define MS_PIPE 1                 // 1: software-pipelined single-target Euclidean consumers
#endif
#ifndef MS_ST_MAXKRE
#define MS_ST_MAXKRE 10           // largest single-target stage, in 4 KiB units (10 = 40 KiB)
#endif
#ifndef MS_SUB_UNPACK
#define MS_SUB_UNPACK 0           // 1: t - s via ALU unpack + FFMA2 instead of FHFMA.BF16
#endif
constexpr int kConsumerWarps = MS_CONSUMER_WARPS;
static_assert(kConsumerWarps % 4 == 0, "partials are read as float4");
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;
constexpr int kStageBytes = MS_STAGE_BYTES;
constexpr int kStages = MS_STAGES;
constexpr int kR = kStageBytes / 16 / kConsumers;   // uint4 chunks per consumer thread per stage
static_assert(kR * 16 * kConsumers == kStageBytes, "stage must split evenly over consumers");
constexpr int kAnchors = MS_ANCHORS;                // targets (anchors) per item
static_assert(kAnchors >= 1 && kAnchors <= 4, "anchor registers are unrolled for <= 4");
constexpr int kItemPairs = 64;                      // pairs per item
constexpr int kMetaEnt = 4;                         // pairs evaluated against one stage
constexpr int kPlanThreads = 1024;

constexpr int F_STOP = 1;
constexpr int H_STOP = 1, H_ANCHOR = 2, H_PAIR = 4;

// the single-target consumer's view of a stage (one 16-byte shared load)
__device__ __forceinline__ int4 make_hdr(int64_t out, int32_t bytes, int32_t code) {
  return make_int4((int32_t)(uint32_t)(uint64_t)out, (int32_t)((uint64_t)out >> 32), bytes, code);
}

// One work item: <= kAnchors targets of one pair-graph component, with the pair range of each.
struct ItemRec {
  int32_t na;
  int32_t tgt[kAnchors];
  int32_t lo[kAnchors];
  int32_t hi[kAnchors];
};

// One ring stage: which slice it holds and which pairs to evaluate against it.
struct Meta {
  int4 hdr;                // consumer header: {out lo, out hi, bytes, code} (code: bit0 stop, bit1 anchor, bit2 pair)
  int32_t pair[kMetaEnt];
  int8_t anc[kMetaEnt];    // anchor slot holding the other operand of pair[e]
  int32_t nent;
  int32_t anchor;          // >= 0: this slice becomes anchor slot `anchor`
  int32_t layer, kv, sub, bytes, flags;
};

struct DistWs {
  unsigned int* ticket;
  int64_t* n_items;
  ItemRec* items;        // [item_cap]
  int32_t* cnt;          // [target_cap] items starting at each sorted position
  int64_t* item_off;     // [target_cap + 1]
  float* wpart;          // [pair_cap][N][2][n_sub][kConsumerWarps]  squared sums (Euclidean) / dot (cosine)
  float* wsn;            // cosine only: [pair_cap][N][2][n_sub][W] source squared norms
  float* wtn;            // cosine only: [target_cap][N][2][n_sub][W] target squared norms
};

int64_t item_cap_of(int64_t pair_cap, int64_t target_cap) { return target_cap + pair_cap / kItemPairs + 2; }

DistWs dist_layout(Ws& w, int32_t N, int32_t n_sub, int32_t num_blocks, int64_t pair_cap, int64_t target_cap,
                   int32_t metric) {
  (void)num_blocks;
  DistWs d;
  d.ticket = w.take<unsigned int>(1);
  d.n_items = w.take<int64_t>(1);
  d.items = w.take<ItemRec>(item_cap_of(pair_cap, target_cap));
  d.cnt = w.take<int32_t>(target_cap + 1);
  d.item_off = w.take<int64_t>(target_cap + 2);
  const size_t per = (size_t)N * 2 * n_sub * kConsumerWarps;
  d.wpart = w.take<float>((size_t)pair_cap * per + 1);
  const bool cosine = metric == MEMSHARE_METRIC_COSINE;
  d.wsn = w.take<float>(cosine ? (size_t)pair_cap * per + 1 : 1);
  d.wtn = w.take<float>(cosine ? (size_t)target_cap * per + 1 : 1);
  return d;
}

struct DistArgs {
  const uint8_t* kbase;
  const uint8_t* vbase;
  int64_t layer_stride_b;
  int64_t block_stride_b;
  int32_t num_blocks;
  int32_t N, d, h_global;
  int32_t slice_bytes, n_sub, sub_bytes;
  int32_t lpi, n_chunks;
  int32_t plan_sort_cap;     // targets the planner can sort in its shared memory
  const memshare_block_pair* pairs;
  const int64_t* target_off;
  const int64_t* num_pairs;
  const int64_t* num_targets;
  int64_t pair_cap, target_cap;
  int32_t mode;
  int32_t metric;        // MEMSHARE_METRIC_EUCLIDEAN | MEMSHARE_METRIC_COSINE
  float* partial_sq;
  const float* const* peers;  // FINALIZE over peer memory: every rank's partial_sq, rank order
  int32_t num_peers;
  float tau_b;
  float* distance;
  uint8_t* under;
  memshare_decision* decisions;
  int32_t* status;
  DistWs ws;
};

constexpr int kMaxTemplates = 2 * kAnchors + 2 * kItemPairs;

struct StageTpl {             // one stage of an item, the same for every (layer, K|V, sub-slice)
  int32_t phys;
  int32_t anchor;
  int32_t nent;
  int32_t pair[kMetaEnt];
  int8_t anc[kMetaEnt];
};

struct ProdSmem {               // producer-private staging of one item
  int32_t ent_pair[kItemPairs];
  int32_t ent_phys[kItemPairs];
  int8_t ent_anc[kItemPairs];
  int8_t ent_kind[kItemPairs];   // -1: streamed (first of its phys); -2: streamed duplicate; >= 0: anchor
  int32_t aphys[kAnchors];
  StageTpl tpl[kMaxTemplates];
  int32_t ntpl;
};

struct DistSmem {
  alignas(128) uint8_t ring[kStages][kStageBytes];
  alignas(8) uint64_t full[kStages];
  uint64_t empty[kStages];
  Meta meta[kStages];
  ProdSmem prod;
};

// ------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float2 bf2_to_f2(uint32_t x) {
  return make_float2(__uint_as_float(x << 16), __uint_as_float(x & 0xFFFF0000u));
}

__device__ __forceinline__ int64_t clamp_count(const int64_t* p, int64_t cap) {
  const int64_t v = __ldcg(p);
  return v < 0 ? 0 : (v < cap ? v : cap);
}

// fixed-order fp32 sum of the per-warp partials of (row, layer l, kv) of one workspace buffer
__device__ __forceinline__ float sum_warps(const DistArgs& a, const float* buf, int64_t row, int32_t l, int32_t kv) {
  const float4* w = reinterpret_cast<const float4*>(buf + (((row * a.N + l) * 2 + kv) * a.n_sub) * kConsumerWarps);
  float s = 0.f;
  for (int sub = 0; sub < a.n_sub; ++sub) {
    float4 v[kConsumerWarps / 4];
#pragma unroll
    for (int j = 0; j < kConsumerWarps / 4; ++j) v[j] = __ldcg(w + sub * (kConsumerWarps / 4) + j);
#pragma unroll
    for (int j = 0; j < kConsumerWarps / 4; ++j) s = (((s + v[j].x) + v[j].y) + v[j].z) + v[j].w;
  }
  return s;
}

__device__ __forceinline__ float sum_part(const DistArgs& a, int64_t p, int32_t l, int32_t kv, bool from_partial) {
  if (from_partial) {
    const int64_t o = (p * a.N + l) * 2 + kv;
    if (a.num_peers == 0) return __ldcg(a.partial_sq + o);
    // the cross-rank reduction fused into finalisation: one load per rank over NVLink (peer
    // mappings of the ranks' partial_sq), summed in rank order -> identical on every rank
    float s = __ldcv(a.peers[0] + o);
    for (int r = 1; r < a.num_peers; ++r) s += __ldcv(a.peers[r] + o);
    return s;
  }
  return sum_warps(a, a.ws.wpart, p, l, kv);
}

// cosine of one (pair, layer, K|V) from fp32 dot and squared norms, in fp64 (f2 metric, reading R34)
__device__ __forceinline__ double cos_of(float dot, float tn, float sn) {
  if (tn == 0.f && sn == 0.f) return 1.0;               // two zero slices are identical
  if (tn == 0.f || sn == 0.f) return 0.0;
  return (double)dot / __dsqrt_rn((double)tn * (double)sn);
}

// Finalise target t with the kConsumers threads (tid in [0, kConsumers)); `sync` is the barrier
// among exactly those threads.
template <class Sync>
__device__ void finalize_target(const DistArgs& a, int64_t t, double* terms, int tid, bool from_partial, Sync sync) {
  const int64_t P = clamp_count(a.num_pairs, a.pair_cap);
  const int64_t p0 = __ldcg(a.target_off + t);
  int64_t p1 = __ldcg(a.target_off + t + 1);
  if (p1 > P) p1 = P;
  const int N = a.N;
  const int ppc = kConsumers / N;                       // whole pairs per chunk
  const double inv = 1.0 / (2.0 * (double)a.d * (double)a.h_global);
  const int lane = tid & 31, w = tid >> 5;
  for (int64_t pc = p0; pc < p1; pc += ppc) {
    const int64_t p = pc + tid / N;
    const int32_t l = tid % N;
    if (tid < ppc * N && p < p1) {
      if (a.metric == MEMSHARE_METRIC_COSINE) {
        // f2: PAPER.md:271-273 cosine block similarity, averaged over K|V and layers
        const double ck = cos_of(sum_part(a, p, l, 0, false), sum_warps(a, a.ws.wtn, t, l, 0), sum_warps(a, a.ws.wsn, p, l, 0));
        const double cv = cos_of(sum_part(a, p, l, 1, false), sum_warps(a, a.ws.wtn, t, l, 1), sum_warps(a, a.ws.wsn, p, l, 1));
        terms[tid] = 0.5 * (ck + cv);
      } else {
        const float sk = sum_part(a, p, l, 0, from_partial);
        const float sv = sum_part(a, p, l, 1, from_partial);
        if (!from_partial && a.partial_sq != nullptr) {
          a.partial_sq[(p * N + l) * 2 + 0] = sk;
          a.partial_sq[(p * N + l) * 2 + 1] = sv;
        }
        // Alg. 1 line 5: (Delta_K + Delta_V) / (2dh)
        terms[tid] = (__dsqrt_rn((double)sk) + __dsqrt_rn((double)sv)) * inv;
      }
    }
    sync();
    if (a.mode != MEMSHARE_DIST_PARTIAL) {
      for (int q = w; q < ppc; q += kConsumerWarps) {
        const int64_t pp = pc + q;
        if (pp >= p1) break;
        double acc = 0.0;
        for (int l2 = lane; l2 < N; l2 += 32) acc += terms[q * N + l2];
        acc = warp_sum(acc);
        if (lane == 0) {
          // Alg. 1 line 7: return D / N  (cosine metric: D = 1 - mean similarity)
          const float D = (float)(a.metric == MEMSHARE_METRIC_COSINE ? 1.0 - acc / (double)N : acc / (double)N);
          a.distance[pp] = D;
          a.under[pp] = D < a.tau_b ? 1 : 0;
        }
      }
    }
    sync();
  }
  if (a.mode == MEMSHARE_DIST_PARTIAL) return;
  if (tid == 0) {
    __threadfence_block();
    memshare_decision dc;
    dc.num_candidates = (int32_t)(p1 > p0 ? p1 - p0 : 0);
    if (p1 <= p0) {
      dc.seq = -1; dc.target_logical = -1; dc.target_phys = -1; dc.source_logical = -1; dc.source_phys = -1;
      dc.accepted = 0; dc.distance = INFINITY;
    } else {
      int64_t b = p0;
      float bd = a.distance[p0];
      int32_t bl = a.pairs[p0].source_logical;
      for (int64_t p = p0 + 1; p < p1; ++p) {
        const float dp = a.distance[p];
        const int32_t lp = a.pairs[p].source_logical;
        if (dp < bd || (dp == bd && lp < bl)) { b = p; bd = dp; bl = lp; }
      }
      const memshare_block_pair pr = a.pairs[b];
      dc.seq = pr.seq; dc.target_logical = pr.target_logical; dc.target_phys = pr.target_phys;
      dc.source_logical = pr.source_logical; dc.source_phys = pr.source_phys;
      dc.distance = bd;
      dc.accepted = bd < a.tau_b ? 1 : 0;              // strict (reading R21)
    }
    if (t < a.target_cap) a.decisions[t] = dc;
  }
}


__device__ __forceinline__ int32_t checked_phys(const DistArgs& a, int32_t p) {
  if (p < 0 || p >= a.num_blocks) {
    set_status(a.status, MEMSHARE_ERR_CORRUPTION);
    return 0;
  }
  return p;
}

// ------------------------------------------------------------------------------ planning
// Items: targets that share their first (smallest-logical) source block are near-copies of one
// earlier step at the same block offset (redundant steps repeat an earlier
// one), so they share most of their sources. Targets are sorted by (first source, index) in
// shared memory; each run of <= kAnchors consecutive targets with the same key whose pairs fit
// in kItemPairs becomes one item, otherwise each target becomes its own item(s) of <= 64 pairs.
// Larger inputs (T > kPlanSortCap) use one-target items. One CTA, fully parallel, deterministic.
constexpr int kPlanSortCap = 8192;

__device__ __forceinline__ int64_t pair_lo(const DistArgs& a, int64_t t) { return __ldcg(a.target_off + t); }

__device__ __forceinline__ int64_t pairs_of(const DistArgs& a, int64_t t, int64_t P) {
  const int64_t lo = __ldcg(a.target_off + t);
  int64_t hi = __ldcg(a.target_off + t + 1);
  if (hi > P) hi = P;
  return hi > lo ? hi - lo : 0;
}

__device__ __forceinline__ int32_t solo_items(int64_t np) { return (int32_t)((np + kItemPairs - 1) / kItemPairs); }

__device__ void write_solo(const DistArgs& a, int64_t t, int64_t P, int64_t at) {
  const int64_t lo = pair_lo(a, t);
  const int64_t hi = lo + pairs_of(a, t, P);
  for (int64_t c0 = lo; c0 < hi; c0 += kItemPairs, ++at) {
    ItemRec r;
    r.na = 1; r.tgt[0] = (int32_t)t; r.lo[0] = (int32_t)c0;
    r.hi[0] = (int32_t)(c0 + kItemPairs < hi ? c0 + kItemPairs : hi);
    a.ws.items[at] = r;
  }
}

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(DistArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ unsigned long long keys[];           // [pow2(T)] when T <= kPlanSortCap
  __shared__ int64_t sh[kPlanThreads / 32 + 1];
  const int tid = threadIdx.x;
  const int64_t T = clamp_count(a.num_targets, a.target_cap);
  const int64_t P = clamp_count(a.num_pairs, a.pair_cap);
  if (T > a.plan_sort_cap) {                               // one-target items
    for (int64_t t = tid; t < T; t += kPlanThreads) a.ws.cnt[t] = solo_items(pairs_of(a, t, P));
    __syncthreads();
    cta_scan_counts<kPlanThreads>(a.ws.cnt, a.ws.item_off, T, sh);
    __syncthreads();
    for (int64_t t = tid; t < T; t += kPlanThreads) write_solo(a, t, P, __ldcg(a.ws.item_off + t));
    if (tid == 0) *a.ws.n_items = __ldcg(a.ws.item_off + T);
    return;
  }
  int np2 = 1;
  while (np2 < T) np2 <<= 1;
  for (int q = tid; q < np2; q += kPlanThreads) {
    unsigned long long k = ~0ull;
    if (q < T) {
      const int64_t n = pairs_of(a, q, P);
      const uint32_t first = n > 0 ? (uint32_t)checked_phys(a, a.pairs[pair_lo(a, q)].source_phys) : 0xFFFFFFFFu;
      k = ((unsigned long long)first << 32) | (uint32_t)q;
    }
    keys[q] = k;
  }
  __syncthreads();
  for (int k = 2; k <= np2; k <<= 1)                      // bitonic sort, ascending
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < np2; i += kPlanThreads) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long x = keys[i], y = keys[ixj];
          if (((i & k) == 0) ? (x > y) : (x < y)) { keys[i] = y; keys[ixj] = x; }
        }
      }
      __syncthreads();
    }
  // run starts: position q whose rank within its key group is a multiple of kAnchors
  for (int q = tid; q < T; q += kPlanThreads) {
    const unsigned long long kq = keys[q] >> 32;
    int lo = 0, hi = q;                                    // first position with the same key
    while (lo < hi) { const int mid = (lo + hi) >> 1; if ((keys[mid] >> 32) < kq) lo = mid + 1; else hi = mid; }
    const int gstart = lo;
    int32_t items = 0;
    if ((q - gstart) % kAnchors == 0 && kq != 0xFFFFFFFFull) {
      int glen = 1;
      while (glen < kAnchors && q + glen < T && (keys[q + glen] >> 32) == kq) ++glen;
      int64_t sum = 0;
      for (int m = 0; m < glen; ++m) sum += pairs_of(a, (int64_t)(keys[q + m] & 0xFFFFFFFFu), P);
      if (sum <= kItemPairs) items = 1;
      else for (int m = 0; m < glen; ++m) items += solo_items(pairs_of(a, (int64_t)(keys[q + m] & 0xFFFFFFFFu), P));
    }
    a.ws.cnt[q] = items;
  }
  __syncthreads();
  cta_scan_counts<kPlanThreads>(a.ws.cnt, a.ws.item_off, T, sh);
  __syncthreads();
  for (int q = tid; q < T; q += kPlanThreads) {
    if (__ldcg(a.ws.cnt + q) == 0) continue;
    const unsigned long long kq = keys[q] >> 32;
    int glen = 1;
    while (glen < kAnchors && q + glen < T && (keys[q + glen] >> 32) == kq) ++glen;
    int64_t at = __ldcg(a.ws.item_off + q);
    int64_t sum = 0;
    for (int m = 0; m < glen; ++m) sum += pairs_of(a, (int64_t)(keys[q + m] & 0xFFFFFFFFu), P);
    if (sum <= kItemPairs) {
      ItemRec r;
      r.na = glen;
      for (int m = 0; m < glen; ++m) {
        const int64_t t = (int64_t)(keys[q + m] & 0xFFFFFFFFu);
        r.tgt[m] = (int32_t)t; r.lo[m] = (int32_t)pair_lo(a, t); r.hi[m] = (int32_t)(pair_lo(a, t) + pairs_of(a, t, P));
      }
      a.ws.items[at] = r;
    } else {
      for (int m = 0; m < glen; ++m) {
        const int64_t t = (int64_t)(keys[q + m] & 0xFFFFFFFFu);
        write_solo(a, t, P, at);
        at += solo_items(pairs_of(a, t, P));
      }
    }
  }
  __syncthreads();
  if (tid == 0) *a.ws.n_items = __ldcg(a.ws.item_off + T);
}

// ------------------------------------------------------------------------------ streaming
#if MS_ANCHOR_FP32
using AnchorT = float2[kR * 4];
#else
using AnchorT = uint4[kR];
#endif

// d = t - s in ONE mixed-precision FMA straight from the packed bf16 source (SASS FHFMA.BF16 with
// .H0/.H1 half selection, sm_100): fma(s, -1, t) = RN(t - s) exactly as before, no unpack.
__device__ __forceinline__ float2 sub_bf2(uint32_t x, float2 t) {
  float2 d;
  asm("{\n.reg .b16 lo, hi;\nmov.b32 {lo, hi}, %2;\n"
      "fma.rn.f32.bf16 %0, lo, %5, %3;\nfma.rn.f32.bf16 %1, hi, %5, %4;\n}\n"
      : "=f"(d.x), "=f"(d.y)
      : "r"(x), "f"(t.x), "f"(t.y), "h"((unsigned short)0xBF80u));
  return d;
}

template <int K>
__device__ __forceinline__ float dist2_anchor(const AnchorT (&A)[kAnchors], const uint4 (&x)[kR]) {
  float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#if !MS_ANCHOR_FP32
  const float2 neg1 = make_float2(-1.f, -1.f);
#endif
#pragma unroll
  for (int r = 0; r < kR; ++r) {
#if MS_ANCHOR_FP32
    const float2 d0 = sub_bf2(x[r].x, A[K][4 * r + 0]);
    const float2 d1 = sub_bf2(x[r].y, A[K][4 * r + 1]);
    const float2 d2 = sub_bf2(x[r].z, A[K][4 * r + 2]);
    const float2 d3 = sub_bf2(x[r].w, A[K][4 * r + 3]);
#else
    const float2 t0 = bf2_to_f2(A[K][r].x), t1 = bf2_to_f2(A[K][r].y), t2 = bf2_to_f2(A[K][r].z),
                 t3 = bf2_to_f2(A[K][r].w);
    const float2 d0 = __ffma2_rn(bf2_to_f2(x[r].x), neg1, t0);
    const float2 d1 = __ffma2_rn(bf2_to_f2(x[r].y), neg1, t1);
    const float2 d2 = __ffma2_rn(bf2_to_f2(x[r].z), neg1, t2);
    const float2 d3 = __ffma2_rn(bf2_to_f2(x[r].w), neg1, t3);
#endif
    acc0 = __ffma2_rn(d0, d0, acc0);                     // acc += d*d, packed (FFMA2)
    acc1 = __ffma2_rn(d1, d1, acc1);
    acc0 = __ffma2_rn(d2, d2, acc0);
    acc1 = __ffma2_rn(d3, d3, acc1);
  }
  return (acc0.x + acc0.y) + (acc1.x + acc1.y);
}

#if MS_SUB_UNPACK
// d = t - s with s unpacked on the ALU pipe (SHF / LOP3) and one packed FFMA2 on the FMA pipe:
// moves half of the per-element work off the FMA pipe (variant MS_SUB_UNPACK).
__device__ __forceinline__ float2 sub_bf2_unpack(uint32_t x, float2 t) {
  const float2 s = bf2_to_f2(x);
  return __ffma2_rn(s, make_float2(-1.f, -1.f), t);
}
#endif

__device__ __forceinline__ float dist2_regs(const float2 (&T)[kR * 4], const uint4 (&x)[kR]) {
  float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
  for (int r = 0; r < kR; ++r) {
#if MS_SUB_UNPACK
    const float2 d0 = sub_bf2_unpack(x[r].x, T[4 * r + 0]);
    const float2 d1 = sub_bf2_unpack(x[r].y, T[4 * r + 1]);
    const float2 d2 = sub_bf2_unpack(x[r].z, T[4 * r + 2]);
    const float2 d3 = sub_bf2_unpack(x[r].w, T[4 * r + 3]);
#else
    const float2 d0 = sub_bf2(x[r].x, T[4 * r + 0]);
    const float2 d1 = sub_bf2(x[r].y, T[4 * r + 1]);
    const float2 d2 = sub_bf2(x[r].z, T[4 * r + 2]);
    const float2 d3 = sub_bf2(x[r].w, T[4 * r + 3]);
#endif
    acc0 = __ffma2_rn(d0, d0, acc0);
    acc1 = __ffma2_rn(d1, d1, acc1);
    acc0 = __ffma2_rn(d2, d2, acc0);
    acc1 = __ffma2_rn(d3, d3, acc1);
  }
  return (acc0.x + acc0.y) + (acc1.x + acc1.y);
}

// Consumer loop of the single-target Euclidean kernel (the shipped configuration), software
// pipelined with two register buffers (ping-pong, no register copies): the next stage is loaded
// into one buffer while the other is evaluated, so the shared-memory loads overlap the FMA work.
// Each stage is described by a 16-byte header the producer precomputes (output offset, bytes,
// anchor / pair / stop), so the consumer does no index arithmetic.
struct StageView {
  int64_t out;
  int32_t bytes, code;
};

__device__ __forceinline__ StageView view_of(const DistSmem& sm, int st) {
  const int4 h = *reinterpret_cast<const int4*>(&sm.meta[st].hdr);
  StageView v;
  v.out = (int64_t)(((uint64_t)(uint32_t)h.y << 32) | (uint32_t)h.x);
  v.bytes = h.z;
  v.code = h.w;
  return v;
}

__device__ __forceinline__ void load_stage(const DistSmem& sm, int st, int tid, int bytes, uint4 (&dst)[kR]) {
  const uint4* src = reinterpret_cast<const uint4*>(sm.ring[st]);
  if (bytes == kStageBytes) {                       // full stage: no predicates
#pragma unroll
    for (int r = 0; r < kR; ++r) dst[r] = src[tid + r * kConsumers];
  } else {
    const int nchunk = bytes >> 4;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int c = tid + r * kConsumers;
      dst[r] = c < nchunk ? src[c] : make_uint4(0u, 0u, 0u, 0u);
    }
  }
}

__device__ __forceinline__ void eval_stage(const DistArgs& a, const StageView& v, const uint4 (&x)[kR],
                                           float2 (&T)[kR * 4], int warp, int lane) {
  if (v.code & H_ANCHOR) {
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      T[4 * r + 0] = bf2_to_f2(x[r].x);
      T[4 * r + 1] = bf2_to_f2(x[r].y);
      T[4 * r + 2] = bf2_to_f2(x[r].z);
      T[4 * r + 3] = bf2_to_f2(x[r].w);
    }
  } else if (v.code & H_PAIR) {
    const float s = warp_sum(dist2_regs(T, x));
    if (lane == 0) a.ws.wpart[v.out + warp] = s;
  }
}

__device__ __forceinline__ void consume_euclid(DistSmem& sm, const DistArgs& a, int tid, int warp, int lane) {
  float2 T[kR * 4];
  uint4 xa[kR], xb[kR];
  int stage = 0;
  uint32_t ph = 0;
  auto advance = [&]() { if (++stage == kStages) { stage = 0; ph ^= 1u; } };
  auto release = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[stage]);
    advance();
  };
  mbar_wait(&sm.full[stage], ph);
  StageView va = view_of(sm, stage), vb;
  if (va.code & H_STOP) return;
  load_stage(sm, stage, tid, va.bytes, xa);
  release();
  for (;;) {
    mbar_wait(&sm.full[stage], ph);
    vb = view_of(sm, stage);
    if (!(vb.code & H_STOP)) load_stage(sm, stage, tid, vb.bytes, xb);
    eval_stage(a, va, xa, T, warp, lane);            // overlaps the loads of xb
    if (vb.code & H_STOP) break;
    release();
    mbar_wait(&sm.full[stage], ph);
    va = view_of(sm, stage);
    if (!(va.code & H_STOP)) load_stage(sm, stage, tid, va.bytes, xa);
    eval_stage(a, vb, xb, T, warp, lane);
    if (va.code & H_STOP) break;
    release();
  }
}

template <int kMetric>
__global__ void __launch_bounds__(kThreads, 1) distance_kernel(DistArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  DistSmem& sm = *reinterpret_cast<DistSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();                       // setup above overlaps the predecessor's tail

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------------ producer warp
    // with one anchor an item is a target (no planning launch); otherwise plan_kernel's items
    const int64_t I = kAnchors == 1 ? clamp_count(a.num_targets, a.target_cap) : __ldcg(a.ws.n_items);
    const int64_t Pn = clamp_count(a.num_pairs, a.pair_cap);
    const int64_t total = I * a.n_chunks;
    int stage = 0;
    uint32_t ph = 0;
    if (kAnchors == 1) {
      // One target per item. The next unit's metadata (target range, target and source ids) is
      // loaded into registers one unit ahead, so issuing never waits on metadata latency.
      struct UnitMeta { int64_t lc, t; int32_t lo, np, tphys, sp0, sp1; };
      auto load_meta = [&](int64_t u) {
        UnitMeta m{0, 0, 0, 0, 0, 0, 0};
        if (u >= total) return m;
        m.lc = u / I;
        m.t = u - m.lc * I;
        const int64_t lo = __ldcg(a.target_off + m.t);
        int64_t hi = __ldcg(a.target_off + m.t + 1);
        if (hi > Pn) hi = Pn;
        m.lo = (int32_t)lo;
        m.np = (int32_t)(hi > lo ? hi - lo : 0);
        if (m.np > 0) m.tphys = a.pairs[lo].target_phys;
        if (lane < m.np) m.sp0 = a.pairs[lo + lane].source_phys;
        if (lane + 32 < m.np) m.sp1 = a.pairs[lo + 32 + lane].source_phys;
        return m;
      };
      int64_t unit = 0, next = 0;
      if (lane == 0) {
        unit = (int64_t)atomicAdd(a.ws.ticket, 1u);
        next = (int64_t)atomicAdd(a.ws.ticket, 1u);
      }
      unit = __shfl_sync(0xffffffffu, unit, 0);
      next = __shfl_sync(0xffffffffu, next, 0);
      UnitMeta cur = load_meta(unit);
      while (unit < total) {
        int64_t next2 = 0;
        if (lane == 0) next2 = (int64_t)atomicAdd(a.ws.ticket, 1u);
        const UnitMeta nm = load_meta(next);                  // consumed next iteration
        if (cur.np > 0) {
          const int32_t tphys = checked_phys(a, cur.tphys);
          const int32_t l0 = (int32_t)cur.lc * a.lpi;
          const int32_t l1 = (l0 + a.lpi < a.N) ? l0 + a.lpi : a.N;
          for (int32_t c0 = 0; c0 < cur.np; c0 += 64) {       // pairs in chunks of 64 (register-staged)
            const int32_t cn = (cur.np - c0) < 64 ? cur.np - c0 : 64;
            int32_t sa = cur.sp0, sb = cur.sp1;
            if (c0 > 0) {
              sa = (lane < cn) ? a.pairs[cur.lo + c0 + lane].source_phys : 0;
              sb = (lane + 32 < cn) ? a.pairs[cur.lo + c0 + 32 + lane].source_phys : 0;
            }
            for (int32_t l = l0; l < l1; ++l) {
              for (int32_t kv = 0; kv < 2; ++kv) {
                const uint8_t* base = (kv ? a.vbase : a.kbase) + (int64_t)l * a.layer_stride_b;
                for (int32_t sub = 0; sub < a.n_sub; ++sub) {
                  const int32_t boff = sub * a.sub_bytes;
                  const int32_t bytes = (a.slice_bytes - boff) < a.sub_bytes ? (a.slice_bytes - boff) : a.sub_bytes;
                  for (int32_t q = -1; q < cn; ++q) {          // q = -1: the target (anchor 0)
                    const int32_t v = __shfl_sync(0xffffffffu, (q & 32) ? sb : sa, q < 0 ? 0 : (q & 31));
                    if (lane == 0) {
                      const int32_t phys = q < 0 ? tphys : checked_phys(a, v);
                      mbar_wait(&sm.empty[stage], ph ^ 1u);
                      Meta& m = sm.meta[stage];
                      m.anchor = q < 0 ? 0 : -1;
                      m.nent = q < 0 ? 0 : 1;
                      m.pair[0] = q < 0 ? (int32_t)cur.t : cur.lo + c0 + q;   // target slot: target index
                      m.anc[0] = 0;
                      m.layer = l; m.kv = kv; m.sub = sub; m.bytes = bytes; m.flags = 0;
                      const int64_t po = q < 0 ? 0 : (int64_t)(cur.lo + c0 + q);
                      m.hdr = make_hdr((((po * a.N + l) * 2 + kv) * a.n_sub + sub) * kConsumerWarps, bytes,
                                       q < 0 ? H_ANCHOR : H_PAIR);
                      mbar_expect_tx(&sm.full[stage], (uint32_t)bytes);
                      bulk_g2s(sm.ring[stage], base + (int64_t)phys * a.block_stride_b + boff, (uint32_t)bytes,
                               &sm.full[stage]);
                      if (++stage == kStages) { stage = 0; ph ^= 1u; }
                    }
                  }
                }
              }
            }
          }
        }
        __syncwarp();
        unit = next;
        next = __shfl_sync(0xffffffffu, next2, 0);
        cur = nm;
      }
      stage = __shfl_sync(0xffffffffu, stage, 0);
      ph = __shfl_sync(0xffffffffu, ph, 0);
      if (lane == 0) {
        mbar_wait(&sm.empty[stage], ph ^ 1u);
        sm.meta[stage].flags = F_STOP;
        sm.meta[stage].hdr = make_hdr(0, 0, H_STOP);
        sm.meta[stage].nent = 0;
        sm.meta[stage].anchor = -1;
        mbar_arrive(&sm.full[stage]);
      }
      return;
    }
    ProdSmem& ps = sm.prod;
    int64_t unit = 0;
    if (lane == 0) unit = (int64_t)atomicAdd(a.ws.ticket, 1u);
    unit = __shfl_sync(0xffffffffu, unit, 0);
    while (unit < total) {
      int64_t next = 0;
      if (lane == 0) next = (int64_t)atomicAdd(a.ws.ticket, 1u);   // consumed at the end of the unit
      const int64_t lc = unit / I, it = unit - lc * I;
      ItemRec rec0;
      if (kAnchors == 1) {
        rec0.na = 1; rec0.tgt[0] = (int32_t)it;
        const int64_t lo = __ldcg(a.target_off + it);
        int64_t hi = __ldcg(a.target_off + it + 1);
        if (hi > Pn) hi = Pn;
        rec0.lo[0] = (int32_t)lo; rec0.hi[0] = (int32_t)(hi > lo ? hi : lo);
      } else {
        rec0 = a.ws.items[it];
      }
      // a target with more than kItemPairs pairs is processed in chunks (anchor reloaded per chunk)
      for (int32_t c0 = rec0.lo[0]; c0 < rec0.hi[0] || (c0 == rec0.lo[0] && rec0.na > 1); c0 += kItemPairs) {
      ItemRec rec = rec0;
      if (rec0.na == 1) { rec.lo[0] = c0; rec.hi[0] = (c0 + kItemPairs < rec0.hi[0]) ? c0 + kItemPairs : rec0.hi[0]; }
      // stage the item's pairs: entry e -> (anchor, pair, source phys)
      int32_t off[kAnchors + 1];
      off[0] = 0;
#pragma unroll
      for (int i = 0; i < kAnchors; ++i) off[i + 1] = off[i] + (i < rec.na ? rec.hi[i] - rec.lo[i] : 0);
      const int32_t ne = off[kAnchors];
      if (lane < rec.na) ps.aphys[lane] = checked_phys(a, a.pairs[rec.lo[lane]].target_phys);
      for (int32_t e = lane; e < ne; e += 32) {
        int i = 0;
        while (i + 1 < rec.na && e >= off[i + 1]) ++i;
        const int32_t p = rec.lo[i] + (e - off[i]);
        ps.ent_pair[e] = p;
        ps.ent_anc[e] = (int8_t)i;
        ps.ent_phys[e] = checked_phys(a, a.pairs[p].source_phys);
      }
      __syncwarp();
      // classify: source is an anchor block -> evaluated at the later anchor's stage;
      // otherwise streamed once per distinct physical block (first occurrence streams).
      for (int32_t e = lane; e < ne; e += 32) {
        const int32_t ph_e = ps.ent_phys[e];
        int kind = -1;
        for (int j = 0; j < rec.na; ++j)
          if (ps.aphys[j] == ph_e) { kind = j; break; }
        if (kind < 0) {
          for (int32_t e2 = 0; e2 < e; ++e2)
            if (ps.ent_phys[e2] == ph_e) {
              bool e2_anchor = false;
              for (int j = 0; j < rec.na; ++j) e2_anchor |= (ps.aphys[j] == ph_e);
              if (!e2_anchor) { kind = -2; break; }
            }
        }
        ps.ent_kind[e] = (int8_t)kind;
      }
      __syncwarp();
      if (lane == 0) {
        // stage templates, built once per unit: anchors first (each carrying the anchor-anchor
        // pairs completed by its arrival), then one stage per distinct streamed source
        int32_t nt = 0;
        auto open_tpl = [&](int32_t phys, int32_t anchor) {
          StageTpl& t = ps.tpl[nt++];
          t.phys = phys; t.anchor = anchor; t.nent = 0;
          return &t;
        };
        for (int j = 0; j < rec.na; ++j) {
          StageTpl* t = open_tpl(ps.aphys[j], j);
          for (int32_t e = 0; e < ne; ++e) {
            const int k = ps.ent_kind[e];
            if (k < 0) continue;
            const int i = ps.ent_anc[e];
            if ((i > k ? i : k) != j) continue;
            if (t->nent == kMetaEnt) t = open_tpl(ps.aphys[j], j);   // overflow: reload the anchor
            t->pair[t->nent] = ps.ent_pair[e];
            t->anc[t->nent] = (int8_t)(i > k ? k : i);
            t->nent += 1;
          }
        }
        for (int32_t e = 0; e < ne; ++e) {
          if (ps.ent_kind[e] != -1) continue;
          const int32_t phe = ps.ent_phys[e];
          StageTpl* t = open_tpl(phe, -1);
          for (int32_t e2 = e; e2 < ne; ++e2) {
            if (ps.ent_kind[e2] >= 0 || ps.ent_phys[e2] != phe) continue;
            if (t->nent == kMetaEnt) t = open_tpl(phe, -1);
            t->pair[t->nent] = ps.ent_pair[e2];
            t->anc[t->nent] = ps.ent_anc[e2];
            t->nent += 1;
          }
        }
        const int32_t l0 = (int32_t)lc * a.lpi;
        const int32_t l1 = (l0 + a.lpi < a.N) ? l0 + a.lpi : a.N;
        for (int32_t l = l0; l < l1; ++l) {
          for (int32_t kv = 0; kv < 2; ++kv) {
            const uint8_t* base = (kv ? a.vbase : a.kbase) + (int64_t)l * a.layer_stride_b;
            for (int32_t sub = 0; sub < a.n_sub; ++sub) {
              const int32_t boff = sub * a.sub_bytes;
              const int32_t bytes = (a.slice_bytes - boff) < a.sub_bytes ? (a.slice_bytes - boff) : a.sub_bytes;
              for (int32_t ti = 0; ti < nt; ++ti) {
                const StageTpl& t = ps.tpl[ti];
                mbar_wait(&sm.empty[stage], ph ^ 1u);
                Meta& m = sm.meta[stage];
#pragma unroll
                for (int e = 0; e < kMetaEnt; ++e) { m.pair[e] = t.pair[e]; m.anc[e] = t.anc[e]; }
                m.nent = t.nent; m.anchor = t.anchor;
                m.layer = l; m.kv = kv; m.sub = sub; m.bytes = bytes; m.flags = 0;
                m.hdr = make_hdr(0, bytes, 0);    // the multi-anchor path uses the generic consumer
                mbar_expect_tx(&sm.full[stage], (uint32_t)bytes);
                bulk_g2s(sm.ring[stage], base + (int64_t)t.phys * a.block_stride_b + boff, (uint32_t)bytes,
                         &sm.full[stage]);
                if (++stage == kStages) { stage = 0; ph ^= 1u; }
              }
            }
          }
        }
      }
      __syncwarp();
      if (rec0.na > 1) break;
      }
      __syncwarp();
      unit = __shfl_sync(0xffffffffu, next, 0);
    }
    if (lane == 0) {
      mbar_wait(&sm.empty[stage], ph ^ 1u);
      sm.meta[stage].flags = F_STOP;
      sm.meta[stage].hdr = make_hdr(0, 0, H_STOP);
      sm.meta[stage].nent = 0;
      sm.meta[stage].anchor = -1;
      mbar_arrive(&sm.full[stage]);
    }
    return;
  }

  // -------------------------------------------------------------------- consumer warps
#if MS_PIPE && MS_ANCHOR_FP32 && !MS_DIAG_NO_COMPUTE
  if (kMetric == MEMSHARE_METRIC_EUCLIDEAN && kAnchors == 1) {
    consume_euclid(sm, a, tid, warp, lane);
    return;
  }
#endif
  AnchorT A[kAnchors];
  int stage = 0;
  uint32_t ph = 0;
  for (;;) {
    mbar_wait(&sm.full[stage], ph);
    const Meta& mr = sm.meta[stage];
    const int flags = mr.flags;
    if (flags & F_STOP) break;
    const int anchor = mr.anchor, nent = mr.nent, layer = mr.layer, kv = mr.kv, sub = mr.sub;
    uint32_t ent[kMetaEnt];                                  // pair id << 2 | anchor slot
#pragma unroll
    for (int e = 0; e < kMetaEnt; ++e) ent[e] = ((uint32_t)mr.pair[e] << 2) | ((uint32_t)mr.anc[e] & 3u);
    const int nchunk = mr.bytes >> 4;
    const uint4* src = reinterpret_cast<const uint4*>(sm.ring[stage]);
    uint4 x[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int c = tid + r * kConsumers;
      x[r] = (!MS_DIAG_NO_COMPUTE && c < nchunk) ? src[c] : make_uint4(0u, 0u, 0u, 0u);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[stage]);            // stage free: data is in registers
    if (++stage == kStages) { stage = 0; ph ^= 1u; }
    if (MS_DIAG_NO_COMPUTE) continue;
    if (kMetric == MEMSHARE_METRIC_COSINE) {
      // f2 (kAnchors == 1): target slot -> cache + squared norm; source slot -> dot + squared norm
      float2 n0 = make_float2(0.f, 0.f), n1 = make_float2(0.f, 0.f);
      if (anchor >= 0) {
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const float2 f0 = bf2_to_f2(x[r].x), f1 = bf2_to_f2(x[r].y), f2 = bf2_to_f2(x[r].z), f3 = bf2_to_f2(x[r].w);
          A[0][4 * r + 0] = f0; A[0][4 * r + 1] = f1; A[0][4 * r + 2] = f2; A[0][4 * r + 3] = f3;
          n0 = __ffma2_rn(f0, f0, n0); n1 = __ffma2_rn(f1, f1, n1);
          n0 = __ffma2_rn(f2, f2, n0); n1 = __ffma2_rn(f3, f3, n1);
        }
        float tn = warp_sum((n0.x + n0.y) + (n1.x + n1.y));
        if (lane == 0)
          a.ws.wtn[((((int64_t)(ent[0] >> 2) * a.N + layer) * 2 + kv) * a.n_sub + sub) * kConsumerWarps + warp] = tn;
      } else if (nent > 0) {
        float2 d0 = make_float2(0.f, 0.f), d1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const float2 f0 = bf2_to_f2(x[r].x), f1 = bf2_to_f2(x[r].y), f2 = bf2_to_f2(x[r].z), f3 = bf2_to_f2(x[r].w);
          d0 = __ffma2_rn(A[0][4 * r + 0], f0, d0); d1 = __ffma2_rn(A[0][4 * r + 1], f1, d1);
          d0 = __ffma2_rn(A[0][4 * r + 2], f2, d0); d1 = __ffma2_rn(A[0][4 * r + 3], f3, d1);
          n0 = __ffma2_rn(f0, f0, n0); n1 = __ffma2_rn(f1, f1, n1);
          n0 = __ffma2_rn(f2, f2, n0); n1 = __ffma2_rn(f3, f3, n1);
        }
        const float dot = warp_sum((d0.x + d0.y) + (d1.x + d1.y));
        const float sn = warp_sum((n0.x + n0.y) + (n1.x + n1.y));
        if (lane == 0) {
          const int64_t o = ((((int64_t)(ent[0] >> 2) * a.N + layer) * 2 + kv) * a.n_sub + sub) * kConsumerWarps + warp;
          a.ws.wpart[o] = dot;
          a.ws.wsn[o] = sn;
        }
      }
      continue;
    }
    if (anchor >= 0) {
#pragma unroll
      for (int j = 0; j < kAnchors; ++j)
        if (j == anchor) {
#pragma unroll
          for (int r = 0; r < kR; ++r) {
#if MS_ANCHOR_FP32
            A[j][4 * r + 0] = bf2_to_f2(x[r].x);
            A[j][4 * r + 1] = bf2_to_f2(x[r].y);
            A[j][4 * r + 2] = bf2_to_f2(x[r].z);
            A[j][4 * r + 3] = bf2_to_f2(x[r].w);
#else
            A[j][r] = x[r];
#endif
          }
        }
    }
#pragma unroll
    for (int e = 0; e < kMetaEnt; ++e) {
      if (e >= nent) break;
      float sacc;
      switch (ent[e] & 3u) {                                 // warp-uniform
        case 0: sacc = dist2_anchor<0>(A, x); break;
#if MS_ANCHORS > 1
        case 1: sacc = dist2_anchor<1>(A, x); break;
#endif
#if MS_ANCHORS > 2
        case 2: sacc = dist2_anchor<2>(A, x); break;
#endif
#if MS_ANCHORS > 3
        case 3: sacc = dist2_anchor<3>(A, x); break;
#endif
        default: sacc = 0.f;
      }
      sacc = warp_sum(sacc);
      if (lane == 0)
        a.ws.wpart[((((int64_t)(ent[e] >> 2) * a.N + layer) * 2 + kv) * a.n_sub + sub) * kConsumerWarps + warp] = sacc;
    }
  }
}

// ------------------------------------------------- single-target kernel, stage size per shape
// The shipped Euclidean path. Template parameter KRE = 16-byte chunks per consumer thread per
// stage, so a stage is KRE * 4 KiB and holds one (layer, K|V) slice or an equal part of it
// (32B shape: 32 KiB slices -> KRE 8, one stage per slice; Phi-4: 40 KiB -> two 20 KiB stages,
// KRE 5; tiny: 4 KiB -> KRE 1). The ring keeps the same ~192 KiB of shared memory, so smaller
// stages mean MORE stages in flight: the ring turns over once per TMA round trip, so the stage
// rate, not the byte rate, is what a fixed-size ring of small stages would limit.
constexpr int kChunkUnit = 16 * kConsumers;                 // 4 KiB: one chunk per consumer thread
constexpr int kRingBytes = 224 * 1024;                    // shared-memory ring of the single-target kernel (of 227 KB)
constexpr int kMaxKre = 10;                                // largest stage: 40 KiB (one Phi-4 slice)
constexpr int kMaxRingStages = 48;

template <int KRE>
struct StCfg {
  static constexpr int kStageB = KRE * kChunkUnit;
  static constexpr int kNSt = (kRingBytes / kStageB) < kMaxRingStages ? kRingBytes / kStageB : kMaxRingStages;
};

template <int KRE>
struct StSmem {
  alignas(128) uint8_t ring[StCfg<KRE>::kNSt][StCfg<KRE>::kStageB];
  alignas(16) int4 hdr[StCfg<KRE>::kNSt];
  alignas(8) uint64_t full[StCfg<KRE>::kNSt];
  uint64_t empty[StCfg<KRE>::kNSt];
};

template <int KRE>
__device__ __forceinline__ void st_producer(StSmem<KRE>& sm, const DistArgs& a, int lane) {
  constexpr int NS = StCfg<KRE>::kNSt;
  const int64_t I = clamp_count(a.num_targets, a.target_cap);
  const int64_t Pn = clamp_count(a.num_pairs, a.pair_cap);
  const int64_t total = I * a.n_chunks;
  int stage = 0;
  uint32_t ph = 0;
  // one unit = (target, chunk of lpi layers); the next unit's ids are loaded one unit ahead
  struct UnitMeta { int64_t lc, t; int32_t lo, np, tphys, sp0, sp1; };
  auto load_meta = [&](int64_t u) {
    UnitMeta m{0, 0, 0, 0, 0, 0, 0};
    if (u >= total) return m;
    m.lc = u / I;
    m.t = u - m.lc * I;
    const int64_t lo = __ldcg(a.target_off + m.t);
    int64_t hi = __ldcg(a.target_off + m.t + 1);
    if (hi > Pn) hi = Pn;
    m.lo = (int32_t)lo;
    m.np = (int32_t)(hi > lo ? hi - lo : 0);
    if (m.np > 0) m.tphys = a.pairs[lo].target_phys;
    if (lane < m.np) m.sp0 = a.pairs[lo + lane].source_phys;
    if (lane + 32 < m.np) m.sp1 = a.pairs[lo + 32 + lane].source_phys;
    return m;
  };
  int64_t unit = 0, next = 0;
  if (lane == 0) {
    unit = (int64_t)atomicAdd(a.ws.ticket, 1u);
    next = (int64_t)atomicAdd(a.ws.ticket, 1u);
  }
  unit = __shfl_sync(0xffffffffu, unit, 0);
  next = __shfl_sync(0xffffffffu, next, 0);
  UnitMeta cur = load_meta(unit);
  while (unit < total) {
    int64_t next2 = 0;
    if (lane == 0) next2 = (int64_t)atomicAdd(a.ws.ticket, 1u);
    const UnitMeta nm = load_meta(next);
    if (cur.np > 0) {
      const int32_t tphys = checked_phys(a, cur.tphys);
      const int32_t l0 = (int32_t)cur.lc * a.lpi;
      const int32_t l1 = (l0 + a.lpi < a.N) ? l0 + a.lpi : a.N;
      for (int32_t c0 = 0; c0 < cur.np; c0 += 64) {
        const int32_t cn = (cur.np - c0) < 64 ? cur.np - c0 : 64;
        int32_t sa = cur.sp0, sb = cur.sp1;
        if (c0 > 0) {
          sa = (lane < cn) ? a.pairs[cur.lo + c0 + lane].source_phys : 0;
          sb = (lane + 32 < cn) ? a.pairs[cur.lo + c0 + 32 + lane].source_phys : 0;
        }
        for (int32_t l = l0; l < l1; ++l)
          for (int32_t kv = 0; kv < 2; ++kv) {
            const uint8_t* base = (kv ? a.vbase : a.kbase) + (int64_t)l * a.layer_stride_b;
            for (int32_t sub = 0; sub < a.n_sub; ++sub) {
              const int32_t boff = sub * StCfg<KRE>::kStageB;
              for (int32_t q = -1; q < cn; ++q) {                 // q = -1: the target
                const int32_t v = __shfl_sync(0xffffffffu, (q & 32) ? sb : sa, q < 0 ? 0 : (q & 31));
                if (lane == 0) {
                  const int32_t phys = q < 0 ? tphys : checked_phys(a, v);
                  // output row: the pair (Euclidean / cosine dot) or, for the target stage, the
                  // target (cosine: its squared norm)
                  const int64_t po = q < 0 ? cur.t : (int64_t)(cur.lo + c0 + q);
                  mbar_wait(&sm.empty[stage], ph ^ 1u);
                  sm.hdr[stage] = make_hdr((((po * a.N + l) * 2 + kv) * a.n_sub + sub) * kConsumerWarps,
                                           StCfg<KRE>::kStageB, q < 0 ? H_ANCHOR : H_PAIR);
                  mbar_expect_tx(&sm.full[stage], (uint32_t)StCfg<KRE>::kStageB);
                  bulk_g2s(sm.ring[stage], base + (int64_t)phys * a.block_stride_b + boff,
                           (uint32_t)StCfg<KRE>::kStageB, &sm.full[stage]);
                  if (++stage == NS) { stage = 0; ph ^= 1u; }
                }
              }
            }
          }
      }
    }
    __syncwarp();
    unit = next;
    next = __shfl_sync(0xffffffffu, next2, 0);
    cur = nm;
  }
  stage = __shfl_sync(0xffffffffu, stage, 0);
  ph = __shfl_sync(0xffffffffu, ph, 0);
  if (lane == 0) {
    mbar_wait(&sm.empty[stage], ph ^ 1u);
    sm.hdr[stage] = make_hdr(0, 0, H_STOP);
    mbar_arrive(&sm.full[stage]);
  }
}

template <int KRE, int MET>
__device__ __forceinline__ void st_eval(const DistArgs& a, int4 h, const uint4 (&x)[KRE], float2 (&T)[KRE * 4],
                                        int warp, int lane) {
  if (MET == MEMSHARE_METRIC_COSINE) {
    // f2 (reading R34): target stage -> cache + squared norm; source stage -> dot + squared norm
    const int64_t o = (int64_t)(((uint64_t)(uint32_t)h.y << 32) | (uint32_t)h.x) + warp;
    float2 n0 = make_float2(0.f, 0.f), n1 = n0;
    if (h.w & H_ANCHOR) {
#pragma unroll
      for (int r = 0; r < KRE; ++r) {
        const float2 f0 = bf2_to_f2(x[r].x), f1 = bf2_to_f2(x[r].y), f2 = bf2_to_f2(x[r].z), f3 = bf2_to_f2(x[r].w);
        T[4 * r + 0] = f0; T[4 * r + 1] = f1; T[4 * r + 2] = f2; T[4 * r + 3] = f3;
        n0 = __ffma2_rn(f0, f0, n0); n1 = __ffma2_rn(f1, f1, n1);
        n0 = __ffma2_rn(f2, f2, n0); n1 = __ffma2_rn(f3, f3, n1);
      }
      const float tn = warp_sum((n0.x + n0.y) + (n1.x + n1.y));
      if (lane == 0) a.ws.wtn[o] = tn;
    } else if (h.w & H_PAIR) {
      float2 d0 = make_float2(0.f, 0.f), d1 = d0;
#pragma unroll
      for (int r = 0; r < KRE; ++r) {
        const float2 f0 = bf2_to_f2(x[r].x), f1 = bf2_to_f2(x[r].y), f2 = bf2_to_f2(x[r].z), f3 = bf2_to_f2(x[r].w);
        d0 = __ffma2_rn(T[4 * r + 0], f0, d0); d1 = __ffma2_rn(T[4 * r + 1], f1, d1);
        d0 = __ffma2_rn(T[4 * r + 2], f2, d0); d1 = __ffma2_rn(T[4 * r + 3], f3, d1);
        n0 = __ffma2_rn(f0, f0, n0); n1 = __ffma2_rn(f1, f1, n1);
        n0 = __ffma2_rn(f2, f2, n0); n1 = __ffma2_rn(f3, f3, n1);
      }
      const float dot = warp_sum((d0.x + d0.y) + (d1.x + d1.y));
      const float sn = warp_sum((n0.x + n0.y) + (n1.x + n1.y));
      if (lane == 0) { a.ws.wpart[o] = dot; a.ws.wsn[o] = sn; }
    }
    return;
  }
  if (h.w & H_ANCHOR) {
#pragma unroll
    for (int r = 0; r < KRE; ++r) {
      T[4 * r + 0] = bf2_to_f2(x[r].x);
      T[4 * r + 1] = bf2_to_f2(x[r].y);
      T[4 * r + 2] = bf2_to_f2(x[r].z);
      T[4 * r + 3] = bf2_to_f2(x[r].w);
    }
  } else if (h.w & H_PAIR) {
    float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < KRE; ++r) {
      const float2 d0 = sub_bf2(x[r].x, T[4 * r + 0]);
      const float2 d1 = sub_bf2(x[r].y, T[4 * r + 1]);
      const float2 d2 = sub_bf2(x[r].z, T[4 * r + 2]);
      const float2 d3 = sub_bf2(x[r].w, T[4 * r + 3]);
      acc0 = __ffma2_rn(d0, d0, acc0);
      acc1 = __ffma2_rn(d1, d1, acc1);
      acc0 = __ffma2_rn(d2, d2, acc0);
      acc1 = __ffma2_rn(d3, d3, acc1);
    }
    const float s = warp_sum((acc0.x + acc0.y) + (acc1.x + acc1.y));
    if (lane == 0) a.ws.wpart[(int64_t)(((uint64_t)(uint32_t)h.y << 32) | (uint32_t)h.x) + warp] = s;
  }
}

template <int KRE, int MET>
__global__ void __launch_bounds__(kThreads, 1) distance_st_kernel(DistArgs a) {
  constexpr int NS = StCfg<KRE>::kNSt;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  StSmem<KRE>& sm = *reinterpret_cast<StSmem<KRE>*>(smem_raw);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  if (warp == kConsumerWarps) {
    st_producer<KRE>(sm, a, lane);
    return;
  }
  // consumers: ping-pong register buffers (the next stage is copied while this one is evaluated)
  float2 T[KRE * 4];
  uint4 xa[KRE], xb[KRE];
  int stage = 0;
  uint32_t ph = 0;
  auto load = [&](uint4 (&dst)[KRE]) {
    const uint4* src = reinterpret_cast<const uint4*>(sm.ring[stage]);
#pragma unroll
    for (int r = 0; r < KRE; ++r) dst[r] = src[tid + r * kConsumers];
  };
  auto release = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[stage]);
    if (++stage == NS) { stage = 0; ph ^= 1u; }
  };
  mbar_wait(&sm.full[stage], ph);
  int4 ha = sm.hdr[stage], hb;
  if (ha.w & H_STOP) return;
  load(xa);
  release();
  for (;;) {
    mbar_wait(&sm.full[stage], ph);
    hb = sm.hdr[stage];
    if (!(hb.w & H_STOP)) load(xb);
    st_eval<KRE, MET>(a, ha, xa, T, warp, lane);
    if (hb.w & H_STOP) break;
    release();
    mbar_wait(&sm.full[stage], ph);
    ha = sm.hdr[stage];
    if (!(ha.w & H_STOP)) load(xa);
    st_eval<KRE, MET>(a, hb, xb, T, warp, lane);
    if (ha.w & H_STOP) break;
    release();
  }
}

template <int KRE, int MET>
static cudaError_t launch_st(const DistArgs& a, cudaStream_t st) {
  static bool attr_set_dev[kMaxDevices] = {};
  bool& attr_set = attr_set_dev[current_device()];
  if (!attr_set) {
    const cudaError_t e = cudaFuncSetAttribute(distance_st_kernel<KRE, MET>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(StSmem<KRE>));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  return launch_pdl(distance_st_kernel<KRE, MET>, dim3(sm_count()), dim3(kThreads), sizeof(StSmem<KRE>), st, a);
}

// stage sizes with a single-target kernel: every KRE for the Euclidean metric; the cosine metric
// for the shapes of the configs (tiny 4 KiB, 32B 32 KiB, Phi-4 40 KiB), others run the generic kernel
static bool st_has(int kre, int metric) {
  if (kre < 1 || kre > kMaxKre) return false;
  return metric == MEMSHARE_METRIC_EUCLIDEAN || kre == 1 || kre == 8 || kre == 10;
}

static cudaError_t launch_st_any(int kre, int metric, const DistArgs& a, cudaStream_t st) {
  if (metric == MEMSHARE_METRIC_COSINE) {
    switch (kre) {
      case 1: return launch_st<1, MEMSHARE_METRIC_COSINE>(a, st);
      case 8: return launch_st<8, MEMSHARE_METRIC_COSINE>(a, st);
      case 10: return launch_st<10, MEMSHARE_METRIC_COSINE>(a, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (kre) {
    case 1: return launch_st<1, MEMSHARE_METRIC_EUCLIDEAN>(a, st);
    case 2: return launch_st<2, MEMSHARE_METRIC_EUCLIDEAN>(a, st);
    case 3: return launch_st<3, MEMSHARE_METRIC_EUCLIDEAN>(a, st);
    case 4: return launch_st<4, MEMSHARE_METRIC_EUCLIDEAN>(a, st);
    case 5: return launch_st<5, MEMSHARE_METRIC_EUCLIDEAN>(a, st);
    case 6: return launch_st<6, MEMSHARE_METRIC_EUCLIDEAN>(a, st);
    case 7: return launch_st<7, MEMSHARE_METRIC_EUCLIDEAN>(a, st);
    case 8: return launch_st<8, MEMSHARE_METRIC_EUCLIDEAN>(a, st);
    case 9: return launch_st<9, MEMSHARE_METRIC_EUCLIDEAN>(a, st);
    case 10: return launch_st<10, MEMSHARE_METRIC_EUCLIDEAN>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

// Finalisation: one CTA per target (grid-stride). FULL/PARTIAL read the per-warp partials the
// streaming kernel left in the workspace (kernel boundary = the only synchronisation needed);
// FINALIZE reads partial squared sums already reduced across ranks.
__global__ void __launch_bounds__(kConsumers) finalize_kernel(DistArgs a, int from_partial) {
  pdl_trigger();
  pdl_wait();
  __shared__ double terms[kConsumers];
  const int64_t T = clamp_count(a.num_targets, a.target_cap);
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x)
    finalize_target(a, t, terms, threadIdx.x, from_partial != 0, [] { __syncthreads(); });
}


}  // namespace
}  // namespace ms

using namespace ms;

// host: stage geometry of the single-target kernel for this slice size -- KRE (16-byte chunks per
// consumer thread, stage = KRE * 4 KiB) and the number of equal sub-slices; KRE = 0 when the slice
// is not a multiple of 4 KiB that splits evenly (then the generic kernel runs).
// MEMSHARE_ST_MAXKRE (1..10, tuning) caps KRE, i.e. forces smaller stages and a deeper ring.
static int st_maxk() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MEMSHARE_ST_MAXKRE");
    v = e ? atoi(e) : MS_ST_MAXKRE;
    if (v < 1 || v > kMaxKre) v = kMaxKre;
  }
  return v;
}

static int st_kre(int64_t slice_bytes, int32_t* n_sub) {
  if (slice_bytes <= 0 || slice_bytes % kChunkUnit != 0) return 0;
  const int64_t units = slice_bytes / kChunkUnit;
  const int maxk = st_maxk();
  for (int64_t ns = (units + maxk - 1) / maxk; ns <= units; ++ns)
    if (units % ns == 0) {
      if (n_sub) *n_sub = (int32_t)ns;
      return (int)(units / ns);
    }
  return 0;
}

static int32_t n_sub_of(int64_t slice_bytes) {
  return (int32_t)((slice_bytes + kStageBytes - 1) / kStageBytes);
}

// workspace: room for either kernel's sub-slice count
static int32_t n_sub_ws(int64_t slice_bytes) {
  int32_t ns = 0;
  const int32_t g = n_sub_of(slice_bytes);
  return (st_kre(slice_bytes, &ns) > 0 && ns > g) ? ns : g;
}

static thread_local cudaEvent_t g_prof_begin = nullptr, g_prof_end = nullptr;

extern "C" void memshare_profile_distance_events(void* begin, void* end) {
  g_prof_begin = static_cast<cudaEvent_t>(begin);
  g_prof_end = static_cast<cudaEvent_t>(end);
}

extern "C" size_t memshare_block_distance_workspace_size(const memshare_dims* dims, int32_t num_blocks,
                                                         int64_t pair_cap, int64_t target_cap, int32_t metric) {
  if (!dims || pair_cap < 0 || target_cap < 0 || num_blocks < 0 || dims->num_layers < 1) return 0;
  if (metric != MEMSHARE_METRIC_EUCLIDEAN && metric != MEMSHARE_METRIC_COSINE) return 0;
  const int64_t slice = (int64_t)dims->block_size * dims->num_kv_heads_local * dims->head_dim * 2;
  Ws w{nullptr, 0};
  dist_layout(w, dims->num_layers, n_sub_ws(slice), num_blocks, pair_cap, target_cap, metric);
  return w.size();
}

extern "C" memshare_status memshare_block_distance(const memshare_kv_pool* pool, const memshare_dims* dims,
                                                   const memshare_block_pair* pairs, const int64_t* target_off,
                                                   const int64_t* num_pairs, const int64_t* num_targets,
                                                   int64_t pair_cap, int64_t target_cap, int32_t mode,
                                                   int32_t metric, float* partial_sq, float tau_b, float* distance,
                                                   uint8_t* under,
                                                   memshare_decision* decisions, void* workspace,
                                                   size_t workspace_bytes, int32_t* device_status, void* stream) {
  if (!dims || !pairs || !target_off || !num_pairs || !num_targets || !workspace || !device_status)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (mode < MEMSHARE_DIST_FULL || mode > MEMSHARE_DIST_FINALIZE) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (metric != MEMSHARE_METRIC_EUCLIDEAN && metric != MEMSHARE_METRIC_COSINE) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (metric == MEMSHARE_METRIC_COSINE && (mode != MEMSHARE_DIST_FULL || kAnchors != 1))
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (pair_cap < 0 || pair_cap > ((int64_t)1 << 30) || target_cap < 0 || target_cap > (int64_t)INT32_MAX)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  const memshare_dims dm = *dims;
  if (dm.num_layers < 1 || dm.num_layers > 256 || dm.num_kv_heads_local < 1 || dm.num_kv_heads_global < 1 ||
      dm.num_kv_heads_local > dm.num_kv_heads_global || dm.head_dim < 8 || dm.head_dim % 8 != 0 || dm.block_size < 1)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (!(tau_b >= 0.f)) return MEMSHARE_ERR_INVALID_ARGUMENT;   // rejects NaN too
  if (mode != MEMSHARE_DIST_PARTIAL && (!distance || !under || !decisions)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (mode != MEMSHARE_DIST_FULL && !partial_sq) return MEMSHARE_ERR_INVALID_ARGUMENT;
  const int64_t slice_bytes = (int64_t)dm.block_size * dm.num_kv_heads_local * dm.head_dim * 2;
  if (slice_bytes > (int64_t)INT32_MAX / 2) return MEMSHARE_ERR_INVALID_ARGUMENT;
  int32_t num_blocks = 0;
  if (mode != MEMSHARE_DIST_FINALIZE) {
    if (!pool || !pool->k || !pool->v || pool->num_blocks < 0) return MEMSHARE_ERR_INVALID_ARGUMENT;
    if (!aligned16(pool->k) || !aligned16(pool->v) || (pool->layer_stride * 2) % 16 != 0 ||
        (pool->block_stride * 2) % 16 != 0 || pool->layer_stride < 0 || pool->block_stride < 0)
      return MEMSHARE_ERR_INVALID_ARGUMENT;
    num_blocks = pool->num_blocks;
  }
  if (workspace_bytes < memshare_block_distance_workspace_size(dims, num_blocks, pair_cap, target_cap, metric))
    return MEMSHARE_ERR_INVALID_ARGUMENT;

  DistArgs a{};
  if (mode != MEMSHARE_DIST_FINALIZE) {
    a.kbase = static_cast<const uint8_t*>(pool->k);
    a.vbase = static_cast<const uint8_t*>(pool->v);
    a.layer_stride_b = pool->layer_stride * 2;
    a.block_stride_b = pool->block_stride * 2;
  }
  a.num_blocks = num_blocks;
  a.N = dm.num_layers; a.d = dm.block_size; a.h_global = dm.num_kv_heads_global;
  a.slice_bytes = (int32_t)slice_bytes;
  a.n_sub = n_sub_of(slice_bytes);
  a.sub_bytes = (int32_t)(((slice_bytes / a.n_sub) + 15) / 16 * 16);
  int32_t st_nsub = 0;
  int kre = (kAnchors == 1 && MS_PIPE && mode != MEMSHARE_DIST_FINALIZE) ? st_kre(slice_bytes, &st_nsub) : 0;
  if (!st_has(kre, metric)) kre = 0;
  if (kre > 0) {                                      // equal sub-slices of exactly one stage each
    a.n_sub = st_nsub;
    a.sub_bytes = kre * kChunkUnit;
  }
  static int lpi_env = -1;
  if (lpi_env < 0) {
    const char* e = getenv("MEMSHARE_LAYERS_PER_ITEM");
    lpi_env = e ? atoi(e) : 0;
    if (lpi_env < 0) lpi_env = 0;
  }
  a.lpi = lpi_env > 0 ? lpi_env : 2;
  if (a.lpi > a.N) a.lpi = a.N;
  a.n_chunks = (a.N + a.lpi - 1) / a.lpi;
  a.pairs = pairs; a.target_off = target_off; a.num_pairs = num_pairs; a.num_targets = num_targets;
  a.pair_cap = pair_cap; a.target_cap = target_cap; a.mode = mode; a.metric = metric; a.partial_sq = partial_sq; a.tau_b = tau_b;
  a.distance = distance; a.under = under; a.decisions = decisions; a.status = device_status;
  Ws w{static_cast<char*>(workspace), 0};
  a.ws = dist_layout(w, a.N, a.n_sub, num_blocks, pair_cap, target_cap, metric);
  {
    int64_t np2 = 1;
    while (np2 < target_cap && np2 < kPlanSortCap) np2 <<= 1;
    a.plan_sort_cap = (int32_t)np2;
  }

  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t tc = target_cap < 1 ? 1 : target_cap;
  const int fin_grid = (int)(tc < 8 * sm_count() ? tc : 8 * sm_count());
  if (mode == MEMSHARE_DIST_FINALIZE) {
    launch_pdl(finalize_kernel, dim3(fin_grid), dim3(kConsumers), 0, st, a, 1);
    return launch_status();
  }
  static bool attr_set_dev[kMaxDevices] = {};
  bool& attr_set = attr_set_dev[current_device()];
  if (!attr_set) {
    if (cudaFuncSetAttribute(distance_kernel<MEMSHARE_METRIC_EUCLIDEAN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(DistSmem)) != cudaSuccess ||
        cudaFuncSetAttribute(distance_kernel<MEMSHARE_METRIC_COSINE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(DistSmem)) != cudaSuccess ||
        cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kPlanSortCap * sizeof(unsigned long long))) != cudaSuccess)
      return MEMSHARE_ERR_CUDA;
    attr_set = true;
  }
  if (cudaMemsetAsync(a.ws.ticket, 0, sizeof(unsigned int), st) != cudaSuccess) return MEMSHARE_ERR_CUDA;
  int64_t plan_np2 = 1;
  while (plan_np2 < target_cap && plan_np2 < kPlanSortCap) plan_np2 <<= 1;
  if (kAnchors > 1) launch_pdl(plan_kernel, dim3(1), dim3(kPlanThreads), (size_t)plan_np2 * sizeof(unsigned long long), st, a);
  const bool prof = g_prof_begin != nullptr && g_prof_end != nullptr;
  if (prof && cudaEventRecord(g_prof_begin, st) != cudaSuccess) return MEMSHARE_ERR_CUDA;
  if (kre > 0) {
    if (launch_st_any(kre, metric, a, st) != cudaSuccess) return MEMSHARE_ERR_CUDA;
  } else if (metric == MEMSHARE_METRIC_COSINE)
    launch_pdl(distance_kernel<MEMSHARE_METRIC_COSINE>, dim3(sm_count()), dim3(kThreads), sizeof(DistSmem), st, a);
  else
    launch_pdl(distance_kernel<MEMSHARE_METRIC_EUCLIDEAN>, dim3(sm_count()), dim3(kThreads), sizeof(DistSmem), st, a);
  if (prof && cudaEventRecord(g_prof_end, st) != cudaSuccess) return MEMSHARE_ERR_CUDA;
  launch_pdl(finalize_kernel, dim3(fin_grid), dim3(kConsumers), 0, st, a, 0);
  return launch_status();
}

extern "C" memshare_status memshare_block_distance_finalize_peers(
    const float* const* partial_peers, int32_t num_peers, const memshare_dims* dims,
    const memshare_block_pair* pairs, const int64_t* target_off, const int64_t* num_pairs,
    const int64_t* num_targets, int64_t pair_cap, int64_t target_cap, float tau_b, float* distance, uint8_t* under,
    memshare_decision* decisions, void* workspace, size_t workspace_bytes, int32_t* device_status, void* stream) {
  if (!partial_peers || num_peers < 1 || num_peers > 64 || !dims || !pairs || !target_off || !num_pairs ||
      !num_targets || !distance || !under || !decisions || !workspace || !device_status)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (pair_cap < 0 || pair_cap > ((int64_t)1 << 30) || target_cap < 0 || target_cap > (int64_t)INT32_MAX)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  const memshare_dims dm = *dims;
  if (dm.num_layers < 1 || dm.num_layers > 256 || dm.num_kv_heads_global < 1 || dm.block_size < 1 ||
      dm.head_dim < 8 || dm.head_dim % 8 != 0)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (!(tau_b >= 0.f)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < memshare_block_distance_workspace_size(dims, 0, pair_cap, target_cap, MEMSHARE_METRIC_EUCLIDEAN))
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  DistArgs a{};
  a.N = dm.num_layers; a.d = dm.block_size; a.h_global = dm.num_kv_heads_global;
  const int64_t slice_bytes = (int64_t)dm.block_size * dm.num_kv_heads_local * dm.head_dim * 2;
  a.slice_bytes = (int32_t)slice_bytes;
  a.n_sub = n_sub_of(slice_bytes);
  a.pairs = pairs; a.target_off = target_off; a.num_pairs = num_pairs; a.num_targets = num_targets;
  a.pair_cap = pair_cap; a.target_cap = target_cap; a.mode = MEMSHARE_DIST_FINALIZE;
  a.metric = MEMSHARE_METRIC_EUCLIDEAN; a.tau_b = tau_b;
  a.distance = distance; a.under = under; a.decisions = decisions; a.status = device_status;
  a.peers = partial_peers; a.num_peers = num_peers;
  Ws w{static_cast<char*>(workspace), 0};
  a.ws = dist_layout(w, a.N, a.n_sub, 0, pair_cap, target_cap, MEMSHARE_METRIC_EUCLIDEAN);
  const int64_t tc = target_cap < 1 ? 1 : target_cap;
  const int fin_grid = (int)(tc < 8 * sm_count() ? tc : 8 * sm_count());
  launch_pdl(finalize_kernel, dim3(fin_grid), dim3(kConsumers), 0, static_cast<cudaStream_t>(stream), a, 1);
  return launch_status();
}

