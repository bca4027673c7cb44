// a5-a6 -- Stage 2 block distance + threshold + per-target selection.
// PAPER.md:237-248 (Alg. 1 Stage 2):  D = (1/N) sum_l (||K_l[Bt]-K_l[Bs]||_F + ||V_l[Bt]-V_l[Bs]||_F)/(2dh)
// PAPER.md:268 ("small Euclidean distance are flagged as reusable"), :319-320 (minimal distance).
//
// B200 design. The op is a bf16 reduction bound by HBM, not a contraction: no
// tensor cores. Two launches:
//  distance_kernel -- one persistent CTA per SM:
//   * warp 16 (producer) takes work items (target t, layer chunk) from a global ticket, in
//     layer-chunk-major order so that concurrently running items touch the same layers and a
//     source block shared by several targets is re-read from L2, not HBM; it stages the item's
//     source ids in smem with its 32 lanes and, for every (layer, K|V, sub-slice), issues 1-D
//     TMA bulk copies (cp.async.bulk, SASS UBLKCP) of the target slice and then of each source
//     slice into a 6-stage shared-memory ring, signalled through mbarrier complete_tx;
//   * warps 0-15 (consumers) cache the target sub-slice in registers as fp32 and release its
//     stage at once, then for each source stage compute sum (t - s)^2 with packed FFMA2 (32
//     terms per thread), reduce over the warp with shuffles and store one fp32 partial per warp
//     (no fp atomics, fixed order). Consumers never synchronise beyond the ring barriers.
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
#define MS_CONSUMER_WARPS 16
#endif
#ifndef MS_STAGE_BYTES
#define MS_STAGE_BYTES 32768
#endif
#ifndef MS_STAGES
#define MS_STAGES 6
#endif
#ifndef MS_COPY_PIECE
#define MS_COPY_PIECE 8192
#endif
#ifndef MS_DIAG_NO_COMPUTE
#define MS_DIAG_NO_COMPUTE 0      // 1 = consumers release stages without reading them (bandwidth probe)
#endif
constexpr int kConsumerWarps = MS_CONSUMER_WARPS;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;
constexpr int kStageBytes = MS_STAGE_BYTES;
constexpr int kStages = MS_STAGES;
constexpr int kR = kStageBytes / 16 / kConsumers;   // uint4 chunks per consumer thread per stage
constexpr int kCopyPiece = MS_COPY_PIECE;
constexpr int kMaxStagedPairs = 1024;   // source ids staged in smem per item

constexpr int F_TARGET = 1, F_ITEM_END = 2, F_STOP = 4, F_SKIP = 8;

struct Meta {
  int64_t pair;
  int64_t target;
  int32_t layer;
  int32_t kv;
  int32_t sub;
  int32_t bytes;
  int32_t flags;
  int32_t pad;
};

struct DistWs {
  unsigned int* ticket;
  float* wpart;          // [pair_cap][N][2][n_sub][kConsumerWarps]
};

DistWs dist_layout(Ws& w, int32_t N, int32_t n_sub, int64_t pair_cap, int64_t target_cap) {
  DistWs d;
  d.ticket = w.take<unsigned int>(1);
  d.wpart = w.take<float>((size_t)pair_cap * N * 2 * n_sub * kConsumerWarps + 1);
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
  const memshare_block_pair* pairs;
  const int64_t* target_off;
  const int64_t* num_pairs;
  const int64_t* num_targets;
  int64_t pair_cap, target_cap;
  int32_t mode;
  float* partial_sq;
  float tau_b;
  float* distance;
  uint8_t* under;
  memshare_decision* decisions;
  int32_t* status;
  DistWs ws;
};

struct DistSmem {
  alignas(128) uint8_t ring[kStages][kStageBytes];
  alignas(8) uint64_t full[kStages];
  uint64_t empty[kStages];
  Meta meta[kStages];
  int32_t src_phys[kMaxStagedPairs];
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

// fixed-order fp32 sum of the per-warp partials of (pair p, layer l, kv)
__device__ __forceinline__ float sum_part(const DistArgs& a, int64_t p, int32_t l, int32_t kv, bool from_partial) {
  if (from_partial) return __ldcg(a.partial_sq + ((p * a.N + l) * 2 + kv));
  const float* w = a.ws.wpart + (((p * a.N + l) * 2 + kv) * a.n_sub) * kConsumerWarps;
  float s = 0.f;
  for (int j = 0; j < a.n_sub * kConsumerWarps; ++j) s += __ldcg(w + j);
  return s;
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
      const float sk = sum_part(a, p, l, 0, from_partial);
      const float sv = sum_part(a, p, l, 1, from_partial);
      if (!from_partial && a.partial_sq != nullptr) {
        a.partial_sq[(p * N + l) * 2 + 0] = sk;
        a.partial_sq[(p * N + l) * 2 + 1] = sv;
      }
      // Alg. 1 line 5: (Delta_K + Delta_V) / (2dh)
      terms[tid] = (__dsqrt_rn((double)sk) + __dsqrt_rn((double)sv)) * inv;
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
          const float D = (float)(acc / (double)N);     // Alg. 1 line 7: return D / N
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

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------------ producer warp
    // All 32 lanes stage the item's source ids into smem (one coalesced round trip instead of
    // a dependent global load per copy) and lane 0 fetches the next ticket while the current
    // item's copies are issued, so the ring never waits on metadata latency.
    const int64_t T = clamp_count(a.num_targets, a.target_cap);
    const int64_t P = clamp_count(a.num_pairs, a.pair_cap);
    const int64_t total = T * a.n_chunks;
    int stage = 0;
    uint32_t ph = 0;
    auto push = [&](const Meta& m, const uint8_t* src) {
      mbar_wait(&sm.empty[stage], ph ^ 1u);
      sm.meta[stage] = m;
      if (src != nullptr) {
        mbar_expect_tx(&sm.full[stage], (uint32_t)m.bytes);
        for (int off = 0; off < m.bytes; off += kCopyPiece) {
          const int nb = (m.bytes - off) < kCopyPiece ? (m.bytes - off) : kCopyPiece;
          bulk_g2s(sm.ring[stage] + off, src + off, (uint32_t)nb, &sm.full[stage]);
        }
      } else {
        mbar_arrive(&sm.full[stage]);
      }
      if (++stage == kStages) { stage = 0; ph ^= 1u; }
    };
    int64_t item = 0;
    if (lane == 0) item = (int64_t)atomicAdd(a.ws.ticket, 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    while (item < total) {
      int64_t next = 0;
      if (lane == 0) next = (int64_t)atomicAdd(a.ws.ticket, 1u);   // consumed at the end of the item
      const int64_t lc = item / T, t = item - lc * T;
      const int64_t p0 = __ldcg(a.target_off + t);
      int64_t p1 = __ldcg(a.target_off + t + 1);
      if (p1 > P) p1 = P;
      const int64_t np = p1 - p0;
      for (int64_t q = lane; q < np && q < kMaxStagedPairs; q += 32)
        sm.src_phys[q] = checked_phys(a, a.pairs[p0 + q].source_phys);
      const int32_t tphys = np > 0 ? checked_phys(a, a.pairs[p0].target_phys) : 0;
      __syncwarp();
      if (lane == 0) {
        Meta m{};
        m.target = t;
        if (np <= 0) {
          m.pair = -1; m.flags = F_ITEM_END | F_SKIP;
          push(m, nullptr);
        } else {
          const int32_t l0 = (int32_t)lc * a.lpi;
          const int32_t l1 = (l0 + a.lpi < a.N) ? l0 + a.lpi : a.N;
          for (int32_t l = l0; l < l1; ++l) {
            for (int32_t kv = 0; kv < 2; ++kv) {
              const uint8_t* base = (kv ? a.vbase : a.kbase) + (int64_t)l * a.layer_stride_b;
              for (int32_t sub = 0; sub < a.n_sub; ++sub) {
                const int32_t off = sub * a.sub_bytes;
                const int32_t bytes = (a.slice_bytes - off) < a.sub_bytes ? (a.slice_bytes - off) : a.sub_bytes;
                m.layer = l; m.kv = kv; m.sub = sub; m.bytes = bytes;
                m.pair = -1; m.flags = F_TARGET;
                push(m, base + (int64_t)tphys * a.block_stride_b + off);
                for (int64_t q = 0; q < np; ++q) {
                  const int32_t sphys = q < kMaxStagedPairs ? sm.src_phys[q]
                                                            : checked_phys(a, a.pairs[p0 + q].source_phys);
                  m.pair = p0 + q;
                  m.flags = (l == l1 - 1 && kv == 1 && sub == a.n_sub - 1 && q == np - 1) ? F_ITEM_END : 0;
                  push(m, base + (int64_t)sphys * a.block_stride_b + off);
                }
              }
            }
          }
        }
      }
      __syncwarp();
      item = __shfl_sync(0xffffffffu, next, 0);
    }
    if (lane == 0) {
      Meta stop{};
      stop.flags = F_STOP;
      push(stop, nullptr);
    }
    return;
  }

  // -------------------------------------------------------------------- consumer warps
  float2 tv[kR * 4];
  int stage = 0;
  uint32_t ph = 0;
  for (;;) {
    mbar_wait(&sm.full[stage], ph);
    const Meta m = sm.meta[stage];
    if (m.flags & F_STOP) break;
    if (!(m.flags & F_SKIP) && !MS_DIAG_NO_COMPUTE) {
      const uint4* src = reinterpret_cast<const uint4*>(sm.ring[stage]);
      const int nchunk = m.bytes >> 4;
      if (m.flags & F_TARGET) {
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const int c = tid + r * kConsumers;
          uint4 x = make_uint4(0u, 0u, 0u, 0u);
          if (c < nchunk) x = src[c];
          tv[4 * r + 0] = bf2_to_f2(x.x);
          tv[4 * r + 1] = bf2_to_f2(x.y);
          tv[4 * r + 2] = bf2_to_f2(x.z);
          tv[4 * r + 3] = bf2_to_f2(x.w);
        }
      } else {
        float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
        const float2 neg1 = make_float2(-1.f, -1.f);
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const int c = tid + r * kConsumers;
          if (c < nchunk) {
            const uint4 x = src[c];
            // d = t - s exactly rounded (fma with -1), acc += d*d; packed f32x2 (FFMA2)
            const float2 d0 = __ffma2_rn(bf2_to_f2(x.x), neg1, tv[4 * r + 0]);
            const float2 d1 = __ffma2_rn(bf2_to_f2(x.y), neg1, tv[4 * r + 1]);
            const float2 d2 = __ffma2_rn(bf2_to_f2(x.z), neg1, tv[4 * r + 2]);
            const float2 d3 = __ffma2_rn(bf2_to_f2(x.w), neg1, tv[4 * r + 3]);
            acc0 = __ffma2_rn(d0, d0, acc0);
            acc1 = __ffma2_rn(d1, d1, acc1);
            acc0 = __ffma2_rn(d2, d2, acc0);
            acc1 = __ffma2_rn(d3, d3, acc1);
          }
        }
        float s = (acc0.x + acc0.y) + (acc1.x + acc1.y);
        s = warp_sum(s);
        if (lane == 0)
          a.ws.wpart[(((m.pair * a.N + m.layer) * 2 + m.kv) * a.n_sub + m.sub) * kConsumerWarps + warp] = s;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[stage]);
    if (++stage == kStages) { stage = 0; ph ^= 1u; }
  }
}

// Finalisation: one CTA per target (grid-stride). FULL/PARTIAL read the per-warp partials the
// streaming kernel left in the workspace (kernel boundary = the only synchronisation needed);
// FINALIZE reads partial squared sums already reduced across ranks.
__global__ void __launch_bounds__(kConsumers) finalize_kernel(DistArgs a, int from_partial) {
  __shared__ double terms[kConsumers];
  const int64_t T = clamp_count(a.num_targets, a.target_cap);
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x)
    finalize_target(a, t, terms, threadIdx.x, from_partial != 0, [] { __syncthreads(); });
}

}  // namespace
}  // namespace ms

using namespace ms;

static int32_t n_sub_of(int64_t slice_bytes) {
  return (int32_t)((slice_bytes + kStageBytes - 1) / kStageBytes);
}

extern "C" size_t memshare_block_distance_workspace_size(const memshare_dims* dims, int64_t pair_cap,
                                                         int64_t target_cap) {
  if (!dims || pair_cap < 0 || target_cap < 0 || dims->num_layers < 1) return 0;
  const int64_t slice = (int64_t)dims->block_size * dims->num_kv_heads_local * dims->head_dim * 2;
  Ws w{nullptr, 0};
  dist_layout(w, dims->num_layers, n_sub_of(slice), pair_cap, target_cap);
  return w.size();
}

extern "C" memshare_status memshare_block_distance(const memshare_kv_pool* pool, const memshare_dims* dims,
                                                   const memshare_block_pair* pairs, const int64_t* target_off,
                                                   const int64_t* num_pairs, const int64_t* num_targets,
                                                   int64_t pair_cap, int64_t target_cap, int32_t mode,
                                                   float* partial_sq, float tau_b, float* distance, uint8_t* under,
                                                   memshare_decision* decisions, void* workspace,
                                                   size_t workspace_bytes, int32_t* device_status, void* stream) {
  if (!dims || !pairs || !target_off || !num_pairs || !num_targets || !workspace || !device_status)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (mode < MEMSHARE_DIST_FULL || mode > MEMSHARE_DIST_FINALIZE) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (pair_cap < 0 || target_cap < 0) return MEMSHARE_ERR_INVALID_ARGUMENT;
  const memshare_dims dm = *dims;
  if (dm.num_layers < 1 || dm.num_layers > 256 || dm.num_kv_heads_local < 1 || dm.num_kv_heads_global < 1 ||
      dm.num_kv_heads_local > dm.num_kv_heads_global || dm.head_dim < 8 || dm.head_dim % 8 != 0 || dm.block_size < 1)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (!(tau_b >= 0.f)) return MEMSHARE_ERR_INVALID_ARGUMENT;   // rejects NaN too
  if (mode != MEMSHARE_DIST_PARTIAL && (!distance || !under || !decisions)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (mode != MEMSHARE_DIST_FULL && !partial_sq) return MEMSHARE_ERR_INVALID_ARGUMENT;
  const int64_t slice_bytes = (int64_t)dm.block_size * dm.num_kv_heads_local * dm.head_dim * 2;
  if (slice_bytes > (int64_t)INT32_MAX / 2) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (mode != MEMSHARE_DIST_FINALIZE) {
    if (!pool || !pool->k || !pool->v || pool->num_blocks < 0) return MEMSHARE_ERR_INVALID_ARGUMENT;
    if (!aligned16(pool->k) || !aligned16(pool->v) || (pool->layer_stride * 2) % 16 != 0 ||
        (pool->block_stride * 2) % 16 != 0 || pool->layer_stride < 0 || pool->block_stride < 0)
      return MEMSHARE_ERR_INVALID_ARGUMENT;
  }
  if (workspace_bytes < memshare_block_distance_workspace_size(dims, pair_cap, target_cap))
    return MEMSHARE_ERR_INVALID_ARGUMENT;

  DistArgs a{};
  if (mode != MEMSHARE_DIST_FINALIZE) {
    a.kbase = static_cast<const uint8_t*>(pool->k);
    a.vbase = static_cast<const uint8_t*>(pool->v);
    a.layer_stride_b = pool->layer_stride * 2;
    a.block_stride_b = pool->block_stride * 2;
    a.num_blocks = pool->num_blocks;
  }
  a.N = dm.num_layers; a.d = dm.block_size; a.h_global = dm.num_kv_heads_global;
  a.slice_bytes = (int32_t)slice_bytes;
  a.n_sub = n_sub_of(slice_bytes);
  a.sub_bytes = (int32_t)(((slice_bytes / a.n_sub) + 15) / 16 * 16);
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
  a.pair_cap = pair_cap; a.target_cap = target_cap; a.mode = mode; a.partial_sq = partial_sq; a.tau_b = tau_b;
  a.distance = distance; a.under = under; a.decisions = decisions; a.status = device_status;
  Ws w{static_cast<char*>(workspace), 0};
  a.ws = dist_layout(w, a.N, a.n_sub, pair_cap, target_cap);

  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t tc = target_cap < 1 ? 1 : target_cap;
  const int fin_grid = (int)(tc < 8 * sm_count() ? tc : 8 * sm_count());
  if (mode == MEMSHARE_DIST_FINALIZE) {
    finalize_kernel<<<fin_grid, kConsumers, 0, st>>>(a, 1);
    return launch_status();
  }
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(distance_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DistSmem)) !=
        cudaSuccess)
      return MEMSHARE_ERR_CUDA;
    attr_set = true;
  }
  if (cudaMemsetAsync(a.ws.ticket, 0, sizeof(unsigned int), st) != cudaSuccess) return MEMSHARE_ERR_CUDA;
  distance_kernel<<<sm_count(), kThreads, sizeof(DistSmem), st>>>(a);
  finalize_kernel<<<fin_grid, kConsumers, 0, st>>>(a, 0);
  return launch_status();
}
