// f1 -- decode-loop integration: the steps on either side of the MemShare path.
//   memshare_kv_append               one decode token per active sequence into the paged pool,
//                                    fresh blocks popped from the free list remap() fills
//   memshare_paged_attention_decode  one layer of GQA decode attention read THROUGH the (remapped)
//                                    block table: split-KV over 256-token chunks + combine
//   memshare_admit                   host-side FCFS block-budget admission
// PAPER.md:276-284 (shared blocks are read through the block table, no copy), :322 (vLLM paged
// attention), :177-193 (Theorem 1); readings R35-R37.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>

#include "common.cuh"

namespace ms {
namespace {

// ------------------------------------------------------------------------------ KV append
constexpr int kAppNT = 1024;

struct AppWs {
  int32_t* slot_blk;   // [num_seqs] physical block of the appended token, -1 = none
  int32_t* slot_off;   // [num_seqs]
  int32_t* ok;         // 1 = state updated, copy the rows
};

AppWs app_layout(Ws& w, int32_t num_seqs) {
  AppWs a;
  a.slot_blk = w.take<int32_t>((size_t)num_seqs + 1);
  a.slot_off = w.take<int32_t>((size_t)num_seqs + 1);
  a.ok = w.take<int32_t>(1);
  return a;
}

// One CTA: validate every sequence (all-or-nothing), then pop fresh blocks LIFO in sequence
// order (rank = exclusive scan of the needs), update table / refcount / free_count / seq_len.
__global__ void __launch_bounds__(kAppNT) append_alloc_kernel(int32_t* table, int32_t stride, int32_t num_seqs,
                                                              int32_t* seq_len, const uint8_t* active,
                                                              int32_t* refcount, int32_t num_blocks,
                                                              const int32_t* free_list, int64_t* free_count,
                                                              int32_t block_size, AppWs ws, int32_t* status) {
  __shared__ int64_t sh[kAppNT / 32 + 1];
  const int64_t fc = *free_count;
  int err = 0;          // 2 capacity, 3 corruption, 1 invalid
  int64_t need_total = 0;
  for (int32_t base = 0; base < num_seqs; base += kAppNT) {
    const int32_t s = base + threadIdx.x;
    int64_t need = 0;
    if (s < num_seqs && (active == nullptr || active[s])) {
      const int32_t pos = seq_len[s];
      if (pos < 0) {
        err = max(err, 1);
      } else {
        const int32_t lb = pos / block_size, off = pos % block_size;
        if (lb >= stride) {
          err = max(err, 2);
        } else if (off == 0) {
          need = 1;
        } else {
          const int32_t b = table[(int64_t)s * stride + lb];
          if (b < 0 || b >= num_blocks || refcount[b] != 1) err = 3;
        }
      }
    }
    int64_t tot;
    block_excl_scan<kAppNT>(need, tot, sh);
    need_total += tot;
  }
  if (need_total > fc) err = max(err, 2);
  for (int64_t r = threadIdx.x; r < need_total && r < fc; r += kAppNT) {
    const int32_t b = free_list[fc - 1 - r];
    if (b < 0 || b >= num_blocks || refcount[b] != 0) err = 3;
  }
  // precedence as in the oracle's single pass is irrelevant for the state: any error leaves it
  // untouched; the reported code is the largest one seen (corruption > capacity > invalid)
  const int e3 = __syncthreads_or(err == 3), e2 = __syncthreads_or(err == 2), e1 = __syncthreads_or(err == 1);
  const int code = e3 ? MEMSHARE_ERR_CORRUPTION : e2 ? MEMSHARE_ERR_CAPACITY : e1 ? MEMSHARE_ERR_INVALID_ARGUMENT : 0;
  if (code != 0) {
    if (threadIdx.x == 0) { set_status(status, code); *ws.ok = 0; }
    return;
  }
  int64_t carry = 0;
  for (int32_t base = 0; base < num_seqs; base += kAppNT) {
    const int32_t s = base + threadIdx.x;
    const bool act = s < num_seqs && (active == nullptr || active[s]);
    int32_t pos = 0, lb = 0, off = 0;
    if (act) { pos = seq_len[s]; lb = pos / block_size; off = pos % block_size; }
    const int64_t need = (act && off == 0) ? 1 : 0;
    int64_t tot;
    const int64_t rank = carry + block_excl_scan<kAppNT>(need, tot, sh);
    carry += tot;
    if (s < num_seqs) {
      int32_t b = -1;
      if (act) {
        if (need) {
          b = free_list[fc - 1 - rank];
          refcount[b] = 1;
          table[(int64_t)s * stride + lb] = b;
        } else {
          b = table[(int64_t)s * stride + lb];
        }
        seq_len[s] = pos + 1;
      }
      ws.slot_blk[s] = b;
      ws.slot_off[s] = off;
    }
  }
  if (threadIdx.x == 0) { *free_count = fc - need_total; *ws.ok = 1; }
}

// Copy the new K/V rows (h * d_h bf16 each, one per (layer, sequence)) into their slots.
__global__ void append_copy_kernel(uint16_t* k, uint16_t* v, int64_t layer_stride, int64_t block_stride,
                                   int32_t num_layers, int32_t num_seqs, int32_t row_elems, const uint16_t* new_k,
                                   const uint16_t* new_v, AppWs ws) {
  if (__ldcg(ws.ok) == 0) return;
  const int vec = row_elems / 8;                 // 16-byte vectors per row
  const int64_t total = (int64_t)num_layers * num_seqs * vec;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / vec;
    const int c = (int)(i % vec);
    const int32_t l = (int32_t)(r / num_seqs), s = (int32_t)(r % num_seqs);
    const int32_t b = __ldcg(ws.slot_blk + s);
    if (b < 0) continue;
    const int64_t dst = (int64_t)l * layer_stride + (int64_t)b * block_stride +
                        (int64_t)__ldcg(ws.slot_off + s) * row_elems + c * 8;
    const int64_t src = r * row_elems + c * 8;
    *reinterpret_cast<uint4*>(k + dst) = __ldg(reinterpret_cast<const uint4*>(new_k + src));
    *reinterpret_cast<uint4*>(v + dst) = __ldg(reinterpret_cast<const uint4*>(new_v + src));
  }
}

// ------------------------------------------------------------------ paged decode attention
constexpr int kBlk = 16;               // tokens per KV block (the lane mapping assumes 16)
constexpr int kChunkBlocks = 16;       // blocks per CTA work item (256 tokens)
constexpr int kAttWarps = 4;
constexpr int kAttNT = kAttWarps * 32;
constexpr int kBlocksPerWarp = kChunkBlocks / kAttWarps;
constexpr int kMaxG = 8;               // query heads per KV head

struct AttArgs {
  const uint16_t* k;
  const uint16_t* v;
  int64_t layer_stride, block_stride;
  int32_t layer, h, G, num_blocks;
  const uint16_t* q;
  const int32_t* table;
  int32_t stride;
  const int32_t* seq_len;
  int32_t num_seqs, max_chunks;
  float scale;
  float* out;
  float* pm;          // [S][h][max_chunks][G]
  float* pl;
  float* pacc;        // [S][h][max_chunks][G][d_h]
  int32_t* status;
};

__device__ __forceinline__ float2 bf2f(uint32_t x) {
  return make_float2(__uint_as_float(x << 16), __uint_as_float(x & 0xFFFF0000u));
}

// One CTA per (chunk, kv head g, sequence s); warp w handles kBlocksPerWarp consecutive blocks.
// Lanes map to (token t = lane / 2, half) for the q.k scores (d_h / 2 dims each, q in smem) and to
// d_h / 32 contiguous dims for the p.V accumulation (p in smem).
template <int DH>
__global__ void __launch_bounds__(kAttNT) attn_split_kernel(AttArgs a) {
  constexpr int HALF = DH / 2;
  constexpr int QROW = DH + 4;                       // padded: the two halves sit in different banks
  constexpr int VPL = DH / 32;                        // V dims per lane
  __shared__ __align__(16) float sq[kMaxG][QROW];
  __shared__ float sp[kAttWarps][kMaxG][kBlk];
  __shared__ float s_m[kAttWarps][kMaxG], s_l[kAttWarps][kMaxG];
  __shared__ __align__(16) float s_acc[kAttWarps][kMaxG][DH];
  const int chunk = blockIdx.x, g = blockIdx.y, s = blockIdx.z;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int G = a.G;
  const int32_t len = a.seq_len[s];
  const int32_t tok0 = chunk * kChunkBlocks * kBlk;
  if (tok0 >= len) return;
  // q of this KV head's query heads -> fp32 smem
  for (int i = threadIdx.x; i < G * DH; i += kAttNT) {
    const int qi = i / DH, x = i % DH;
    const uint16_t b = a.q[((int64_t)s * a.h * G + (int64_t)g * G + qi) * DH + x];
    sq[qi][x + (x >= HALF ? 4 : 0)] = __uint_as_float((uint32_t)b << 16);
  }
  __syncthreads();
  float m[kMaxG], l[kMaxG], acc[kMaxG][VPL];
#pragma unroll
  for (int i = 0; i < kMaxG; ++i) {
    m[i] = -INFINITY;
    l[i] = 0.f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) acc[i][j] = 0.f;
  }
  const int t = lane >> 1, half = lane & 1;
  const float* qh_base = &sq[0][half * (HALF + 4)];
  const int32_t* trow = a.table + (int64_t)s * a.stride;
  const uint16_t* kl = a.k + (int64_t)a.layer * a.layer_stride;
  const uint16_t* vl = a.v + (int64_t)a.layer * a.layer_stride;
  const int64_t row = (int64_t)a.h * DH;
  for (int bi = 0; bi < kBlocksPerWarp; ++bi) {
    const int32_t lb = chunk * kChunkBlocks + w * kBlocksPerWarp + bi;
    const int32_t j0 = lb * kBlk;
    if (j0 >= len) break;
    const int ntok = min(kBlk, len - j0);
    const int32_t blk = trow[lb];
    if (blk < 0 || blk >= a.num_blocks) {
      if (lane == 0) set_status(a.status, MEMSHARE_ERR_CORRUPTION);
      break;
    }
    const uint16_t* kb = kl + (int64_t)blk * a.block_stride + g * DH;
    const uint16_t* vb = vl + (int64_t)blk * a.block_stride + g * DH;
    // issue the V loads of this block first (independent of the scores)
    uint2 vr[kBlk];
#pragma unroll
    for (int tt = 0; tt < kBlk; ++tt) {
      vr[tt] = make_uint2(0u, 0u);
      if (tt < ntok) {
        if constexpr (VPL == 4) vr[tt] = __ldg(reinterpret_cast<const uint2*>(vb + tt * row) + lane);
        else vr[tt].x = __ldg(reinterpret_cast<const uint32_t*>(vb + tt * row) + lane);
      }
    }
    // K row half of token t
    uint4 kr[HALF / 8];
    const uint4* kp = reinterpret_cast<const uint4*>(kb + t * row + half * HALF);
#pragma unroll
    for (int c = 0; c < HALF / 8; ++c) kr[c] = t < ntok ? __ldg(kp + c) : make_uint4(0u, 0u, 0u, 0u);
    float sc[kMaxG];
#pragma unroll
    for (int qi = 0; qi < kMaxG; ++qi) {
      if (qi < G) {
        const float* qv = qh_base + qi * QROW;
        float2 d = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < HALF / 8; ++c) {
          const float4 q0 = *reinterpret_cast<const float4*>(qv + c * 8);
          const float4 q1 = *reinterpret_cast<const float4*>(qv + c * 8 + 4);
          d = __ffma2_rn(make_float2(q0.x, q0.y), bf2f(kr[c].x), d);
          d = __ffma2_rn(make_float2(q0.z, q0.w), bf2f(kr[c].y), d);
          d = __ffma2_rn(make_float2(q1.x, q1.y), bf2f(kr[c].z), d);
          d = __ffma2_rn(make_float2(q1.z, q1.w), bf2f(kr[c].w), d);
        }
        float x = d.x + d.y;
        x += __shfl_xor_sync(0xffffffffu, x, 1);
        sc[qi] = t < ntok ? x * a.scale : -INFINITY;
      }
    }
    // online softmax over this block's tokens
#pragma unroll
    for (int qi = 0; qi < kMaxG; ++qi) {
      if (qi < G) {
        float bm = sc[qi];
#pragma unroll
        for (int o = 2; o < 32; o <<= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
        const float mn = fmaxf(m[qi], bm);
        const float corr = __expf(m[qi] - mn);
        const float p = __expf(sc[qi] - mn);
        float ps = half == 0 ? p : 0.f;
#pragma unroll
        for (int o = 2; o < 32; o <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
        l[qi] = l[qi] * corr + ps;
        m[qi] = mn;
#pragma unroll
        for (int j = 0; j < VPL; ++j) acc[qi][j] *= corr;
        if (half == 0) sp[w][qi][t] = p;
      }
    }
    __syncwarp();
#pragma unroll
    for (int tt = 0; tt < kBlk; ++tt) {
      if (tt < ntok) {
        const float2 v01 = bf2f(vr[tt].x);
        float2 v23 = make_float2(0.f, 0.f);
        if (VPL == 4) v23 = bf2f(vr[tt].y);
#pragma unroll
        for (int qi = 0; qi < kMaxG; ++qi) {
          if (qi < G) {
            const float p = sp[w][qi][tt];
            acc[qi][0] = fmaf(p, v01.x, acc[qi][0]);
            acc[qi][1] = fmaf(p, v01.y, acc[qi][1]);
            if (VPL == 4) {
              acc[qi][VPL - 2] = fmaf(p, v23.x, acc[qi][VPL - 2]);
              acc[qi][VPL - 1] = fmaf(p, v23.y, acc[qi][VPL - 1]);
            }
          }
        }
      }
    }
    __syncwarp();
  }
  // merge the warps' (m, l, acc) and write this chunk's partial
#pragma unroll
  for (int qi = 0; qi < kMaxG; ++qi) {
    if (qi < G) {
      if (lane == 0) { s_m[w][qi] = m[qi]; s_l[w][qi] = l[qi]; }
#pragma unroll
      for (int j = 0; j < VPL; ++j) s_acc[w][qi][lane * VPL + j] = acc[qi][j];
    }
  }
  __syncthreads();
  const int64_t pbase = (((int64_t)s * a.h + g) * a.max_chunks + chunk) * G;
  for (int i = threadIdx.x; i < G * DH; i += kAttNT) {
    const int qi = i / DH, x = i % DH;
    float M = -INFINITY;
#pragma unroll
    for (int ww = 0; ww < kAttWarps; ++ww) M = fmaxf(M, s_m[ww][qi]);
    float L = 0.f, A = 0.f;
#pragma unroll
    for (int ww = 0; ww < kAttWarps; ++ww) {
      const float f = s_m[ww][qi] == -INFINITY ? 0.f : __expf(s_m[ww][qi] - M);
      L += s_l[ww][qi] * f;
      A += s_acc[ww][qi][x] * f;
    }
    a.pacc[(pbase + qi) * DH + x] = A;
    if (x == 0) { a.pm[pbase + qi] = M; a.pl[pbase + qi] = L; }
  }
}

// One warp per (sequence, query head): combine the chunk partials.
template <int DH>
__global__ void attn_combine_kernel(AttArgs a) {
  constexpr int VPL = DH / 32;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int hq = a.h * a.G;
  if (wid >= (int64_t)a.num_seqs * hq) return;
  const int32_t s = (int32_t)(wid / hq), qh = (int32_t)(wid % hq);
  const int g = qh / a.G, qi = qh % a.G;
  const int32_t len = a.seq_len[s];
  float* o = a.out + wid * DH;
  const int nch = len <= 0 ? 0 : (len + kChunkBlocks * kBlk - 1) / (kChunkBlocks * kBlk);
  float M = -INFINITY;
  for (int c = 0; c < nch; ++c) M = fmaxf(M, a.pm[(((int64_t)s * a.h + g) * a.max_chunks + c) * a.G + qi]);
  float L = 0.f, A[VPL];
#pragma unroll
  for (int j = 0; j < VPL; ++j) A[j] = 0.f;
  for (int c = 0; c < nch; ++c) {
    const int64_t pi = (((int64_t)s * a.h + g) * a.max_chunks + c) * a.G + qi;
    const float f = __expf(a.pm[pi] - M);
    L += a.pl[pi] * f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) A[j] += a.pacc[pi * DH + lane * VPL + j] * f;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
  for (int j = 0; j < VPL; ++j) o[lane * VPL + j] = A[j] * inv;
}

}  // namespace
}  // namespace ms

using namespace ms;

extern "C" size_t memshare_kv_append_workspace_size(int32_t num_seqs) {
  if (num_seqs < 0) return 0;
  Ws w{nullptr, 0};
  app_layout(w, num_seqs);
  return w.size();
}

extern "C" memshare_status memshare_kv_append(void* k_pool, void* v_pool, int64_t layer_stride, int64_t block_stride,
                                              int32_t num_blocks, const memshare_dims* dims_host,
                                              int32_t* block_table, int32_t table_stride, int32_t num_seqs,
                                              int32_t* seq_len, const uint8_t* active, int32_t* refcount,
                                              int32_t* free_list, int64_t* free_count, const void* new_k,
                                              const void* new_v, void* workspace, size_t workspace_bytes,
                                              int32_t* device_status, void* stream) {
  if (!dims_host || num_seqs < 0 || num_blocks < 0 || table_stride < 0 || !workspace || !device_status)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  const memshare_dims d = *dims_host;
  if (d.num_layers < 1 || d.num_kv_heads_local < 1 || d.head_dim < 1 || d.block_size < 1) return MEMSHARE_ERR_INVALID_ARGUMENT;
  const int64_t row = (int64_t)d.num_kv_heads_local * d.head_dim;
  if (row % 8 != 0 || layer_stride < (int64_t)num_blocks * block_stride || block_stride < row * d.block_size)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < memshare_kv_append_workspace_size(num_seqs)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (num_seqs == 0) return MEMSHARE_OK;
  if (!k_pool || !v_pool || !block_table || !seq_len || !refcount || !free_list || !free_count || !new_k || !new_v)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (!aligned16(k_pool) || !aligned16(v_pool) || !aligned16(new_k) || !aligned16(new_v) || block_stride % 8 != 0 ||
      layer_stride % 8 != 0)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  Ws w{static_cast<char*>(workspace), 0};
  const AppWs ws = app_layout(w, num_seqs);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  append_alloc_kernel<<<1, kAppNT, 0, st>>>(block_table, table_stride, num_seqs, seq_len, active, refcount, num_blocks,
                                            free_list, free_count, d.block_size, ws, device_status);
  const int64_t work = (int64_t)d.num_layers * num_seqs * (row / 8);
  const int grid = (int)std::min<int64_t>((work + 255) / 256, 8 * sm_count());
  append_copy_kernel<<<grid, 256, 0, st>>>(static_cast<uint16_t*>(k_pool), static_cast<uint16_t*>(v_pool),
                                           layer_stride, block_stride, d.num_layers, num_seqs, (int32_t)row,
                                           static_cast<const uint16_t*>(new_k), static_cast<const uint16_t*>(new_v),
                                           ws);
  return launch_status();
}

extern "C" size_t memshare_paged_attention_workspace_size(const memshare_dims* dims_host, int32_t num_seqs,
                                                          int32_t num_q_heads, int32_t max_seq_len) {
  if (!dims_host || num_seqs < 0 || num_q_heads < 1 || max_seq_len < 0) return 0;
  const int64_t chunks = (max_seq_len + kChunkBlocks * kBlk - 1) / (kChunkBlocks * kBlk);
  const int64_t parts = (int64_t)num_seqs * num_q_heads * (chunks < 1 ? 1 : chunks);
  Ws w{nullptr, 0};
  w.take<float>(parts);
  w.take<float>(parts);
  w.take<float>(parts * dims_host->head_dim);
  return w.size();
}

extern "C" memshare_status memshare_paged_attention_decode(
    const memshare_kv_pool* pool_host, const memshare_dims* dims_host, int32_t layer, const void* q,
    int32_t num_q_heads, const int32_t* block_table, int32_t table_stride, const int32_t* seq_len, int32_t num_seqs,
    int32_t max_seq_len, float scale, float* out, void* workspace, size_t workspace_bytes, int32_t* device_status,
    void* stream) {
  if (!pool_host || !dims_host || !workspace || !device_status || num_seqs < 0 || max_seq_len < 0)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  const memshare_dims d = *dims_host;
  if (d.block_size != kBlk || (d.head_dim != 64 && d.head_dim != 128) || d.num_kv_heads_local < 1 || layer < 0 ||
      layer >= d.num_layers)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (num_q_heads < d.num_kv_heads_local || num_q_heads % d.num_kv_heads_local != 0 || num_q_heads / d.num_kv_heads_local > kMaxG)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (!(scale > 0.f) || table_stride < (max_seq_len + kBlk - 1) / kBlk) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < memshare_paged_attention_workspace_size(dims_host, num_seqs, num_q_heads, max_seq_len))
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (num_seqs == 0) return MEMSHARE_OK;
  const memshare_kv_pool p = *pool_host;
  if (!p.k || !p.v || !q || !block_table || !seq_len || !out) return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (!aligned16(p.k) || !aligned16(p.v) || p.block_stride % 8 != 0 || p.layer_stride % 8 != 0)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (num_seqs > 65535) return MEMSHARE_ERR_INVALID_ARGUMENT;
  AttArgs a{};
  a.k = static_cast<const uint16_t*>(p.k);
  a.v = static_cast<const uint16_t*>(p.v);
  a.layer_stride = p.layer_stride;
  a.block_stride = p.block_stride;
  a.layer = layer;
  a.h = d.num_kv_heads_local;
  a.G = num_q_heads / d.num_kv_heads_local;
  a.num_blocks = p.num_blocks;
  a.q = static_cast<const uint16_t*>(q);
  a.table = block_table;
  a.stride = table_stride;
  a.seq_len = seq_len;
  a.num_seqs = num_seqs;
  const int chunks = (max_seq_len + kChunkBlocks * kBlk - 1) / (kChunkBlocks * kBlk);
  a.max_chunks = chunks < 1 ? 1 : chunks;
  a.scale = scale;
  a.out = out;
  const int64_t parts = (int64_t)num_seqs * num_q_heads * a.max_chunks;
  Ws w{static_cast<char*>(workspace), 0};
  a.pm = w.take<float>(parts);
  a.pl = w.take<float>(parts);
  a.pacc = w.take<float>(parts * d.head_dim);
  a.status = device_status;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 grid(a.max_chunks, d.num_kv_heads_local, num_seqs);
  const int64_t warps = (int64_t)num_seqs * num_q_heads;
  const int cgrid = (int)((warps * 32 + 255) / 256);
  if (d.head_dim == 128) {
    attn_split_kernel<128><<<grid, kAttNT, 0, st>>>(a);
    attn_combine_kernel<128><<<cgrid, 256, 0, st>>>(a);
  } else {
    attn_split_kernel<64><<<grid, kAttNT, 0, st>>>(a);
    attn_combine_kernel<64><<<cgrid, 256, 0, st>>>(a);
  }
  return launch_status();
}

// Host-side FCFS block-budget admission (reading R37): returns the number of waiting requests
// admitted (a prefix of the queue), or -1 for invalid arguments.
extern "C" int32_t memshare_admit(const int32_t* prompt_len_host, int32_t num_waiting, int32_t reserve,
                                  int32_t block_size, int64_t free_blocks, int64_t* blocks_used_host) {
  if (num_waiting < 0 || reserve < 0 || block_size < 1 || free_blocks < 0 || (num_waiting > 0 && !prompt_len_host))
    return -1;
  int64_t used = 0;
  int32_t i = 0;
  for (; i < num_waiting; ++i) {
    if (prompt_len_host[i] < 0) return -1;
    const int64_t need = ((int64_t)prompt_len_host[i] + reserve + block_size - 1) / block_size;
    if (used + need > free_blocks) break;
    used += need;
  }
  if (blocks_used_host) *blocks_used_host = used;
  return i;
}
