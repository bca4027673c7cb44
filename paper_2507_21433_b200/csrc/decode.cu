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
  // wait first, then let the copy kernel launch: it reads the new rows before its own wait, so
  // everything earlier on the stream (whoever wrote new_k / new_v) must be complete by then
  pdl_wait();
  pdl_trigger();
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

// Copy the new K/V rows (h * d_h bf16 each, one per (layer, sequence)) into their slots. A warp
// moves one row per iteration (16-byte vectors, K and V loads issued together, 32-bit index
// math: the row index is split once per row, not per vector). The first row of each warp is
// loaded BEFORE the grid-dependency wait (the new rows are inputs, not written by the alloc
// kernel), so those HBM reads overlap the allocation; only the destination waits for it.
__global__ void __launch_bounds__(256) append_copy_kernel(uint16_t* k, uint16_t* v, int64_t layer_stride,
                                                          int64_t block_stride, int32_t num_layers, int32_t num_seqs,
                                                          int32_t row_elems, const uint16_t* new_k,
                                                          const uint16_t* new_v, AppWs ws) {
  constexpr int kPre = 4;                        // 16-byte vectors per lane preloaded (rows <= 2 KiB per K|V)
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int32_t vec = row_elems / 8;             // 16-byte vectors per row
  const int32_t rows = num_layers * num_seqs;
  const int32_t warps = (int32_t)(gridDim.x * (blockDim.x / 32));
  const int32_t r0 = (int32_t)(blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5));
  uint4 pk[kPre], pv[kPre];
  const bool pre = r0 < rows && vec <= 32 * kPre;
  if (pre) {
    const uint4* sk = reinterpret_cast<const uint4*>(new_k + (int64_t)r0 * row_elems);
    const uint4* sv = reinterpret_cast<const uint4*>(new_v + (int64_t)r0 * row_elems);
#pragma unroll
    for (int i = 0; i < kPre; ++i) {
      const int32_t c = lane + 32 * i;
      if (c < vec) { pk[i] = __ldg(sk + c); pv[i] = __ldg(sv + c); }
    }
  }
  pdl_wait();
  if (__ldcg(ws.ok) == 0) return;
  if (pre) {
    const int32_t l = r0 / num_seqs, s = r0 - l * num_seqs;
    const int32_t b = __ldcg(ws.slot_blk + s);
    if (b >= 0) {
      const int64_t dst = (int64_t)l * layer_stride + (int64_t)b * block_stride +
                          (int64_t)__ldcg(ws.slot_off + s) * row_elems;
      uint4* dk = reinterpret_cast<uint4*>(k + dst);
      uint4* dv = reinterpret_cast<uint4*>(v + dst);
#pragma unroll
      for (int i = 0; i < kPre; ++i) {
        const int32_t c = lane + 32 * i;
        if (c < vec) { dk[c] = pk[i]; dv[c] = pv[i]; }
      }
    }
  }
  for (int32_t r = pre ? r0 + warps : r0; r < rows; r += warps) {
    const int32_t l = r / num_seqs, s = r - l * num_seqs;
    const int32_t b = __ldcg(ws.slot_blk + s);
    if (b < 0) continue;
    const int64_t dst = (int64_t)l * layer_stride + (int64_t)b * block_stride + (int64_t)__ldcg(ws.slot_off + s) * row_elems;
    const uint4* sk = reinterpret_cast<const uint4*>(new_k + (int64_t)r * row_elems);
    const uint4* sv = reinterpret_cast<const uint4*>(new_v + (int64_t)r * row_elems);
    uint4* dk = reinterpret_cast<uint4*>(k + dst);
    uint4* dv = reinterpret_cast<uint4*>(v + dst);
    for (int32_t c = lane; c < vec; c += 32) {
      const uint4 xk = __ldg(sk + c), xv = __ldg(sv + c);
      dk[c] = xk;
      dv[c] = xv;
    }
  }
}

// ------------------------------------------------------------------ paged decode attention
constexpr int kBlk = 16;               // tokens per KV block (the lane mapping assumes 16)
// Blocks per CTA work item: chosen per call on the host (attn_chunk_blocks) from {64, 32, 16} --
// the largest that still gives the split grid >= 4 CTAs per SM. 64 blocks (1,024 tokens) per
// item: f1 row 230 -> 204 us (0.85 -> 0.96 of HBM; each warp's cp.async pipeline prologue is
// amortised over 16 blocks instead of 4 and the combine reads a quarter of the partials).
constexpr int kChunkBlocksMin = 16;
constexpr int kAttWarps = 4;
constexpr int kAttNT = kAttWarps * 32;
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
  int32_t cb;         // blocks per chunk (work item)
  int32_t max_len;    // min(max_seq_len, table_stride * block): the grid and the partials are sized by it
  float scale;
  float* out;
  float* pm;          // [S][h][max_chunks][G]
  float* pl;
  float* pacc;        // [S][h][max_chunks][G][d_h]
  int32_t* status;
};

// ---- tensor-core building blocks (mma.sync m16n8k16 bf16 -> fp32, ldmatrix, cp.async) ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;                     // src-size 0: zero-fill (rows past the sequence end)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D (fp32)
__device__ __forceinline__ void mma_bf16(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf16_lo(uint32_t x) { return __uint_as_float(x << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t x) { return __uint_as_float(x & 0xFFFF0000u); }

// One CTA per (256-token chunk, KV head g, sequence s); warp w handles blocks w, w+4, w+8, w+12
// of the chunk. Per 16-token block and KV head, the K and V rows (16 x d_h bf16 each) are staged
// in XOR-swizzled smem by cp.async (double-buffered per warp) and both contractions run on the
// tensor cores (mma.sync m16n8k16, fp32 accumulate):
//   S   = Q K^T   A = Q (the G <= 8 query heads of g, zero-padded to 16 rows, in registers),
//                 B = K rows via ldmatrix; C rows = query heads, cols = tokens
//   O^T += V^T P^T  A = V^T via ldmatrix.trans, B = P taken straight from S's C fragments,
//                 split into bf16 hi + lo parts (two MMAs: ~16-bit P keeps the result within
//                 fp32-accumulation error of the fp64 oracle); C rows = dims, cols = query heads
// with an fp32 online softmax in between (row statistics per query head).
// a seq_len beyond the host max_seq_len (or the table row) would index partials / table entries
// that were never sized: clamp it and report INVALID_ARGUMENT (one reporter per sequence)
__device__ __forceinline__ int32_t clamp_len(const AttArgs& a, int32_t len, bool report) {
  if (len > a.max_len) {
    if (report) set_status(a.status, MEMSHARE_ERR_INVALID_ARGUMENT);
    return a.max_len;
  }
  return len < 0 ? 0 : len;
}

template <int DH>
__global__ void __launch_bounds__(kAttNT) attn_split_kernel(AttArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int KS = DH / 16;                 // k-steps of Q K^T
  constexpr int MT = DH / 16;                 // m-tiles (16 dims) of O^T
  constexpr int CH = DH / 8;                  // 16-byte chunks per row
  constexpr int ROWB = DH * 2;                // bytes per K/V row in smem
  constexpr int TILE = kBlk * ROWB;           // one K or V tile
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* s_kv = smem;                                        // [warp][stage][K|V][TILE]
  float* s_acc = reinterpret_cast<float*>(smem);                     // [warp][kMaxG][DH], after the loop
  __shared__ float s_m[kAttWarps][kMaxG], s_l[kAttWarps][kMaxG];
  const int chunk = blockIdx.x, g = blockIdx.y, s = blockIdx.z;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int G = a.G;
  const int32_t len = clamp_len(a, a.seq_len[s], chunk == 0 && g == 0 && threadIdx.x == 0);
  const int32_t tok0 = chunk * a.cb * kBlk;
  if (tok0 >= len) return;
  const int r0 = lane >> 2, c2 = 2 * (lane & 3);
  // Q as A fragments (rows = query heads of g; rows >= G and rows 8..15 are zero)
  uint32_t qa0[KS], qa2[KS];
  {
    const uint16_t* qb = a.q + ((int64_t)s * a.h * G + (int64_t)g * G) * DH;
    const bool v0 = r0 < G;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      const int c = kk * 16 + c2;
      qa0[kk] = v0 ? *reinterpret_cast<const uint32_t*>(qb + r0 * DH + c) : 0u;
      qa2[kk] = v0 ? *reinterpret_cast<const uint32_t*>(qb + r0 * DH + c + 8) : 0u;
    }
  }
  float o[MT][4];                              // O^T: rows dims mt*16 + r0 (+8), cols q = c2 (+1)
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
  float m_r = -INFINITY, l_r = 0.f;           // softmax statistics of query head r0
  const int32_t* trow = a.table + (int64_t)s * a.stride;
  const uint16_t* kl = a.k + (int64_t)a.layer * a.layer_stride + g * DH;
  const uint16_t* vl = a.v + (int64_t)a.layer * a.layer_stride + g * DH;
  const int64_t row = (int64_t)a.h * DH;
  const int32_t nblk_seq = (len + kBlk - 1) / kBlk;
  bool bad = false;
  auto tile = [&](int st, int kv) { return smem_addr(s_kv + (((w * 2 + st) * 2 + kv) * TILE)); };
  auto issue = [&](int bi, int st) -> bool {
    const int32_t lb = chunk * a.cb + w + bi * kAttWarps;
    if (bi * kAttWarps >= a.cb || lb >= nblk_seq) return false;
    const int32_t blk = trow[lb];
    if (blk < 0 || blk >= a.num_blocks) { bad = true; return false; }
    const int ntok = min(kBlk, len - lb * kBlk);
    const uint16_t* kb = kl + (int64_t)blk * a.block_stride;
    const uint16_t* vb = vl + (int64_t)blk * a.block_stride;
    const uint32_t sk = tile(st, 0), sv = tile(st, 1);
#pragma unroll
    for (int i = 0; i < (kBlk * CH) / 32; ++i) {
      const int id = lane + 32 * i, t = id / CH, c = id % CH;
      const uint32_t off = t * ROWB + ((c ^ (t & 7)) << 4);
      cp_async16(sk + off, kb + t * row + c * 8, t < ntok);
      cp_async16(sv + off, vb + t * row + c * 8, t < ntok);
    }
    return true;
  };
  const uint32_t zero = 0u;
  bool have = issue(0, 0);
  cp_async_commit();
  for (int bi = 0; have; ++bi) {
    const int st = bi & 1;
    const bool next = issue(bi + 1, st ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const int32_t lb = chunk * a.cb + w + bi * kAttWarps;
    const int ntok = min(kBlk, len - lb * kBlk);
    const uint32_t sk = tile(st, 0), sv = tile(st, 1);
    // S = Q K^T, two n-tiles of 8 tokens
    float sc[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < KS; kk += 2) {
        const int t = nt * 8 + (lane & 7), c = kk * 2 + (lane >> 3);     // 4 matrices: 2 k-steps
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sk + t * ROWB + ((c ^ (t & 7)) << 4), b0, b1, b2, b3);
        mma_bf16(sc[nt], qa0[kk], zero, qa2[kk], zero, b0, b1);
        mma_bf16(sc[nt], qa0[kk + 1], zero, qa2[kk + 1], zero, b2, b3);
      }
    }
    // online softmax of query head r0 over this block's tokens
    float mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int t = nt * 8 + c2 + j;
        sc[nt][j] = t < ntok ? sc[nt][j] * a.scale : -INFINITY;
        mx = fmaxf(mx, sc[nt][j]);
      }
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mn = fmaxf(m_r, mx);
    const float corr = __expf(m_r - mn);
    m_r = mn;
    float p[2][2], ps = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j) { p[nt][j] = __expf(sc[nt][j] - mn); ps += p[nt][j]; }
    l_r = l_r * corr + ps;
    // O^T columns are query heads c2, c2 + 1: their rescale factors live in lanes 4*c2, 4*(c2+1)
    const float cq0 = __shfl_sync(0xffffffffu, corr, 4 * c2), cq1 = __shfl_sync(0xffffffffu, corr, 4 * (c2 + 1));
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) { o[mt][0] *= cq0; o[mt][1] *= cq1; o[mt][2] *= cq0; o[mt][3] *= cq1; }
    // P^T as B fragments: (k = token, n = query head) = S C fragments of the two n-tiles
    const uint32_t bh0 = pack_bf16(p[0][0], p[0][1]), bh1 = pack_bf16(p[1][0], p[1][1]);
    const uint32_t bl0 = pack_bf16(p[0][0] - bf16_lo(bh0), p[0][1] - bf16_hi(bh0));
    const uint32_t bl1 = pack_bf16(p[1][0] - bf16_lo(bh1), p[1][1] - bf16_hi(bh1));
    // O^T += V^T P^T; V^T fragments via ldmatrix.trans of the [token][dim] rows
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int mi = lane >> 3, t = (mi >> 1) * 8 + (lane & 7), c = mt * 2 + (mi & 1);
      uint32_t a0, a1, a2, a3;
      ldsm_x4_t(sv + t * ROWB + ((c ^ (t & 7)) << 4), a0, a1, a2, a3);
      mma_bf16(o[mt], a0, a1, a2, a3, bh0, bh1);
      mma_bf16(o[mt], a0, a1, a2, a3, bl0, bl1);
    }
    __syncwarp();
    have = next;
  }
  cp_async_wait<0>();
  if (bad) set_status(a.status, MEMSHARE_ERR_CORRUPTION);
  l_r += __shfl_xor_sync(0xffffffffu, l_r, 1);
  l_r += __shfl_xor_sync(0xffffffffu, l_r, 2);
  __syncthreads();                            // the K/V stages become s_acc
  if ((lane & 3) == 0 && r0 < kMaxG) { s_m[w][r0] = m_r; s_l[w][r0] = l_r; }
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int q = c2 + j;
      if (q < G) {
        s_acc[(w * kMaxG + q) * DH + mt * 16 + r0] = o[mt][j];
        s_acc[(w * kMaxG + q) * DH + mt * 16 + r0 + 8] = o[mt][2 + j];
      }
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
      A += s_acc[(ww * kMaxG + qi) * DH + x] * f;
    }
    a.pacc[(pbase + qi) * DH + x] = A;
    if (x == 0) { a.pm[pbase + qi] = M; a.pl[pbase + qi] = L; }
  }
}

template <int DH>
constexpr size_t attn_smem_bytes() {
  const size_t kv = (size_t)kAttWarps * 2 * 2 * kBlk * DH * 2;
  const size_t acc = (size_t)kAttWarps * kMaxG * DH * 4;
  return kv > acc ? kv : acc;
}

// One warp per (sequence, query head): combine the chunk partials.
template <int DH>
__global__ void attn_combine_kernel(AttArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int VPL = DH / 32;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int hq = a.h * a.G;
  if (wid >= (int64_t)a.num_seqs * hq) return;
  const int32_t s = (int32_t)(wid / hq), qh = (int32_t)(wid % hq);
  const int g = qh / a.G, qi = qh % a.G;
  const int32_t len = clamp_len(a, a.seq_len[s], false);
  float* o = a.out + wid * DH;
  const int nch = len <= 0 ? 0 : (len + a.cb * kBlk - 1) / (a.cb * kBlk);
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
  MS_NVTX("memshare_kv_append");
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
  launch_pdl(append_alloc_kernel, dim3(1), dim3(kAppNT), 0, st, block_table, table_stride, num_seqs, seq_len, active, refcount, num_blocks,
                                            free_list, free_count, d.block_size, ws, device_status);
  const int64_t rows = (int64_t)d.num_layers * num_seqs;
  if (rows > INT32_MAX) return MEMSHARE_ERR_INVALID_ARGUMENT;
  const int grid = (int)std::min<int64_t>((rows + 7) / 8, 8 * sm_count());    // 8 warps (rows) per CTA
  launch_pdl(append_copy_kernel, dim3(grid), dim3(256), 0, st, static_cast<uint16_t*>(k_pool), static_cast<uint16_t*>(v_pool),
                                           layer_stride, block_stride, d.num_layers, num_seqs, (int32_t)row,
                                           static_cast<const uint16_t*>(new_k), static_cast<const uint16_t*>(new_v),
                                           ws);
  return launch_status();
}

namespace ms {
namespace {
// the largest work item in {64, 32, 16} blocks whose split grid has >= 4 CTAs per SM
int attn_chunk_blocks(int32_t max_seq_len, int32_t h, int32_t num_seqs) {
  for (int cb = 64; cb > kChunkBlocksMin; cb /= 2) {
    const int64_t ch = ((int64_t)max_seq_len + cb * kBlk - 1) / (cb * kBlk);
    if (ch * h * num_seqs >= 4LL * sm_count()) return cb;
  }
  return kChunkBlocksMin;
}
}  // namespace
}  // namespace ms

extern "C" size_t memshare_paged_attention_workspace_size(const memshare_dims* dims_host, int32_t num_seqs,
                                                          int32_t num_q_heads, int32_t max_seq_len) {
  if (!dims_host || num_seqs < 0 || num_q_heads < 1 || max_seq_len < 0) return 0;
  // sized for the smallest work item (any chunk choice fits)
  const int64_t chunks = (max_seq_len + kChunkBlocksMin * kBlk - 1) / (kChunkBlocksMin * kBlk);
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
  MS_NVTX("memshare_paged_attention_decode");
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
  a.cb = attn_chunk_blocks(max_seq_len, d.num_kv_heads_local, num_seqs);
  const int chunks = (max_seq_len + a.cb * kBlk - 1) / (a.cb * kBlk);
  a.max_chunks = chunks < 1 ? 1 : chunks;
  {
    const int64_t row = (int64_t)table_stride * kBlk;
    a.max_len = row < (int64_t)max_seq_len ? (int32_t)row : max_seq_len;
  }
  a.scale = scale;
  a.out = out;
  const int64_t parts = (int64_t)num_seqs * num_q_heads * a.max_chunks;
  Ws w{static_cast<char*>(workspace), 0};
  a.pm = w.take<float>(parts);
  a.pl = w.take<float>(parts);
  a.pacc = w.take<float>(parts * d.head_dim);
  a.status = device_status;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static bool attr_set_dev[kMaxDevices] = {};
  bool& attr_set = attr_set_dev[current_device()];
  if (!attr_set) {
    cudaFuncSetAttribute(attn_split_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)attn_smem_bytes<128>());
    cudaFuncSetAttribute(attn_split_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)attn_smem_bytes<64>());
    attr_set = true;
  }
  const dim3 grid(a.max_chunks, d.num_kv_heads_local, num_seqs);
  const int64_t warps = (int64_t)num_seqs * num_q_heads;
  const int cgrid = (int)((warps * 32 + 255) / 256);
  if (d.head_dim == 128) {
    launch_pdl(attn_split_kernel<128>, grid, dim3(kAttNT), attn_smem_bytes<128>(), st, a);
    launch_pdl(attn_combine_kernel<128>, dim3(cgrid), dim3(256), 0, st, a);
  } else {
    launch_pdl(attn_split_kernel<64>, grid, dim3(kAttNT), attn_smem_bytes<64>(), st, a);
    launch_pdl(attn_combine_kernel<64>, dim3(cgrid), dim3(256), 0, st, a);
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
