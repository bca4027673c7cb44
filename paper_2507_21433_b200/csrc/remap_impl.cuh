// a7 zero-copy remap as a CTA-wide device routine, shared by remap_kernel (remap.cu, one
// 1024-thread CTA) and the fused a5-a7 call (distance.cu: the last CTA of the finalisation kernel
// to finish runs it, memshare_block_distance_remap).
// PAPER.md:276-278 ("simply updates the block table"), :283-284 (no extra GPU bandwidth);
// SPEC.md:358-366; readings R23, R26.
//
// Three phases separated by CTA barriers:
//   0. validate: canonical ascending order, ids in range -- on failure nothing is written;
//   1. apply: table[T] = new, refcount[new]++, refcount[old]--, last-decrement index per old
//      block (atomicMax);
//   2. free: decision i frees old_i iff i is old_i's last decrement and refcount[old_i] == 0;
//      freed ids are compacted in decision order (block scan) onto the free list.
// No KV byte is touched.
#pragma once
#include "common.cuh"

namespace ms {

struct RemapWs {
  int32_t* last_dec;   // [num_blocks]; entries of blocks a call decrements are reset to -1 first
  int32_t* old_of;     // [target_cap]
};

inline RemapWs remap_layout(Ws& w, int32_t num_blocks, int64_t target_cap) {
  RemapWs r;
  r.last_dec = w.take<int32_t>((size_t)num_blocks + 1);
  r.old_of = w.take<int32_t>((size_t)target_cap + 1);
  return r;
}

struct RemapArgs {
  int32_t* table;
  int32_t table_stride;
  int32_t num_seqs;
  int32_t* refcount;
  int32_t num_blocks;
  int32_t* free_list;
  int64_t* free_count;
  const memshare_decision* dec;
  const int64_t* num_targets;
  int64_t target_cap;
  int32_t block_size;
  int64_t* num_freed;
  int64_t* affected;
  RemapWs ws;
  int32_t* status;
};

// Run by all NT threads of one CTA (NT a multiple of 32, <= 1024). `sh` holds >= NT/32 + 1
// int64; `bad` is a CTA-shared flag. Decisions are read through L2 (__ldcg: the fused path reads
// decisions other CTAs wrote; the caller orders them with a fence). Each thread keeps its first
// kCache decisions (i = tid, tid + NT, ...) and their old table entries in registers across the
// phases, so a round of <= kCache x NT decisions reads every decision and table entry once.
template <int NT>
__device__ void remap_cta(const RemapArgs& r, int64_t* sh, int* bad) {
  constexpr int kCache = 4;
  const memshare_decision* dec = r.dec;
  int64_t T = __ldcg(r.num_targets);
  T = T < 0 ? 0 : (T < r.target_cap ? T : r.target_cap);
  if (threadIdx.x == 0) *bad = 0;
  __syncthreads();
  auto ld_dec = [&](int64_t i) {
    memshare_decision d;
    const int4* p = reinterpret_cast<const int4*>(dec + i);
    const int4 x = __ldcg(p), y = __ldcg(p + 1);
    d.seq = x.x; d.target_logical = x.y; d.target_phys = x.z; d.source_logical = x.w;
    d.source_phys = y.x; d.accepted = y.y; d.distance = __int_as_float(y.z); d.num_candidates = y.w;
    return d;
  };
  // what phase 1 needs of decision i: the entry's address, the new and the old physical block
  struct Item { int64_t e; int32_t nw, old; };   // e < 0: not accepted
  Item c[kCache];
  auto item = [&](int64_t i, bool check, int& err) {
    const memshare_decision d = ld_dec(i);
    Item it{-1, 0, 0};
    if (check && i > 0) {
      const int4 q = __ldcg(reinterpret_cast<const int4*>(dec + i - 1));   // (seq, target_logical) of i - 1
      if (d.seq < q.x || (d.seq == q.x && d.target_logical <= q.y)) err = MEMSHARE_ERR_INVALID_ARGUMENT;
    }
    if (d.accepted) {
      if (d.seq < 0 || d.seq >= r.num_seqs || d.target_logical < 0 || d.target_logical >= r.table_stride ||
          d.source_phys < 0 || d.source_phys >= r.num_blocks) {
        err = MEMSHARE_ERR_CORRUPTION;
      } else {
        it.e = (int64_t)d.seq * r.table_stride + d.target_logical;
        it.nw = d.source_phys;
        it.old = r.table[it.e];
        if (it.old < 0 || it.old >= r.num_blocks) err = MEMSHARE_ERR_CORRUPTION;
      }
    }
    return it;
  };
  // phase 0: validation (read-only)
  int err = 0;
#pragma unroll
  for (int k = 0; k < kCache; ++k) {
    const int64_t i = threadIdx.x + (int64_t)k * NT;
    c[k] = i < T ? item(i, true, err) : Item{-1, 0, 0};
  }
  for (int64_t i = threadIdx.x + (int64_t)kCache * NT; i < T; i += NT) item(i, true, err);
  if (err) { set_status(r.status, err); atomicExch(bad, 1); }
  __syncthreads();
  if (*bad) return;
  // reset the last-decrement slot of every block this call may decrement (no O(num_blocks) memset)
#pragma unroll
  for (int k = 0; k < kCache; ++k)
    if (c[k].e >= 0) r.ws.last_dec[c[k].old] = -1;
  for (int64_t i = threadIdx.x + (int64_t)kCache * NT; i < T; i += NT) {
    int e2 = 0;
    const Item it = item(i, false, e2);
    if (it.e >= 0) r.ws.last_dec[it.old] = -1;
  }
  __syncthreads();
  // phase 1: apply in parallel (distinct targets -> distinct table entries)
  int64_t aff = 0;
  auto apply = [&](const Item& it, int64_t i) -> int32_t {
    if (it.e < 0 || it.old == it.nw) return -1;
    r.table[it.e] = it.nw;
    atomicAdd(r.refcount + it.nw, 1);
    atomicSub(r.refcount + it.old, 1);
    atomicMax(r.ws.last_dec + it.old, (int32_t)i);
    aff += r.block_size;
    return it.old;
  };
  int32_t oc[kCache];
#pragma unroll
  for (int k = 0; k < kCache; ++k) {
    const int64_t i = threadIdx.x + (int64_t)k * NT;
    oc[k] = i < T ? apply(c[k], i) : -1;
  }
  for (int64_t i = threadIdx.x + (int64_t)kCache * NT; i < T; i += NT) {
    int e2 = 0;
    r.ws.old_of[i] = apply(item(i, false, e2), i);
  }
  aff = block_sum<NT>(aff, sh);
  __syncthreads();
  // phase 2: freed = last decrement and final count 0, compacted in decision order
  const int64_t fc0 = *r.free_count;
  int64_t carry = 0;
  int kk = 0;
  for (int64_t base = 0; base < T; base += NT, ++kk) {
    const int64_t i = base + threadIdx.x;
    int32_t o = -1;
    bool f = false;
    if (i < T) {
      if (kk < kCache) {
#pragma unroll
        for (int k = 0; k < kCache; ++k)
          if (k == kk) o = oc[k];
      } else {
        o = r.ws.old_of[i];
      }
      if (o >= 0) {
        const int32_t rc = __ldcg(r.refcount + o);
        if (rc < 0) set_status(r.status, MEMSHARE_ERR_CORRUPTION);
        f = rc == 0 && __ldcg(r.ws.last_dec + o) == (int32_t)i;
      }
    }
    int64_t tot;
    const int64_t ex = block_excl_scan<NT>(f ? 1 : 0, tot, sh);
    if (f) {
      const int64_t pos = fc0 + carry + ex;
      if (pos < r.num_blocks) r.free_list[pos] = o;
      else set_status(r.status, MEMSHARE_ERR_CORRUPTION);
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    *r.num_freed = carry;
    *r.free_count = fc0 + carry;
    *r.affected = aff;
  }
}

// host-side argument check shared by memshare_remap and the fused call
inline bool remap_args_ok(const int32_t* block_table, int32_t table_stride, int32_t num_seqs, const int32_t* refcount,
                          int32_t num_blocks, const int32_t* free_list, const int64_t* free_count,
                          const int64_t* num_freed, const int64_t* affected, int32_t block_size) {
  if (!block_table || !refcount || !free_list || !free_count || !num_freed || !affected) return false;
  return table_stride >= 0 && num_seqs >= 0 && num_blocks >= 0 && block_size >= 1;
}

}  // namespace ms
