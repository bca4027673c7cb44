// a7 -- zero-copy remap: block-table rewrite, refcounts, free list.
// PAPER.md:276-278 ("simply updates the block table"), :283-284 (no extra GPU bandwidth);
// SPEC.md:358-366; readings R23, R26.
//
// One CTA of 1024 threads (the decision count of a round is small; the whole update is a few
// thousand integer atomics), three phases separated by CTA barriers:
//   0. validate: canonical ascending order, ids in range -- on failure nothing is written;
//   1. apply: table[T] = new, refcount[new]++, refcount[old]--, last-decrement index per old
//      block (atomicMax);
//   2. free: decision i frees old_i iff i is old_i's last decrement and refcount[old_i] == 0;
//      freed ids are compacted in decision order (block scan) onto the free list.
// No KV byte is touched.
#include "common.cuh"

namespace ms {
namespace {

constexpr int kNT = 1024;

struct RemapWs {
  int32_t* last_dec;   // [num_blocks]; entries of blocks a call decrements are reset to -1 first
  int32_t* old_of;     // [target_cap]
};

RemapWs remap_layout(Ws& w, int32_t num_blocks, int64_t target_cap) {
  RemapWs r;
  r.last_dec = w.take<int32_t>((size_t)num_blocks + 1);
  r.old_of = w.take<int32_t>((size_t)target_cap + 1);
  return r;
}

__global__ void __launch_bounds__(kNT) remap_kernel(int32_t* __restrict__ table, int32_t table_stride, int32_t num_seqs,
                                                    int32_t* __restrict__ refcount, int32_t num_blocks,
                                                    int32_t* __restrict__ free_list, int64_t* __restrict__ free_count,
                                                    const memshare_decision* __restrict__ dec,
                                                    const int64_t* __restrict__ num_targets, int64_t target_cap,
                                                    int32_t block_size, int64_t* __restrict__ num_freed,
                                                    int64_t* __restrict__ affected, RemapWs ws, int32_t* status) {
  pdl_trigger();
  TL_SCOPE(8);
  __shared__ int64_t sh[kNT / 32 + 1];
  __shared__ int bad;
  int64_t T = *num_targets;
  T = T < 0 ? 0 : (T < target_cap ? T : target_cap);
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  // phase 0: validation (read-only)
  for (int64_t i = threadIdx.x; i < T; i += kNT) {
    const memshare_decision d = dec[i];
    int err = 0;
    if (i > 0) {
      const memshare_decision q = dec[i - 1];
      if (d.seq < q.seq || (d.seq == q.seq && d.target_logical <= q.target_logical)) err = MEMSHARE_ERR_INVALID_ARGUMENT;
    }
    if (d.accepted) {
      if (d.seq < 0 || d.seq >= num_seqs || d.target_logical < 0 || d.target_logical >= table_stride ||
          d.source_phys < 0 || d.source_phys >= num_blocks)
        err = MEMSHARE_ERR_CORRUPTION;
      else {
        const int32_t old = table[(int64_t)d.seq * table_stride + d.target_logical];
        if (old < 0 || old >= num_blocks) err = MEMSHARE_ERR_CORRUPTION;
      }
    }
    if (err) { set_status(status, err); atomicExch(&bad, 1); }
  }
  __syncthreads();
  if (bad) return;
  // reset the last-decrement slot of every block this call may decrement (no O(num_blocks) memset)
  for (int64_t i = threadIdx.x; i < T; i += kNT) {
    const memshare_decision d = dec[i];
    if (d.accepted) ws.last_dec[table[(int64_t)d.seq * table_stride + d.target_logical]] = -1;
  }
  __syncthreads();
  // phase 1: apply in parallel (distinct targets -> distinct table entries)
  int64_t aff = 0;
  for (int64_t i = threadIdx.x; i < T; i += kNT) {
    const memshare_decision d = dec[i];
    int32_t o = -1;
    if (d.accepted) {
      int32_t* e = table + (int64_t)d.seq * table_stride + d.target_logical;
      const int32_t old = *e, nw = d.source_phys;
      if (old != nw) {
        *e = nw;
        atomicAdd(refcount + nw, 1);
        atomicSub(refcount + old, 1);
        atomicMax(ws.last_dec + old, (int32_t)i);
        o = old;
        aff += block_size;
      }
    }
    ws.old_of[i] = o;
  }
  aff = block_sum<kNT>(aff, sh);
  __syncthreads();
  // phase 2: freed = last decrement and final count 0, compacted in decision order
  const int64_t fc0 = *free_count;
  int64_t carry = 0;
  for (int64_t base = 0; base < T; base += kNT) {
    const int64_t i = base + threadIdx.x;
    int32_t o = -1;
    bool f = false;
    if (i < T) {
      o = ws.old_of[i];
      if (o >= 0) {
        const int32_t rc = __ldcg(refcount + o);
        if (rc < 0) set_status(status, MEMSHARE_ERR_CORRUPTION);
        f = rc == 0 && __ldcg(ws.last_dec + o) == (int32_t)i;
      }
    }
    int64_t tot;
    const int64_t ex = block_excl_scan<kNT>(f ? 1 : 0, tot, sh);
    if (f) {
      const int64_t pos = fc0 + carry + ex;
      if (pos < num_blocks) free_list[pos] = o;
      else set_status(status, MEMSHARE_ERR_CORRUPTION);
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    *num_freed = carry;
    *free_count = fc0 + carry;
    *affected = aff;
  }
}

}  // namespace
}  // namespace ms

using namespace ms;

TL_EXPORT(remap)

extern "C" size_t memshare_remap_workspace_size(int32_t num_blocks, int64_t target_cap) {
  if (num_blocks < 0 || target_cap < 0) return 0;
  Ws w{nullptr, 0};
  remap_layout(w, num_blocks, target_cap);
  return w.size();
}

extern "C" memshare_status memshare_remap(int32_t* block_table, int32_t table_stride, int32_t num_seqs,
                                          int32_t* refcount, int32_t num_blocks, int32_t* free_list,
                                          int64_t* free_count, const memshare_decision* decisions,
                                          const int64_t* num_targets, int64_t target_cap, int32_t block_size,
                                          int64_t* num_freed, int64_t* affected_tokens, void* workspace,
                                          size_t workspace_bytes, int32_t* device_status, void* stream) {
  if (!block_table || !refcount || !free_list || !free_count || !decisions || !num_targets || !num_freed ||
      !affected_tokens || !workspace || !device_status)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (table_stride < 0 || num_seqs < 0 || num_blocks < 0 || target_cap < 0 || block_size < 1)
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < memshare_remap_workspace_size(num_blocks, target_cap)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  Ws w{static_cast<char*>(workspace), 0};
  RemapWs ws = remap_layout(w, num_blocks, target_cap);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  launch_pdl(remap_kernel, dim3(1), dim3(kNT), 0, st, block_table, table_stride, num_seqs, refcount, num_blocks, free_list, free_count,
                                  decisions, num_targets, target_cap, block_size, num_freed, affected_tokens, ws,
                                  device_status);
  return launch_status();
}

extern "C" const char* memshare_status_string(memshare_status s) {
  switch (s) {
    case MEMSHARE_OK: return "MEMSHARE_OK";
    case MEMSHARE_ERR_INVALID_ARGUMENT: return "MEMSHARE_ERR_INVALID_ARGUMENT";
    case MEMSHARE_ERR_CAPACITY: return "MEMSHARE_ERR_CAPACITY";
    case MEMSHARE_ERR_CORRUPTION: return "MEMSHARE_ERR_CORRUPTION";
    case MEMSHARE_ERR_CUDA: return "MEMSHARE_ERR_CUDA";
    default: return "MEMSHARE_ERR_UNKNOWN";
  }
}

extern "C" int32_t memshare_abi_version(void) { return MEMSHARE_ABI_VERSION; }
