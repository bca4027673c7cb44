// a7 -- zero-copy remap: block-table rewrite, refcounts, free list.
// PAPER.md:276-278 ("simply updates the block table"), :283-284 (no extra GPU bandwidth);
// SPEC.md:358-366; readings R23, R26.
//
// One CTA of 1024 threads runs the CTA-wide routine of remap_impl.cuh (the decision count of a
// round is small; the whole update is a few thousand integer atomics).
#include "remap_impl.cuh"

namespace ms {
namespace {

constexpr int kNT = 1024;

__global__ void __launch_bounds__(kNT) remap_kernel(RemapArgs r) {
  pdl_trigger();
  TL_SCOPE(8);
  __shared__ int64_t sh[kNT / 32 + 1];
  __shared__ int bad;
  remap_cta<kNT>(r, sh, &bad);
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
  MS_NVTX("memshare_remap");
  if (!decisions || !num_targets || !workspace || !device_status || target_cap < 0 ||
      !remap_args_ok(block_table, table_stride, num_seqs, refcount, num_blocks, free_list, free_count, num_freed,
                     affected_tokens, block_size))
    return MEMSHARE_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < memshare_remap_workspace_size(num_blocks, target_cap)) return MEMSHARE_ERR_INVALID_ARGUMENT;
  Ws w{static_cast<char*>(workspace), 0};
  const RemapArgs r{block_table, table_stride, num_seqs, refcount, num_blocks, free_list, free_count, decisions,
                    num_targets, target_cap, block_size, num_freed, affected_tokens,
                    remap_layout(w, num_blocks, target_cap), device_status};
  launch_pdl(remap_kernel, dim3(1), dim3(kNT), 0, static_cast<cudaStream_t>(stream), r);
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
