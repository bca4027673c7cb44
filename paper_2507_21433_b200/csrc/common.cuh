// Shared device helpers of the CUDA path (sm_100a). Nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <cstddef>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost a pointer test unless a tool is attached

#include "memshare.h"

namespace ms {

constexpr int kWarp = 32;

struct Delims {
  int32_t n;
  int32_t id[MEMSHARE_MAX_DELIMS];
};

__device__ __forceinline__ bool is_delim(int32_t t, const Delims& d) {
  if (t == d.id[0]) return true;            // the common single-delimiter case: one compare
  for (int i = 1; i < d.n; ++i)
    if (t == d.id[i]) return true;
  return false;
}

// Sticky first-error device status (first writer wins).
__device__ __forceinline__ void set_status(int32_t* st, int32_t code) {
  if (st != nullptr) atomicCAS(st, 0, code);
}

// Bound on a cross-CTA spin-wait (a flag another CTA publishes). Work is handed out by atomic
// tickets, so every wait is on a CTA that is already running and the bound is never reached in a
// correct run; if it is (a bug, a corrupted workspace), the waiter reports CORRUPTION and moves on
// instead of hanging the device. The clock is read only every 1024 polls.
struct SpinGuard {
  unsigned long long t0 = 0;
  uint32_t n = 0;
  static constexpr unsigned long long kLimitNs = 2000000000ull;   // 2 s
  __device__ __forceinline__ bool expired() {
    if ((++n & 1023u) != 0u) return false;
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (t0 == 0) { t0 = t; return false; }
    return t - t0 > kLimitNs;
  }
};

// Bump allocator over the caller's workspace; the same sequence of take() calls in
// "measure" mode (base == nullptr) gives the required size.
struct Ws {
  char* base;
  size_t off;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
  size_t size() const { return (off + 255) & ~size_t(255); }
};

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan of int64; `sh` must hold >= NT/32 + 1 entries. Returns the
// exclusive prefix of this thread, writes the block total to `total`.
template <int NT>
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t& total, int64_t* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t s = lane < NT / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) sh[lane] = s;   // inclusive warp totals
  }
  __syncthreads();
  const int64_t warp_prefix = w > 0 ? sh[w - 1] : 0;
  total = sh[NT / 32 - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

template <int NT>
__device__ __forceinline__ int64_t block_sum(int64_t v, int64_t* sh) {
  int64_t t;
  block_excl_scan<NT>(v, t, sh);
  return t;
}

// "Last CTA done" election for fused count -> scan kernels. All threads call it. The CTA's writes
// are ordered before the counter update by the barrier plus ONE cumulative gpu-scope fence in the
// electing thread (not a fence in every thread: that is a MEMBAR + L1 invalidate per thread).
__device__ __forceinline__ bool last_block_done(unsigned int* ctr) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(ctr, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// Exclusive scan of a device array of `n` int32 counts into int64 offsets by ONE CTA.
// out_off[n] receives the total. Reads bypass L1 (values written by other CTAs).
template <int NT>
__device__ void cta_scan_counts(const int32_t* cnt, int64_t* out_off, int64_t n, int64_t* sh) {
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += NT) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < n ? (int64_t)__ldcg(cnt + i) : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan<NT>(v, tot, sh);
    if (i < n) out_off[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) out_off[n] = carry;
}

// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel of the path is launched with programmatic stream serialization (PDL): the next
// kernel's CTAs may be scheduled while the previous kernel drains, and each kernel calls
// pdl_wait() (griddepcontrol.wait: the predecessor grid has completed and its writes are
// visible) before it touches any memory another kernel wrote or reads. pdl_trigger()
// (griddepcontrol.launch_dependents) lets the successor launch early. Both are no-ops when the
// kernel was launched without the attribute. MEMSHARE_PDL=0 disables the attribute (A/B).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Tuning only (-DMS_TIMELINE variant library): per-kernel device timestamps of one round --
// [id][0] first CTA resident, [id][1] first CTA past its dependency wait, [id][2] last CTA done
// (globaltimer ns); read with memshare_debug_tl_<file>(). No effect in the shipped library.
#ifdef MS_TIMELINE
static __device__ unsigned long long ms_tl[16][4];
__device__ __forceinline__ unsigned long long ms_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TL_WAIT(id)                                                       \
  do {                                                                    \
    if (threadIdx.x == 0) atomicMin(&::ms::ms_tl[id][0], ::ms::ms_gtime()); \
    ::ms::pdl_wait();                                                     \
    if (threadIdx.x == 0) atomicMin(&::ms::ms_tl[id][1], ::ms::ms_gtime()); \
  } while (0)
#define TL_END(id)                                                        \
  do {                                                                    \
    if (threadIdx.x == 0) atomicMax(&::ms::ms_tl[id][2], ::ms::ms_gtime()); \
  } while (0)
struct TlGuard {
  int id;
  __device__ ~TlGuard() { TL_END(id); }
};
#define TL_SCOPE(id) TL_WAIT(id); ::ms::TlGuard _ms_tl_guard{id}
#define TL_EXPORT(name)                                                                         \
  extern "C" int memshare_debug_tl_##name(unsigned long long* host, int reset) {               \
    int e = (int)cudaMemcpyFromSymbol(host, ::ms::ms_tl, sizeof(::ms::ms_tl));                 \
    if (reset) {                                                                                \
      unsigned long long init[16][4];                                                           \
      for (int i = 0; i < 16; ++i) { init[i][0] = init[i][1] = ~0ull; init[i][2] = init[i][3] = 0ull; } \
      e |= (int)cudaMemcpyToSymbol(::ms::ms_tl, init, sizeof(init));                            \
    }                                                                                           \
    return e;                                                                                   \
  }
#else
#define TL_WAIT(id) ::ms::pdl_wait()
#define TL_END(id) do { } while (0)
#define TL_SCOPE(id) ::ms::pdl_wait()
#define TL_EXPORT(name)
#endif

inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MEMSHARE_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Per-device state: kernel attributes (cudaFuncSetAttribute) and device properties are per
// device, so a process driving several GPUs sets them once on each.
constexpr int kMaxDevices = 64;

inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < kMaxDevices ? dev : 0;
}

inline int sm_count() {
  static int cached[kMaxDevices] = {};
  const int dev = current_device();
  if (cached[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

// Tracing: every ABI call is an NVTX range named after it (host side: the
// enqueue, and the call's place in an Nsight Systems timeline / a CUDA-graph capture).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define MS_NVTX(name) ::ms::NvtxRange ms_nvtx_range_(name)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline memshare_status launch_status() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MEMSHARE_OK : MEMSHARE_ERR_CUDA;
}

}  // namespace ms
