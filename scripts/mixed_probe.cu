// Tuning probe (not part of the product): can L2-resident re-reads go through the LSU path
// (cp.async 16-byte LDGSTS issued by the producer warp, completion by cp.async.mbarrier.arrive)
// while HBM slices stream through the TMA unit, and do the two overlap?
// Ring of 32 KiB stages (1 CTA per SM, one producer warp, 8 consumer warps that read one word
// and release). Stage k of a CTA is an HBM slice (4 GiB source) when (k % M) < H, else an
// L2-resident slice (32 MiB source), copied by TMA (route 0) or by LDGSTS (route 1), or every
// other L2 slice by LDGSTS (route 2).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mixed_probe mixed_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kSlice = 32768;
constexpr int kStages = 7;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                   smem_u32(b)),
               "r"(ph)
               : "memory");
}

__global__ void __launch_bounds__(288, 1) mixed(const uint8_t* hbm, size_t n_hbm, const uint8_t* l2, size_t n_l2,
                                                int H, int M, int route, size_t stages_total, float* sink, int consume, unsigned long long mult) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  uint8_t* data = sm + 1024;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 8) {
    if (route == 0 && lane != 0) return;               // all-TMA: one producer lane, as tma_sweep.cu
    int st = 0;
    uint32_t ph = 0;
    int nl2 = 0;
    for (size_t i = blockIdx.x, k = 0; i < stages_total; i += gridDim.x, ++k) {
      // lean address math (power-of-two slice counts: a mask, no 64-bit modulo)
      const bool from_hbm = (int)(k % M) < H;
      const uint8_t* src = from_hbm ? hbm + (size_t)((uint32_t)(i * 7919u) & (uint32_t)(n_hbm - 1)) * kSlice
                                    : l2 + (size_t)((uint32_t)(i * (uint32_t)mult) & (uint32_t)(n_l2 - 1)) * kSlice;
      const bool lsu = !from_hbm && (route == 1 || (route == 2 && (nl2++ & 1)));
      uint8_t* dst = data + (size_t)st * kSlice;
      if (!lsu) {
        if (lane == 0) {
          wait(empty + st, ph ^ 1u);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + st)), "r"(kSlice));
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(dst)),
              "l"(src), "r"(kSlice), "r"(smem_u32(full + st))
              : "memory");
        }
        if (route != 0) __syncwarp();
      } else {
        wait(empty + st, ph ^ 1u);
#pragma unroll 8
        for (int j = 0; j < kSlice / 512; ++j) {
          const int off = (j * 32 + lane) * 16;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + off)), "l"(src + off) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(full + st)) : "memory");
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(full + st)) : "memory");
      }
      if (++st == kStages) { st = 0; ph ^= 1u; }
    }
    return;
  }
  int st = 0;
  uint32_t ph = 0;
  float acc = 0.f;
  for (size_t i = blockIdx.x; i < stages_total; i += gridDim.x) {
    wait(full + st, ph);
    const uint4* s = reinterpret_cast<const uint4*>(data + (size_t)st * kSlice);
    uint4 x[8];
    const int nr = consume == 0 ? 8 : consume == 1 ? 1 : 4;   // 32 / 4 / 16 KiB of the stage read
#pragma unroll
    for (int r = 0; r < 8; ++r) x[r] = r < nr ? s[tid + r * 256] : make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + st)) : "memory");
#pragma unroll
    for (int r = 0; r < 8; ++r) acc += __uint_as_float(x[r].x ^ x[r].y ^ x[r].z ^ x[r].w);
    if (++st == kStages) { st = 0; ph ^= 1u; }
  }
  if (acc == 1234.5f) *sink = acc;
}

int main(int argc, char** argv) {
  // optional: "sweep" = pure-L2 delivery for several slice-index strides and L2 footprints only
  const bool sweep = argc > 1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink;
  cudaMalloc(&sink, 4);
  const int smem = kStages * kSlice + 1024;
  cudaFuncSetAttribute(mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const size_t hbm_b = (size_t)4 << 30, l2_b = (size_t)96 << 20;
  uint8_t *hbm, *l2;
  cudaMalloc(&hbm, hbm_b);
  cudaMalloc(&l2, l2_b);
  cudaMemset(hbm, 1, hbm_b);
  cudaMemset(l2, 2, l2_b);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t total = ((size_t)4 << 30) / kSlice;          // 4 GiB delivered per run
  struct P { int H, M; } pats[] = {{1, 1}, {0, 1}, {3, 4}, {5, 9}, {1, 2}, {3, 8}, {1, 3}, {1, 4}};
  if (sweep) {
    for (size_t foot_mb : {8, 16, 32, 64, 96})
      for (unsigned long long mult : {1ull, 131ull, 7919ull}) {
        const size_t n_l2 = (foot_mb << 20) / kSlice;
        for (int w = 0; w < 2; ++w)
          mixed<<<sms, 288, smem>>>(hbm, hbm_b / kSlice, l2, n_l2, 0, 1, 0, total, sink, 0, mult);
        cudaEventRecord(a);
        mixed<<<sms, 288, smem>>>(hbm, hbm_b / kSlice, l2, n_l2, 0, 1, 0, total, sink, 0, mult);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("pure L2: footprint %3zu MiB, slice stride %5llu: %7.0f GB/s\n", foot_mb, mult,
               (double)total * kSlice / (ms * 1e6));
      }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
  }
  for (int consume = 0; consume < 3; ++consume)
  for (const P& p : pats)
    for (int route = 0; route < 3; ++route) {
      if (p.H == p.M && route > 0) continue;
      if (consume > 0 && route > 0) continue;
      for (int w = 0; w < 2; ++w)
        mixed<<<sms, 288, smem>>>(hbm, hbm_b / kSlice, l2, ((size_t)32 << 20) / kSlice, p.H, p.M, route, total, sink, consume, 131ull);
      cudaEventRecord(a);
      mixed<<<sms, 288, smem>>>(hbm, hbm_b / kSlice, l2, ((size_t)32 << 20) / kSlice, p.H, p.M, route, total, sink, consume, 131ull);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double gb = (double)total * kSlice / 1e9;
      const double hbm_gb = gb * p.H / p.M;
      printf("consume %d: HBM %d of %d stages, route %d (%s): %7.3f ms  delivered %6.0f GB/s  HBM part %6.0f GB/s\n",
             consume, p.H, p.M, route, route == 0 ? "all TMA" : route == 1 ? "L2 via LDGSTS" : "half L2 via LDGSTS", ms, gb / ms * 1e3,
             hbm_gb / ms * 1e3);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
