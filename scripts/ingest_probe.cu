// Tuning probe (not part of the product): per-SM ingest bandwidth of L2-resident and HBM data via
// (a) a TMA 1-D bulk-copy ring (1 CTA/SM, 6 x 32 KiB stages), (b) LDG.128 with many warps.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o ingest_probe ingest_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kStages = 6, kStage = 32768;

__global__ void __launch_bounds__(288, 1) tma_ring(const uint8_t* buf, size_t bytes, int reps, float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kStage);
  uint64_t* empty = full + kStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t nslices = bytes / kStage;
  const size_t total = nslices * reps;
  if (warp == 8) {
    if (lane == 0) {
      int st = 0; uint32_t ph = 0;
      for (size_t i = blockIdx.x; i < total; i += gridDim.x) {
        const size_t sl = (i * 7919) % nslices;   // scatter
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(empty + st)), "r"(ph ^ 1u));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + st)), "r"(kStage));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + st * kStage)), "l"(buf + sl * kStage), "r"(kStage), "r"(smem_u32(full + st)) : "memory");
        if (++st == kStages) { st = 0; ph ^= 1u; }
      }
    }
    return;
  }
  int st = 0; uint32_t ph = 0;
  float acc = 0.f;
  for (size_t i = blockIdx.x; i < total; i += gridDim.x) {
    asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(smem_u32(full + st)), "r"(ph) : "memory");
    const uint4* s4 = reinterpret_cast<const uint4*>(sm + st * kStage);
    for (int r = 0; r < 8; ++r) { uint4 x = s4[tid + r * 256]; acc += __uint_as_float(x.x); }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + st)) : "memory");
    if (++st == kStages) { st = 0; ph ^= 1u; }
  }
  if (acc == 1234.5f) *sink = acc;
}

__global__ void ldg_stream(const uint4* buf, size_t n16, int reps, float* sink) {
  float acc = 0.f;
  const size_t nslices = n16 / 2048;       // 32 KiB slices
  const size_t total = nslices * reps;
  // one warp per slice: 32 lanes x 64 uint4
  const int lane = threadIdx.x & 31;
  for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5; i < total;
       i += ((size_t)gridDim.x * blockDim.x) >> 5) {
    const size_t sl = (i * 7919) % nslices;
    const uint4* p = buf + sl * 2048;
#pragma unroll 8
    for (int r = 0; r < 64; ++r) { uint4 x = __ldcg(p + lane + r * 32); acc += __uint_as_float(x.x); }
  }
  if (acc == 1234.5f) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink;
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(tma_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kStage + 128);
  for (size_t mb : {48, 2048}) {          // 48 MiB: L2-resident; 2 GiB: HBM
    const size_t bytes = mb << 20;
    uint8_t* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    const int reps = mb < 100 ? 64 : 2;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) tma_ring<<<sms, 288, kStages * kStage + 128>>>(buf, bytes, reps, sink);
    cudaEventRecord(a);
    tma_ring<<<sms, 288, kStages * kStage + 128>>>(buf, bytes, reps, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("TMA ring  %5zu MiB x%2d: %8.1f GB/s\n", mb, reps, (double)bytes * reps / (ms * 1e6));
    for (int blocks : {2, 4, 8}) {
      for (int w = 0; w < 2; ++w) ldg_stream<<<sms * blocks, 512>>>((const uint4*)buf, bytes / 16, reps, sink);
      cudaEventRecord(a);
      ldg_stream<<<sms * blocks, 512>>>((const uint4*)buf, bytes / 16, reps, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("LDG x%d CTA/SM %5zu MiB x%2d: %8.1f GB/s\n", blocks, mb, reps, (double)bytes * reps / (ms * 1e6));
    }
    cudaFree(buf);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
