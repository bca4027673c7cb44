// Tuning probe (not part of the product): HBM -> shared memory throughput of a TMA 1-D bulk-copy
// ring (1 CTA per SM, 1 producer lane, 8 consumer warps that only release the stage) as a
// function of the bytes per copy, the copies per stage (one mbarrier per stage) and the ring
// depth. Source addresses are scattered copy-sized slices of a 4 GiB buffer (argument: another
// footprint in MiB, e.g. 32 for an L2-resident source).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tma_sweep tma_sweep.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(288, 1) ring(const uint8_t* buf, size_t nslices, int copy, int per_stage, int stages,
                                               size_t total_copies, float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 64;
  uint8_t* data = sm + 1024;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t stages_total = total_copies / per_stage;
  if (warp == 8) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      size_t c = 0;
      for (size_t i = blockIdx.x; i < stages_total; i += gridDim.x) {
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                         smem_u32(empty + st)),
                     "r"(ph ^ 1u));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + st)),
                     "r"(copy * per_stage));
        for (int j = 0; j < per_stage; ++j) {
          const size_t sl = ((i * per_stage + j) * 7919ull) % nslices;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(data + ((size_t)st * per_stage + j) * copy)),
              "l"(buf + sl * copy), "r"(copy), "r"(smem_u32(full + st))
              : "memory");
        }
        (void)c;
        if (++st == stages) { st = 0; ph ^= 1u; }
      }
    }
    return;
  }
  int st = 0;
  uint32_t ph = 0;
  float acc = 0.f;
  for (size_t i = blockIdx.x; i < stages_total; i += gridDim.x) {
    asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(
                     smem_u32(full + st)),
                 "r"(ph)
                 : "memory");
    acc += __uint_as_float(*reinterpret_cast<const uint32_t*>(data + (size_t)st * per_stage * copy + tid * 4));
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + st)) : "memory");
    if (++st == stages) { st = 0; ph ^= 1u; }
  }
  if (acc == 1234.5f) *sink = acc;
}

int main(int argc, char** argv) {
  // optional argument: the source footprint in MiB (default 4096: HBM; e.g. 32: L2-resident, to
  // measure the L2 -> shared-memory rate the sharing regime's re-staged slices run at)
  const size_t foot_mb = argc > 1 ? (size_t)atoll(argv[1]) : 4096;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink;
  cudaMalloc(&sink, 4);
  const int ring_max = 208 * 1024;
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, ring_max + 1024);
  const size_t bytes = foot_mb << 20;
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("source footprint %zu MiB\n", foot_mb);
  for (int copy : {2048, 4096, 8192, 16384, 32768, 65536, 98304}) {
    for (int per_stage : {1, 2, 4}) {
      for (int ring_kb : {64, 128, 208}) {
        const int stage_b = copy * per_stage;
        const int stages = ring_kb * 1024 / stage_b;
        if (stages < 2 || stages > 64 || stages * stage_b > ring_max) continue;
        const size_t nslices = bytes / copy;
        const size_t total = ((size_t)3 << 30) / copy;       // 3 GiB moved
        for (int w = 0; w < 2; ++w)
          ring<<<sms, 288, ring_max + 1024>>>(buf, nslices, copy, per_stage, stages, total, sink);
        cudaEventRecord(a);
        ring<<<sms, 288, ring_max + 1024>>>(buf, nslices, copy, per_stage, stages, total, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("copy %6d B x %d per stage, %2d stages (%3d KiB in flight): %8.1f GB/s\n", copy, per_stage, stages,
               stages * stage_b / 1024, (double)total * copy / (ms * 1e6));
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
