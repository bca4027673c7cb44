// Tuning probe (not part of the product): does TMA multicast across a thread-block cluster raise
// the rate at which re-staged (L2-resident) slices reach the SMs? Pattern of a CROSS-pairing unit:
// every CTA of a cluster of C stages one private 32 KiB slice, then S slices that all C CTAs need.
//   unicast:   every CTA copies all S shared slices itself;
//   multicast: shared slice i is copied once by CTA (i mod C) into the same ring slot of all C CTAs
//              (cp.async.bulk ... .multicast::cluster), every consumer warp releases the slot in all
//              C CTAs (remote mbarrier arrive), so a slot is reused only when the whole cluster is done.
// Consumers only touch the data. Reported: slices delivered to SMs per second x 32 KiB.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tma_mc_probe tma_mc_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

constexpr int kC = 4;              // cluster size
constexpr int kSlice = 32768;
constexpr int kStages = 6;
constexpr int kCW = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void wait_parity(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                   smem_u32(bar)),
               "r"(ph)
               : "memory");
}

template <bool MC, bool RELAXED>
__global__ void __launch_bounds__(288, 1) probe(const uint8_t* buf, size_t nslices, int S, size_t units, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  uint8_t* data = sm + 1024;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = MC ? cta_rank() : 0;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + s)), "r"(MC ? kC * kCW : kCW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (MC) cluster_sync();
  const size_t cluster = MC ? blockIdx.x / kC : blockIdx.x;
  const size_t nclusters = MC ? gridDim.x / kC : gridDim.x;
  const int per_unit = 1 + S;
  if (warp == kCW) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (size_t u = cluster; u < units; u += nclusters) {
        for (int i = 0; i < per_unit; ++i) {
          wait_parity(empty + st, ph ^ 1u);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + st)), "r"(kSlice));
          // slice 0: this CTA's private slice; slices 1..S: shared by the cluster's CTAs
          const size_t sl = i == 0 ? ((u * kC + rank) * 7919ull + 17) % nslices : ((u * 131ull + i) * 7919ull) % nslices;
          if (!MC || i == 0) {
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(data + (size_t)st * kSlice)),
                "l"(buf + sl * kSlice), "r"(kSlice), "r"(smem_u32(full + st))
                : "memory");
          } else if ((uint32_t)(i % kC) == rank) {
            const uint16_t mask = (uint16_t)((1u << kC) - 1u);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, "
                "[%3], %4;" ::"r"(smem_u32(data + (size_t)st * kSlice)),
                "l"(buf + sl * kSlice), "r"(kSlice), "r"(smem_u32(full + st)), "h"(mask)
                : "memory");
          }
          if (++st == kStages) { st = 0; ph ^= 1u; }
        }
      }
    }
  } else {
    int st = 0;
    uint32_t ph = 0;
    float acc = 0.f;
    for (size_t u = cluster; u < units; u += nclusters) {
      for (int i = 0; i < per_unit; ++i) {
        wait_parity(full + st, ph);
        acc += __uint_as_float(*reinterpret_cast<const uint32_t*>(data + (size_t)st * kSlice + tid * 4));
        __syncwarp();
        if (MC) {
          // all consumer warps of this CTA are done with the slot (named barrier), then one thread
          // per CTA arrives on every cluster CTA's empty barrier with the count of this CTA's warps
          asm volatile("bar.sync 1, %0;" ::"n"(kCW * 32) : "memory");
          if (tid < kC) {
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(empty + st)), "r"(tid));
            if (RELAXED)
              asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(remote), "r"(kCW) : "memory");
            else
              asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(remote), "r"(kCW) : "memory");
          }
        } else if (lane == 0) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + st)) : "memory");
        }
        if (++st == kStages) { st = 0; ph ^= 1u; }
      }
    }
    if (acc == 1234.5f) *sink = acc;
  }
  if (MC) cluster_sync();   // no CTA exits while others may still arrive on its barriers
}

int main(int argc, char** argv) {
  const size_t foot_mb = argc > 1 ? (size_t)atoll(argv[1]) : 32;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink;
  cudaMalloc(&sink, 4);
  const size_t bytes = foot_mb << 20;
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  const int smem = 1024 + kStages * kSlice;
  cudaFuncSetAttribute(probe<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = sms / kC * kC;
  printf("source footprint %zu MiB, cluster %d, grid %d\n", foot_mb, kC, grid);
  for (int S : {4, 16, 64}) {
    const size_t units = (size_t)40000 / (1 + S) * 4;
    for (int mc = 0; mc < 3; ++mc) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(288);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = mc ? kC : 1;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      auto k = mc == 2 ? probe<true, true> : mc == 1 ? probe<true, false> : probe<false, false>;
      // unicast: every CTA is its own "cluster" and runs units / kC of the clusters' units x kC CTAs
      const size_t u = mc ? units : units;
      for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, k, (const uint8_t*)buf, bytes / kSlice, S, u, sink);
      cudaEventRecord(a);
      cudaLaunchKernelEx(&cfg, k, (const uint8_t*)buf, bytes / kSlice, S, u, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      // slices delivered to SMs: unicast = units x (1 + S) (each unit on one CTA);
      // multicast = units x kC x (1 + S) (each unit feeds kC CTAs)
      const double slices = (double)u * (1 + S) * (mc ? kC : 1);
      printf("%s S %2d: %8.3f ms, %8.1f GB/s delivered to SMs, L2 reads %8.1f GB/s\n", mc == 2 ? "mc relaxed" : mc == 1 ? "mc release" : "unicast   ", S,
             ms, slices * kSlice / (ms * 1e6), (double)u * (mc ? (kC + S) : (1 + S)) * kSlice / (ms * 1e6));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
