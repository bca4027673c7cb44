// Tuning probe (not part of the product): L2 -> shared memory rate of TMA TENSOR copies
// (cp.async.bulk.tensor.2d, a tensor map over the source) against 1-D bulk copies of the same
// bytes, one producer lane per SM and 8 warps that only release the stage (as tma_sweep.cu).
// A slice = ROWS x 256 B (ROWS = 64 / 128: 16 / 32 KiB), scattered over a `foot` MiB source.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tma_tensor_sweep tma_tensor_sweep.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool TENSOR>
__global__ void __launch_bounds__(288, 1) ring(const __grid_constant__ CUtensorMap tmap, const uint8_t* buf,
                                               size_t nslices, int rows, int stages, size_t total, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 64;
  uint8_t* data = sm + 1024;
  const int copy = rows * 256;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (size_t i = blockIdx.x; i < total; i += gridDim.x) {
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                         smem_u32(empty + st)),
                     "r"(ph ^ 1u));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + st)), "r"(copy));
        const size_t sl = (i * 7919ull) % nslices;
        if (TENSOR) {
          const int32_t y = (int32_t)(sl * rows);     // first row of the slice; x = 0
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  smem_u32(data + (size_t)st * copy)),
              "l"(&tmap), "r"(0), "r"(y), "r"(smem_u32(full + st))
              : "memory");
        } else {
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(data + (size_t)st * copy)),
              "l"(buf + sl * copy), "r"(copy), "r"(smem_u32(full + st))
              : "memory");
        }
        if (++st == stages) { st = 0; ph ^= 1u; }
      }
    }
    return;
  }
  int st = 0;
  uint32_t ph = 0;
  float acc = 0.f;
  for (size_t i = blockIdx.x; i < total; i += gridDim.x) {
    asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(
                     smem_u32(full + st)),
                 "r"(ph)
                 : "memory");
    acc += __uint_as_float(*reinterpret_cast<const uint32_t*>(data + (size_t)st * copy + tid * 4));
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + st)) : "memory");
    if (++st == stages) { st = 0; ph ^= 1u; }
  }
  if (acc == 1234.5f) *sink = acc;
}

int main(int argc, char** argv) {
  const size_t foot_mb = argc > 1 ? (size_t)atoll(argv[1]) : 32;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink;
  cudaMalloc(&sink, 4);
  const int ring_max = 208 * 1024;
  cudaFuncSetAttribute(ring<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, ring_max + 1024);
  cudaFuncSetAttribute(ring<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, ring_max + 1024);
  const size_t bytes = foot_mb << 20;
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("source footprint %zu MiB\n", foot_mb);
  for (int rows : {64, 128, 256}) {
    // the source as a 2-D tensor of 256-byte rows (128 bf16), box = rows x 256 B
    CUtensorMap tm;
    const cuuint64_t gdim[2] = {128, bytes / 256};
    const cuuint64_t gstride[1] = {256};
    const cuuint32_t box[2] = {128, (cuuint32_t)rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gdim, gstride, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("rows %d: cuTensorMapEncodeTiled failed (%d)\n", rows, (int)r);
      continue;
    }
    const int copy = rows * 256;
    const int stages = ring_max / copy;
    const size_t nslices = bytes / copy;
    const size_t total = ((size_t)3 << 30) / copy;
    for (int tensor = 0; tensor < 2; ++tensor) {
      auto k = tensor ? ring<true> : ring<false>;
      for (int w = 0; w < 2; ++w) k<<<sms, 288, ring_max + 1024>>>(tm, buf, nslices, rows, stages, total, sink);
      cudaEventRecord(a);
      k<<<sms, 288, ring_max + 1024>>>(tm, buf, nslices, rows, stages, total, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("%s copy %6d B, %2d stages: %8.1f GB/s\n", tensor ? "tensor" : "bulk  ", copy, stages,
             (double)total * copy / (ms * 1e6));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
