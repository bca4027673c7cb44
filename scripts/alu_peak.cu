// Microbenchmark (not part of the product): the CUDA-core ceiling of the distance kernels' inner
// loop on this GPU -- per bf16 element pair one FHFMA.BF16 (d = t - s from the packed source) and
// half an FFMA2 (acc += d*d), registers only, no memory traffic. Also the alternative with the
// source unpacked on the ALU pipe (PRMT / LOP3) and both steps as FFMA2.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/alu_peak scripts/alu_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 sub_bf2(unsigned x, float2 t) {
  float2 d;
  asm volatile("{\n.reg .b16 lo, hi;\nmov.b32 {lo, hi}, %2;\n"
               "fma.rn.f32.bf16 %0, lo, %5, %3;\nfma.rn.f32.bf16 %1, hi, %5, %4;\n}\n"
               : "=f"(d.x), "=f"(d.y)
               : "r"(x), "f"(t.x), "f"(t.y), "h"((unsigned short)0xBF80u));
  return d;
}

constexpr int kW = 16;   // independent words per thread (ILP)

template <int kMode>
__global__ void __launch_bounds__(256) alu_kernel(const unsigned* in, float* out, int iters) {
  unsigned x[kW];
  float2 t[kW], acc[4];
  for (int i = 0; i < kW; ++i) {
    x[i] = in[(threadIdx.x + i) & 1023];
    t[i] = make_float2(__uint_as_float(x[i] << 16), __uint_as_float(x[i] & 0xffff0000u));
  }
  for (int i = 0; i < 4; ++i) acc[i] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kW; ++i) {
      float2 d;
      if (kMode == 0) {
        d = sub_bf2(x[i], t[i]);
      } else {
        const float2 s = make_float2(__uint_as_float(__byte_perm(x[i], 0u, 0x1054)), __uint_as_float(x[i] & 0xffff0000u));
        d = __ffma2_rn(s, make_float2(-1.f, -1.f), t[i]);
      }
      acc[i & 3] = __ffma2_rn(d, d, acc[i & 3]);
    }
#pragma unroll
    for (int i = 0; i < kW; ++i) x[i] += 0x00010001u;     // keep the loop from being hoisted
  }
  float s = 0.f;
  for (int i = 0; i < 4; ++i) s += acc[i].x + acc[i].y;
  if (s == 12345.f) out[0] = s;
}

int main() {
  unsigned* in;
  float* out;
  cudaMalloc(&in, 4096);
  cudaMalloc(&out, 4);
  cudaMemset(in, 0x3f, 4096);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode) {
    for (int bps : {1, 2, 4, 8}) {
      const int blocks = sms * bps;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) alu_kernel<0><<<blocks, 256>>>(in, out, iters);
        else alu_kernel<1><<<blocks, 256>>>(in, out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      const double ep = (double)blocks * 256 * iters * kW * 2;   // element pairs
      printf("mode %s  warps/SM %2d: %.3f T element-pairs/s\n", mode == 0 ? "FHFMA+FFMA2 " : "unpack+FFMA2",
             bps * 8, ep / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
