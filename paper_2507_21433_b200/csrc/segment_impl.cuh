// a1 segmentation aggregates of seg_kernel (segment.cu: the flat token array, tiles and a
// decoupled look-back). PAPER.md:119; readings R1-R4.
#pragma once
#include "common.cuh"

namespace ms {

// (ends, content, bpos, bcb): bpos = position (flat) of the last boundary or -1, bcb = content
// tokens before bpos counted from the start of the range the aggregate covers.
struct Agg {
  int32_t e, c, bpos, bcb;
};

__device__ __forceinline__ Agg agg_identity() { return Agg{0, 0, -1, 0}; }

// a (earlier range) then b (later range)
__device__ __forceinline__ Agg combine(const Agg& a, const Agg& b) {
  Agg r;
  r.e = a.e + b.e;
  r.c = a.c + b.c;
  if (b.bpos >= 0) { r.bpos = b.bpos; r.bcb = a.c + b.bcb; }
  else { r.bpos = a.bpos; r.bcb = a.bcb; }
  return r;
}

__device__ __forceinline__ Agg shfl_agg_up(const Agg& v, int o) {
  return Agg{__shfl_up_sync(0xffffffffu, v.e, o), __shfl_up_sync(0xffffffffu, v.c, o),
             __shfl_up_sync(0xffffffffu, v.bpos, o), __shfl_up_sync(0xffffffffu, v.bcb, o)};
}

__device__ __forceinline__ Agg shfl_agg_down(const Agg& v, int o) {
  return Agg{__shfl_down_sync(0xffffffffu, v.e, o), __shfl_down_sync(0xffffffffu, v.c, o),
             __shfl_down_sync(0xffffffffu, v.bpos, o), __shfl_down_sync(0xffffffffu, v.bcb, o)};
}

}  // namespace ms
