// hpk_common.cuh — shared device helpers for the B200 plan-search kernels.
//
// Every fp64 operation that must match the reference bit-for-bit is written in
// the reference's operation order and the whole library is compiled with
// -fmad=false (the reference is built without FMA contraction).
#pragma once

#include <cstdint>

#define HPK_FULL_MASK 0xffffffffu

namespace hpk {

__device__ __forceinline__ double shfl(double v, int src) {
  return __shfl_sync(HPK_FULL_MASK, v, src);
}
__device__ __forceinline__ int shfl(int v, int src) { return __shfl_sync(HPK_FULL_MASK, v, src); }
__device__ __forceinline__ long long shfl(long long v, int src) {
  return __shfl_sync(HPK_FULL_MASK, v, src);
}

// Approximate warp sum (tree order). Only used by the exactness filters, whose
// margins absorb its rounding; never for a value the reference reports.
__device__ __forceinline__ double warp_sum_approx(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(HPK_FULL_MASK, v, o);
  return v;
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(HPK_FULL_MASK, v, o);
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(HPK_FULL_MASK, v, o);
    v = w < v ? w : v;
  }
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(HPK_FULL_MASK, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Candidate ranking of P/src/grouping.cpp:112-115 (higher objective, then fewer
// groups); `ia < ib` breaks remaining ties toward the earlier enumeration.
__device__ __forceinline__ bool key_better(double ao, int ag, int ia, double bo, int bg, int ib) {
  if (ao != bo) return ao > bo;
  if (ag != bg) return ag < bg;
  return ia < ib;
}

}  // namespace hpk
