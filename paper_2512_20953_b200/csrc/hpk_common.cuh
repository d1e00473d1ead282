// hpk_common.cuh — shared device helpers for the B200 plan-search kernels.
//
// Every fp64 operation that must match the reference bit-for-bit is written in
// the reference's operation order and the whole library is compiled with
// -fmad=false (the reference is built without FMA contraction).
#pragma once

#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>

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

// 64-bit unsigned warp min / max with two 32-bit redux.sync (high word, then
// the low word among the lanes holding the extreme high word). Used on the bit
// patterns of non-negative doubles, which order like the values.
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
  const unsigned hi = (unsigned)(v >> 32);
  const unsigned mh = __reduce_min_sync(HPK_FULL_MASK, hi);
  const unsigned ml = __reduce_min_sync(HPK_FULL_MASK, hi == mh ? (unsigned)v : 0xffffffffu);
  return ((unsigned long long)mh << 32) | ml;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
  const unsigned hi = (unsigned)(v >> 32);
  const unsigned mh = __reduce_max_sync(HPK_FULL_MASK, hi);
  const unsigned ml = __reduce_max_sync(HPK_FULL_MASK, hi == mh ? (unsigned)v : 0u);
  return ((unsigned long long)mh << 32) | ml;
}

// Candidate ranking of P/src/grouping.cpp:112-115 (higher objective, then fewer
// groups); `ia < ib` breaks remaining ties toward the earlier enumeration.
__device__ __forceinline__ bool key_better(double ao, int ag, int ia, double bo, int bg, int ib) {
  if (ao != bo) return ao > bo;
  if (ag != bg) return ag < bg;
  return ia < ib;
}

}  // namespace hpk

// Host-side staging arena shared by the hpk_* wrappers: one pinned host buffer
// and one device buffer, grown on demand and kept for the next call, so a
// launch costs one H2D and one D2H copy instead of a malloc / copy / free per
// array. Layout: inputs first (copied H2D as one span), outputs after.
struct HpkArena {
  char* h = nullptr;  // pinned
  char* d = nullptr;
  size_t cap = 0;
  size_t used = 0;
  void reset() { used = 0; }
  // reserves bytes (16-aligned); returns the offset
  size_t take(size_t bytes) {
    used = (used + 15) & ~(size_t)15;
    const size_t o = used;
    used += bytes;
    return o;
  }
  // makes room for `used` bytes (contents are not preserved)
  cudaError_t fit() {
    if (used <= cap) return cudaSuccess;
    if (h) cudaFreeHost(h);
    if (d) cudaFree(d);
    h = nullptr;
    d = nullptr;
    size_t want = cap * 2 > used ? cap * 2 : used;
    cudaError_t e = cudaMallocHost(&h, want);
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&d, want);
    if (e != cudaSuccess) return e;
    cap = want;
    return cudaSuccess;
  }
  template <typename T>
  T* hp(size_t off) const { return reinterpret_cast<T*>(h + off); }
  template <typename T>
  T* dp(size_t off) const { return reinterpret_cast<T*>(d + off); }
};
