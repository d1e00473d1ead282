// hpk_stagemap.cu — the DP-affinity pass of the reference stage mapper
// (map_nodes_and_stages, P/src/stage_map.cpp:188-214; P = /root/reference/proj)
// on the B200, batched over every candidate plan of a planning call.
//
// The reference hill-climbs over swaps of same-type units between stage slots:
// it scans (group j, slot sj, group k, slot sk) lexicographically, applies the
// FIRST swap that strictly increases count_intra_node_dp_pairs() (:39-58) and
// restarts the scan. Each count is O(G^2 * stages) with string-keyed maps, so
// the pass costs ~3.5 ms on the host for 64 TP units (cfg4). Here one CTA per
// candidate evaluates the count change of every swap of the scan in parallel
// and applies the lowest-index improving one — the same sequence of swaps.
//
// Count change of swapping slots x, y (both of type t, nodes nx != ny). A
// slot's unit is matched with the units at the same rank (position among its
// group's type-t slots in stage order — fixed, swaps keep types) in every
// other group (:46-54). With H[t][r][v] = number of slots of type t and rank
// r whose unit is on node v (each group has at most one such slot):
//   delta = H[t][rx][ny] + H[t][ry][nx] - H[t][rx][nx] - H[t][ry][ny] + 2
// for rx != ry (or x, y in one group), and 0 when rx == ry (the rank's node
// multiset is unchanged). The swap improves iff delta > 0; integers: exact.
// After a swap only four histogram cells change.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "hetplan_b200.h"
#include "hpk_affinity.cuh"
#include "hpk_common.cuh"

void hpkp_fail(const std::string& msg);  // thread-local error of the hpk_* layer
namespace hpk_timing_bridge {
void add_affinity(double ms, long long h2d, long long d2h);  // this thread's hpk_timing
}

namespace hpks {

constexpr int THREADS = AFF_THREADS;

// dynamic smem: node[S] type[S] rank[S] perm[S] cnt[G*T] H[T*R*NN] red[32]
__global__ void __launch_bounds__(THREADS) affinity_kernel(Prob* probs, const int* goff_all,
                                                           const int* type_all,
                                                           const int* node_all, int* perm_all) {
  extern __shared__ int sm[];
  affinity_body(probs[blockIdx.x], goff_all, type_all, node_all, perm_all, sm);
}

struct Ctx {
  int device = -1;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  HpkArena arena;
  std::mutex mu;
};
Ctx g_ctx[16];

}  // namespace hpks

#define HPKS_CUDA(call)                                                                 \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess) {                                                            \
      hpkp_fail(std::string("hetplan_b200 CUDA error: ") + cudaGetErrorString(_e) +     \
                " at " #call);                                                          \
      return 5;                                                                         \
    }                                                                                   \
  } while (0)

extern "C" int hpk_stage_affinity(hpk_affinity_problem* probs, int n, int device) {
  using namespace hpks;
  if (n <= 0) return 0;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
    cudaGetLastError();
    hpkp_fail("hetplan_b200: no CUDA device visible; the B200 planner has no CPU fallback");
    return 5;
  }
  if (device < 0 && cudaGetDevice(&device) != cudaSuccess) device = 0;
  if (device >= ndev || device >= 16) {
    hpkp_fail("hetplan_b200: bad device ordinal");
    return 6;
  }
  Ctx& cx = g_ctx[device];
  std::lock_guard<std::mutex> lock(cx.mu);
  HPKS_CUDA(cudaSetDevice(device));
  if (cx.device != device) {
    HPKS_CUDA(cudaStreamCreateWithFlags(&cx.stream, cudaStreamNonBlocking));
    HPKS_CUDA(cudaEventCreate(&cx.ev0));
    HPKS_CUDA(cudaEventCreate(&cx.ev1));
    cx.device = device;
  }
  std::vector<Prob> hp;
  std::vector<int> goff, type, node;
  const size_t max_smem = affinity_flatten(probs, n, hp, goff, type, node);
  if (max_smem > 200 * 1024) {
    hpkp_fail("hetplan_b200: stage-affinity problem too large for shared memory");
    return 6;
  }
  const size_t S_total = type.size();
  HpkArena& ar = cx.arena;  // inputs | outputs, one copy each way
  ar.reset();
  const size_t o_probs = ar.take(sizeof(Prob) * n);
  const size_t o_goff = ar.take(sizeof(int) * goff.size());
  const size_t o_type = ar.take(sizeof(int) * S_total);
  const size_t o_node = ar.take(sizeof(int) * S_total);
  const size_t in_end = ar.used;
  const size_t o_perm = ar.take(sizeof(int) * S_total);
  const size_t out_end = ar.used;
  HPKS_CUDA(ar.fit());
  std::memcpy(ar.h + o_probs, hp.data(), sizeof(Prob) * n);
  std::memcpy(ar.h + o_goff, goff.data(), sizeof(int) * goff.size());
  std::memcpy(ar.h + o_type, type.data(), sizeof(int) * S_total);
  std::memcpy(ar.h + o_node, node.data(), sizeof(int) * S_total);
  HPKS_CUDA(cudaMemcpyAsync(ar.d, ar.h, in_end, cudaMemcpyHostToDevice, cx.stream));
  Prob* d_probs = ar.dp<Prob>(o_probs);
  int* d_goff = ar.dp<int>(o_goff);
  int* d_type = ar.dp<int>(o_type);
  int* d_node = ar.dp<int>(o_node);
  int* d_perm = ar.dp<int>(o_perm);
  if (max_smem > 48 * 1024)
    HPKS_CUDA(cudaFuncSetAttribute(affinity_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)max_smem));
  constexpr bool trace = HPK_HOST_TRACE != 0;  // build-time: -DHPK_HOST_TRACE=1
  HPKS_CUDA(cudaEventRecord(cx.ev0, cx.stream));
  affinity_kernel<<<n, THREADS, max_smem, cx.stream>>>(d_probs, d_goff, d_type, d_node, d_perm);
  HPKS_CUDA(cudaGetLastError());
  HPKS_CUDA(cudaEventRecord(cx.ev1, cx.stream));
  // outputs: the permutation, and the problem records (swap counts) again
  HPKS_CUDA(cudaMemcpyAsync(ar.h + o_perm, ar.d + o_perm, out_end - o_perm, cudaMemcpyDeviceToHost,
                            cx.stream));
  HPKS_CUDA(cudaMemcpyAsync(ar.h + o_probs, ar.d + o_probs, sizeof(Prob) * n,
                            cudaMemcpyDeviceToHost, cx.stream));
  HPKS_CUDA(cudaStreamSynchronize(cx.stream));
  const int* perm = ar.hp<int>(o_perm);
  float kms = 0;
  HPKS_CUDA(cudaEventElapsedTime(&kms, cx.ev0, cx.ev1));
  hpk_timing_bridge::add_affinity(kms, (long long)in_end,
                                  (long long)(out_end - o_perm + sizeof(Prob) * n));
  std::memcpy(hp.data(), ar.h + o_probs, sizeof(Prob) * n);
  for (int k = 0; k < n; ++k) {
    for (int s = 0; s < probs[k].n_slots; ++s) probs[k].slot_perm[s] = perm[hp[k].in_off + s];
    probs[k].swaps = hp[k].swaps;
  }
  if (trace) {
    fprintf(stderr, "[hpk-affinity] %d problems, kernel %.3f ms, swaps:", n, kms);
    for (int k = 0; k < n && k < 16; ++k)
      fprintf(stderr, " %d(S=%d,G=%d)", hp[k].swaps, hp[k].n_slots, hp[k].n_groups);
    fprintf(stderr, "\n");
  }
  return 0;
}
