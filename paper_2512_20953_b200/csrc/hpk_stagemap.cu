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
#include "hpk_common.cuh"

void hpkp_fail(const std::string& msg);  // thread-local error of the hpk_* layer
namespace hpk_timing_bridge {
void add_affinity(double ms, long long h2d, long long d2h);  // this thread's hpk_timing
}

namespace hpks {

constexpr int THREADS = 256;

struct Prob {
  int n_groups, n_slots, n_types, n_nodes, n_ranks;
  int in_off;   // into the flat slot arrays
  int goff_off; // into the flat group-offset array
  int swaps;
};

// dynamic smem: node[S] type[S] rank[S] perm[S] cnt[G*T] H[T*R*NN] red[32]
__global__ void __launch_bounds__(THREADS) affinity_kernel(Prob* probs, const int* goff_all,
                                                           const int* type_all,
                                                           const int* node_all, int* perm_all) {
  extern __shared__ int sm[];
  Prob& P = probs[blockIdx.x];
  const int S = P.n_slots, G = P.n_groups, T = P.n_types, NN = P.n_nodes, R = P.n_ranks;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* node = sm;
  int* type = node + S;
  int* rank = type + S;
  int* perm = rank + S;
  int* cnt = perm + S;
  int* H = cnt + G * T;
  int* red = H + T * R * NN;
  const int* goff = goff_all + P.goff_off;
  for (int s = tid; s < S; s += THREADS) {
    node[s] = node_all[P.in_off + s];  // dense node ids (host)
    type[s] = type_all[P.in_off + s];
    perm[s] = s;
  }
  for (int i = tid; i < T * R * NN; i += THREADS) H[i] = 0;
  __syncthreads();
  if (tid == 0) {
    for (int i = 0; i < G * T; ++i) cnt[i] = 0;
    for (int j = 0; j < G; ++j)
      for (int s = goff[j]; s < goff[j + 1]; ++s) {
        rank[s] = cnt[j * T + type[s]]++;
        H[(type[s] * R + rank[s]) * NN + node[s]] += 1;
      }
  }
  __syncthreads();
  const long long total = (long long)S * S;
  int swaps = 0;
  while (true) {
    // lowest scan index (x * S + y) whose swap raises the count
    int best = 0x7fffffff;
    for (long long idx = tid; idx < total; idx += THREADS) {
      const int x = (int)(idx / S), y = (int)(idx - (long long)x * S);
      const int t = type[x];
      if (t != type[y]) continue;
      const int nx = node[x], ny = node[y], rx = rank[x], ry = rank[y];
      if (nx == ny || rx == ry) continue;  // no change (x == y is included)
      const int* hx = H + (t * R + rx) * NN;
      const int* hy = H + (t * R + ry) * NN;
      if (hx[ny] + hy[nx] + 2 > hx[nx] + hy[ny]) {
        best = (int)idx;
        break;  // this thread's indices ascend: its first hit is its minimum
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) red[warp] = best;
    __syncthreads();
    int b = red[0];
    for (int w = 1; w < THREADS / 32; ++w) b = min(b, red[w]);
    if (b == 0x7fffffff) break;
    if (tid == 0) {
      const int x = b / S, y = b % S;
      const int t = type[x], nx = node[x], ny = node[y];
      int* hx = H + (t * R + rank[x]) * NN;
      int* hy = H + (t * R + rank[y]) * NN;
      hx[nx] -= 1;
      hx[ny] += 1;
      hy[ny] -= 1;
      hy[nx] += 1;
      node[x] = ny;
      node[y] = nx;
      const int tp = perm[x];
      perm[x] = perm[y];
      perm[y] = tp;
    }
    ++swaps;
    __syncthreads();
  }
  for (int s = tid; s < S; s += THREADS) perm_all[P.in_off + s] = perm[s];
  if (tid == 0) P.swaps = swaps;
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
  std::vector<Prob> hp(n);
  std::vector<int> goff, type, node;
  size_t max_smem = 0;
  for (int k = 0; k < n; ++k) {
    const hpk_affinity_problem& in = probs[k];
    Prob& p = hp[k];
    p.n_groups = in.n_groups;
    p.n_slots = in.n_slots;
    p.n_types = 0;
    p.in_off = (int)type.size();
    p.goff_off = (int)goff.size();
    p.swaps = 0;
    for (int j = 0; j <= in.n_groups; ++j) goff.push_back(in.group_off[j]);
    std::vector<int> ids(in.slot_node, in.slot_node + in.n_slots);  // dense node ids
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    p.n_nodes = (int)ids.size();
    for (int s = 0; s < in.n_slots; ++s) {
      type.push_back(in.slot_type[s]);
      node.push_back((int)(std::lower_bound(ids.begin(), ids.end(), in.slot_node[s]) - ids.begin()));
      p.n_types = std::max(p.n_types, in.slot_type[s] + 1);
    }
    p.n_ranks = 1;  // max slots of one type in one group
    for (int j = 0; j < in.n_groups; ++j) {
      std::vector<int> c(p.n_types, 0);
      for (int s = in.group_off[j]; s < in.group_off[j + 1]; ++s)
        p.n_ranks = std::max(p.n_ranks, ++c[in.slot_type[s]]);
    }
    const size_t smem = sizeof(int) * (4 * (size_t)p.n_slots + (size_t)p.n_groups * p.n_types +
                                       (size_t)p.n_types * p.n_ranks * p.n_nodes + 32);
    max_smem = std::max(max_smem, smem);
  }
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
