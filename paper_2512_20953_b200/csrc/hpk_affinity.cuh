// hpk_affinity.cuh — the stage mapper's DP-affinity pass (map_nodes_and_stages,
// P/src/stage_map.cpp:188-214; P = /root/reference/proj) as a CTA-level device
// function and its host-side flattening, shared by the stand-alone launch
// (hpk_stagemap.cu, hpk_stage_affinity) and the fused affinity + partition +
// cost launch of the planner (hpk_partition.cu, hpk_affinity_partition_cost).
// The algorithm and its O(1) swap delta are documented in hpk_stagemap.cu.
#pragma once

#include <algorithm>
#include <vector>

#include "hetplan_b200.h"

namespace hpks {

constexpr int AFF_THREADS = 256;

struct Prob {
  int n_groups, n_slots, n_types, n_nodes, n_ranks;
  int in_off;   // into the flat slot arrays
  int goff_off; // into the flat group-offset array
  int swaps;
};

// One candidate's affinity pass by the calling CTA (blockDim.x == AFF_THREADS).
// sm: dynamic shared memory of affinity_smem_bytes(P) bytes.
__device__ inline void affinity_body(Prob& P, const int* goff_all, const int* type_all,
                                     const int* node_all, int* perm_all, int* sm) {
  const int S = P.n_slots, G = P.n_groups, T = P.n_types, NN = P.n_nodes, R = P.n_ranks;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int THREADS = AFF_THREADS;
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

// Host: flattens the problems (dense node ids, per-problem type / rank counts)
// and returns the largest shared-memory need in bytes.
inline size_t affinity_flatten(const hpk_affinity_problem* probs, int n, std::vector<Prob>& hp,
                               std::vector<int>& goff, std::vector<int>& type,
                               std::vector<int>& node) {
  hp.assign(n, Prob{});
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
  return max_smem;
}

}  // namespace hpks
