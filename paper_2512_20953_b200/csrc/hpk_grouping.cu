// hpk_grouping.cu — B200 grouping search (the hot loop of the reference
// planner: dfs() in P/src/grouping.cpp:135-202 under solve_grouping_topk
// :269-335; P = /root/reference/proj).
//
// Three engines, all on the GPU, all exact (bit-identical winners, visits and
// optimal flag):
//
//  * Wave engine (hpk_wave_kernel): one persistent cooperative kernel searches
//    a batch of problems. The lexicographic (preorder) DFS is cut into an
//    ordered list of segments (subtrees). Each wave every warp runs segments
//    (a warp-cooperative DFS: lane g owns DP groups g and g + 32) with the
//    front's exact cutoff and a visit cap / time slice; unfinished segments are
//    split speculatively into a prefix record plus the remainder's pieces; a
//    per-problem scheduler CTA then commits the longest prefix of the list
//    whose runs are exact (cutoff at their position unchanged), applying the
//    budget cut exactly where the serial DFS would abort. A prefix record whose
//    cutoff turned out stale is re-run with an end marker; the ancestor it now
//    prunes deletes the pieces beneath it. The runner is specialised per
//    (top_k > 1, drift check, PREFIX segment, lane slots in use). Covers top_k
//    <= 16, <= 64 units here and <= 128 in the wide build
//    (hpk_grouping_wide.cu), and non-dyadic sums while no += / -= round trip
//    drifts. Exactness argument and data layout: DESIGN.md.
//
//  * Enumeration engine (hpk_enum_kernel): exhaustive top-1 searches of <= 12
//    units (the planner path) as an argmax over every leaf, unranked from the
//    restricted-growth-string index.
//
//  * Serial replica (hpk_serial_kernel): one thread per problem replays the
//    reference DFS statement by statement (including the += / -= group sums
//    and the top_k list). Used for what the wave engine hands back: drifting
//    sums, a node with more than 64 groups, more than 128 units, top_k > 16.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "hetplan_b200.h"
#include "hpk_common.cuh"

namespace cg = cooperative_groups;

// wave-engine tuning (build-time; the defaults are the measured best)
#ifndef HPK_SEG_CAP
#define HPK_SEG_CAP 1024      // visits per segment run per wave
#endif
#ifndef HPK_SPLIT_ONE_DEVICE
#define HPK_SPLIT_ONE_DEVICE 1  // run the long budgeted searches of a small launch
#endif                          // concurrently, each on a share of the SMs
#ifndef HPK_SPLIT_MAX
#define HPK_SPLIT_MAX 2         // partitions (equal shares of the wave-kernel CTA slots)
#endif
#ifndef HPK_CUT_IV_MAX
#define HPK_CUT_IV_MAX 16  // launches of at most this many searches use cutoff intervals
#endif
#ifndef HPK_SEG_CAP_BATCH
#define HPK_SEG_CAP_BATCH 2048  // ... for batches of more than 16 searches
#endif
#ifndef HPK_WAVE_NS
#define HPK_WAVE_NS 275000ull // run-phase time slice (A/B 200/225/250/275 us with the one-device split)
#endif
#ifndef HPK_CHECK_EVERY
#define HPK_CHECK_EVERY 64    // DFS iterations between stop-flag / time-slice checks (A/B: 32/64/128;
                              // a clock read every 16 with the flag read after the slice end:
                              // cfg5 +4 %, cfg4 no gain, profiles/r2_ab_slice_check.txt)
#endif
#ifndef HPK_QMUL
#define HPK_QMUL 4            // run slots per warp per wave
#endif
#ifndef HPK_QONE
#define HPK_QONE 1.7          // one problem's share of run slots, x warps
#endif

#ifndef HPK_TRACE_LEVEL
#define HPK_TRACE_LEVEL 0  // per-wave scheduler trace (debug builds only)
#endif

namespace hpk {

// Units per problem of this build's wave engine. The library links two builds
// of this file: the primary one (64 units: lanes own groups g and g+32) and
// hpk_grouping_wide.cu (128 units, same lane layout, so a node may hold at
// most 64 groups — more hands the problem to the serial replica). Problems
// with 65..128 units go to the wide build; the primary build's smaller
// per-entry paths keep the common case's list traffic low.
#ifndef HPK_MAXN
#define HPK_MAXN 64
#endif
constexpr int MAXN = HPK_MAXN;
#ifndef HPK_WPB
#define HPK_WPB 8
#endif
constexpr int WARPS_PER_BLOCK = HPK_WPB;
constexpr int BLOCK_THREADS = WARPS_PER_BLOCK * 32;
constexpr int TILE = BLOCK_THREADS * 8;  // list positions per expansion / commit tile
constexpr uint8_t KIND_FULL = 0;
constexpr uint8_t KIND_PREFIX = 1;
// top_k of the wave engine (grouping.cpp:117-132 with top_k > 1): the state
// the DFS carries between segments is the vector of the top_k best leaf
// objectives above the prune floor; larger top_k run on the serial replica.
#ifndef HPK_KW
#define HPK_KW 16
#endif
constexpr int KW = HPK_KW;

// ------------------------------------------------------------------ layout

struct GProb {
  int n, K, exact_mem, top_k;
  long long budget;  // < 0: unlimited (exhaustive mode)
  double min_mem;
  double p[MAXN], m[MAXN];
  int tkey[MAXN], nkey[MAXN];
  double f[MAXN + 2];   // f[d] = 1 - (d-1)/(K+d-1): Eq. (2) factor (grouping.cpp:103-108)
  double R[MAXN + 1];   // exact suffix sums of unit powers (contract: exact)
  double RM[MAXN + 1];  // remaining_mem from d, serial as grouping.cpp:156-160
  double mb_abs;        // absolute error bound of the approximate bound sums
  double md_abs;        // same for the deficit sums (0 when they are exact integers)
  int check_drift;      // 1: sums outside the exact-sum contract; every += is checked
                        // for drift (fl(fl(x+p)-p) != x), which sends the problem to
                        // the serial replica
};

// A segment of the ordered DFS list, stored in a per-problem entry pool; the
// list itself holds 4-byte pool ids plus contiguous per-position state.
struct __align__(16) Entry {
  uint8_t u[MAXN];         // segment root (entered by this segment's run)
  uint8_t end[MAXN];       // PREFIX: end marker (first node NOT in the segment)
  uint8_t best_rgs[MAXN];  // run output: best leaf of the segment
  double m;                // max feasible leaf objective (-1: none)
  double best_obj;
  long long visits;
  int best_G;
  int a_star;              // PREFIX re-run: depth of the pruned ancestor of `end`
  int cver;                // cutoff version of the last run (-1: never ran)
  uint8_t du, dend, kind, finished;
  uint8_t has_best, capped, uncapped;
  uint8_t hi;              // the segment is children [u[du-1], hi] of node u[0..du-1)
};

struct GState {
  double C;          // exact cutoff at the commit front
  long long V;       // committed visits
  double best_obj;
  int best_G, has_best;
  int cver;          // version of C (bumped whenever C changes)
  int cur, head, len;
  int done, aborted, rerun_pending, pool_cur;
  int pool_top;      // bump allocator of the active pool (atomic)
  int nagg;          // expansion tiles summarised in agg (0: none valid)
  long long rerun_cap;
  double seed_obj, seed_z;
  int seed_ix, waves;
  long long runs, run_visits, exact_checks;
  long long runs_prev;  // runs at the previous schedule (pieces-per-run estimate)
  int max_list, error;
  uint8_t best_rgs[MAXN];
  uint8_t seed_rgs[MAXN];
  // top_k > 1 (TOPK mode): the cutoff state at the commit front — the top_k
  // best leaf objectives strictly above the floor (seed_obj), descending; the
  // cutoff is T[top_k-1] once nT == top_k, else the floor (kth_objective(),
  // grouping.cpp:129-132) — and the global candidate list best-first
  // (SearchState::best, :99, ranking :112-115, insertion after equals :117-127).
  // parallel push (schedule step S4): published by the problem's commit CTA,
  // valid when pp_wave == the current wave
  int pp_wave, pp_mode, pp_head, pp_len, pp_ashift, pp_qmax, pp_ntile;
  int n_units;  // the problem's TP units (its weight in the run-queue share)
  long long pp_bl;
  double pp_C;
  int nT, nbest;
  double T[KW];
  double bl_obj[KW];
  int bl_G[KW];
  uint8_t bl_rgs[KW][MAXN];
};

// TOPK mode: what one run of a segment used and produced, one record per pool
// entry (allocated only when a batch has a problem with top_k > 1).
struct CandRec {
  double tin[KW];  // the cutoff state the run entered with
  int ntin, n;     // its size; candidates of the run
  double obj[KW];  // the run's own top_k leaves, ranking order
  int G[KW];
  uint8_t rgs[KW][MAXN];
};

// Summary of one expansion tile's output range [ob, ob + n) of the new list,
// written by expand_tile(): lets the commit walk and the queue scan pass a
// fully run, cutoff-consistent tile in O(1) instead of re-reading it.
struct TileAgg {
  int ob, n;        // output range
  int nrun, ndel;   // positions with a finished run; PREFIX re-runs that pruned an ancestor
  double mmax;      // max objective over the runs (-1: none)
  double cutc;      // the cutoff every run used (NaN: not all the same / none)
  double cutx;      // max cutoff the runs used (NaN: none) ...
  double chimin;    // ... and min of their interval ends: all exact for C in [cutx, chimin]
  long long sumvis; // visits of the runs
  double bobj;      // best candidate of the tile: (obj desc, G asc, position asc); -1: none
  int bG, bidx;
};

// Per-tile aggregate of the parallel push (needs, lower-bound visits).
struct PushAgg {
  int stamp, nneed;
  long long vis;
};

struct RunItem {
  int problem, pos, id, front;
  long long cap;
  double cut;  // predicted entering cutoff (exact-checked at commit)
  int ntv, pad;
  double tv[KW];  // TOPK: the predicted entering state (cut = its cutoff)
};

struct RunQueue {
  int len, head;
  int pad[2];
};

struct KParams {
  GProb* probs;
  GState* states;
  Entry* pools;       // [P][2][pcap]
  CandRec* cands;     // TOPK only: [P][2][pcap], parallel to pools (else null)
  int* lists;         // [P][2][5][lcap]: ids, pcver, cnt, pfirst, info
  long long* lvis;    // [P][2][lcap]: visits of the finished run at each position
  double* ldbl;       // [P][2][3][lcap]: cutoff the run at each position used, its max
                      // objective, its best objective
  int* scratch;       // [P][lcap + 1]
  int* xt;            // [P][xtn]: pieces added by this wave's splits, per list tile
  int2* work;         // [2][wcap]: expansion work items (problem, tile) per wave parity
  int* wcount;        // [2]
  int xtn, wcap;
  TileAgg* agg;       // [P][xtn]
  PushAgg* pagg;      // [P][xtn]: the parallel push's per-tile aggregates
  int par_push;       // 1: step D runs as per-tile push items over every CTA
  RunQueue* queues;   // [2]
  RunItem* items;     // [2][qcap]
  int* active;        // problems still running
  int* err;           // watchdog flags
  int* stop;          // run phase: the queue has drained (capped runs stop early)
  unsigned long long wave_ns;  // run-phase time slice (0: none): later runs stop and split
  int runners;        // warps per CTA that run segments (experiment knob; default all)
  int ranges;         // split pieces are sibling ranges (1) or single siblings (0)
  int cut_iv;         // k = 1 runs record their cutoff interval (few problems: the
                      // latency-bound case; a big batch has almost no stale runs)
  int n_problems;
  int lcap, pcap, qcap, qmax, reserve;
  int qmax_one;       // cap of one problem's share (a lone search floods its list past it)
  long long seg_cap;
  int ramp;           // first-wave visit cap, doubled every wave up to seg_cap (0: off)
  long long front_cap;  // visit cap of the list head's run (the time slice stops it)
  int max_waves;
  unsigned long long deadline_ns;  // %globaltimer watchdog (relative at launch)
  unsigned long long* deadline_slot;
  unsigned int* bar;               // grid barrier {count, generation}
  unsigned long long* prof;        // trace >= 2: runner phase cycle counters
  int trace;                       // HPK_TRACE=1: per-wave scheduler printf (debug)
  int trace_p;                     // HPK_TRACE_P: only this problem (-1: all)
};

__device__ __forceinline__ Entry* pool_ptr(const KParams& kp, int p, int which) {
  return kp.pools + ((size_t)p * 2 + which) * kp.pcap;
}
__device__ __forceinline__ CandRec* cand_ptr(const KParams& kp, int p, int which) {
  return kp.cands + ((size_t)p * 2 + which) * kp.pcap;
}
// list arrays of buffer `buf`: 0 ids, 1 pcver (1 = a finished run at this
// position, -1 = needs a run), 2 cnt (expansion count), 3 pfirst, 4 info (the
// run's best_G | 256 has_best | 512 PREFIX re-run that pruned an ancestor)
__device__ __forceinline__ int* list_arr(const KParams& kp, int p, int buf, int which) {
  return kp.lists + (((size_t)p * 2 + buf) * 6 + which) * kp.lcap;
}
__device__ __forceinline__ long long* list_vis(const KParams& kp, int p, int buf) {
  return kp.lvis + ((size_t)p * 2 + buf) * kp.lcap;
}
// which: 0 = cutoff used by the run at the position, 1 = its max leaf
// objective, 2 = its best objective
__device__ __forceinline__ double* list_dbl(const KParams& kp, int p, int buf, int which) {
  return kp.ldbl + (((size_t)p * 2 + buf) * 3 + which) * kp.lcap;
}

// scheduler CTA scratch (dynamic smem after the warps' DFS stacks)
struct SchedSmem {
  long long l[32];
  double d[32];
  int i[64];
  double bo[32];
  int bg[32], bi[32];
  long long v_after, v_before, cap;
  double c_after, c_before;
  int fb, fs, sp_del, ndel, head, flag;
  double part[8 * 8];  // AggAcc partials (8 warps x 64 B)
  // TOPK mode
  double tv[KW];       // predicted cutoff state (push_items)
  int ntv, sp_imp, fi, nq;
};

// --------------------------------------------------------------- warp DFS

struct WarpSmem {
  // the problem's tables, staged per run (all hot-loop loads are LDS)
  double tp[MAXN], tm[MAXN], tf[MAXN + 2], tR[MAXN + 1], tRM[MAXN + 1];
  double S[MAXN + 1];    // approx sum of Eq.(2) effective powers at each level
  double DEF[MAXN + 1];  // approx memory deficit at each level
  unsigned long long mpass[MAXN + 1];   // per level: children that pass the check
  unsigned long long mprune[MAXN + 1];  // per level: children that are pruned
  double mcut[MAXN + 1];                // cutoff the masks were computed with
  unsigned lvl[MAXN + 1];  // per level: path | next child << 8 | G << 16
  uint8_t path[MAXN];
  uint8_t endp[MAXN];
  uint8_t best[MAXN];
  // TOPK mode: the cutoff state (top_k objectives above the floor) and the
  // run's own candidate list (ranking order), grouping.cpp:117-132
  double T[KW];
  double robj[KW];
  int rG[KW];
  int nT, rn;  // (the candidates' RGS rows live in the run's CandRec, global)
  unsigned long long wave_end;  // the current run's time-slice end (0: none)
  int staged;  // problem whose tables tp..tRM hold (-1: none)
};

// ---- TOPK helpers (grouping.cpp:110-132)
// better(): higher objective, then fewer groups; equal keys keep the earlier
// enumeration (upper_bound inserts after equals), so a later candidate never
// wins a tie.
__device__ __forceinline__ bool rank_better(double ao, int ag, double bo, int bg) {
  if (ao != bo) return ao > bo;
  return ag < bg;
}
// kth_objective(): the floor until top_k objectives above it are known.
__device__ __forceinline__ double state_cut(const double* T, int nT, int tk, double floor_) {
  return nT >= tk ? T[tk - 1] : floor_;
}
// Adds objective v (> the state's cutoff, hence > floor) to the state (one thread).
__device__ __forceinline__ void state_insert(double* T, int* nT, int tk, double v) {
  const int n = *nT;
  int pos = n < tk ? n : tk - 1;
  while (pos > 0 && T[pos - 1] < v) {
    T[pos] = T[pos - 1];
    --pos;
  }
  T[pos] = v;
  *nT = n < tk ? n + 1 : tk;
}
// offer() into a best-first candidate list of <= tk entries (warp-cooperative,
// uniform arguments): insertion at upper_bound, the last entry drops out.
// src(i) gives unit i's group of the new candidate.
template <typename Src>
__device__ __forceinline__ void cand_insert(double* obj, int* G, uint8_t (*rgs)[MAXN], int* cnt,
                                            int tk, int nunits, double o, int g, Src src,
                                            int lane) {
  const int n = *cnt;
  int pos = n;
  for (int i = 0; i < n; ++i)
    if (rank_better(o, g, obj[i], G[i])) {
      pos = i;
      break;
    }
  if (pos >= tk) return;
  const int last = n < tk ? n : tk - 1;
  for (int r = last; r > pos; --r)  // each lane moves its own bytes: no hazard
    for (int i = lane; i < nunits; i += 32) rgs[r][i] = rgs[r - 1][i];
  for (int i = lane; i < nunits; i += 32) rgs[pos][i] = src(i);
  __syncwarp();
  if (lane == 0) {
    for (int r = last; r > pos; --r) {
      obj[r] = obj[r - 1];
      G[r] = G[r - 1];
    }
    obj[pos] = o;
    G[pos] = g;
    *cnt = last + 1;
  }
  __syncwarp();
}

// Problem view used by the runner: same member names as GProb, arrays in smem.
struct PView {
  const double* p;
  const double* m;
  const double* f;
  const double* R;
  const double* RM;
  int n, exact_mem, check_drift;
  double min_mem, mb_abs, md_abs;
};

// (the tables are constant after init: a warp re-stages only when its next
// run item belongs to another problem)
__device__ __forceinline__ PView stage_problem(const GProb& G, WarpSmem* sm, int lane, int pid) {
  const int n = G.n;
  if (sm->staged != pid) {
    for (int i = lane; i < n; i += 32) {
      sm->tp[i] = G.p[i];
      sm->tm[i] = G.m[i];
    }
    for (int i = lane; i <= n + 1; i += 32) sm->tf[i] = G.f[i];
    for (int i = lane; i <= n; i += 32) {
      sm->tR[i] = G.R[i];
      sm->tRM[i] = G.RM[i];
    }
    __syncwarp();
    if (lane == 0) sm->staged = pid;
  }
  __syncwarp();
  PView v;
  v.p = sm->tp;
  v.m = sm->tm;
  v.f = sm->tf;
  v.R = sm->tR;
  v.RM = sm->tRM;
  v.n = n;
  v.exact_mem = G.exact_mem;
  v.min_mem = G.min_mem;
  v.mb_abs = G.mb_abs;
  v.md_abs = G.md_abs;
  v.check_drift = G.check_drift;
  return v;
}

enum : int { DEC_PASS = 0, DEC_PRUNE = 1, DEC_EXACT = 2 };

constexpr double kEps52 = 2.220446049250313e-16;  // 2^-52

// Per-lane group registers: lane owns groups lane and lane+32; f0/f1 cache the
// Eq. (2) factors for the current member count and for one more member.
// Updates are branch-free: every lane executes them, the owner's select is
// taken. Under the wave engine's contract every sum is exact, so x + 0.0,
// 0.0 + up (push_back) and up - up (pop_back) equal the reference's values
// (grouping.cpp:180-198) bit for bit.
// The Eq. (2) factors of a slot: f[gc] (current members) and f[gc + 1] (one
// more), cached in registers and rotated on every += / -=. -DHPK_NO_FCACHE
// reads them from the staged table where used instead: fewer registers and
// spills, but measured 2 % slower on the cfg5 sweep (0.655 vs 0.640 s).
#ifndef HPK_NO_FCACHE
#define HPK_FCACHE 1
#endif
#ifdef HPK_FCACHE
#define HPK_F0(P, g, k) ((g).f0[k])
#define HPK_F1(P, g, k) ((g).f1[k])
#else
#define HPK_F0(P, g, k) ((P).f[(g).gc[k]])
#define HPK_F1(P, g, k) ((P).f[(g).gc[k] + 1])
#endif

struct Groups {
  double gp[2], gm[2];
#ifdef HPK_FCACHE
  double f0[2], f1[2];  // cached Eq. (2) factors f[gc], f[gc + 1]
#endif
  int gc[2];
  bool drift;  // check_drift: a += on this lane's groups would not round-trip
};

#ifndef HPK_SELECT_UPDATES
// Only the owner lane's slot changes: a warp-uniform branch on the slot (group
// >> 5) and a one-lane predicated update, instead of branch-free selects on
// both slots of every lane (same values: the other lanes' sums are untouched,
// which x + 0.0 also gave). -DHPK_SELECT_UPDATES restores the select form.
template <bool DRIFT, int NS = 2>
__device__ __forceinline__ void add_unit(const PView& P, Groups& g, int lane, int grp, double up,
                                         double um) {
  const int ks = grp >> 5;  // warp-uniform
  const bool me = (grp & 31) == lane;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    if (k == ks && me) {
      if (DRIFT && g.gc[k] > 0) {
        // the reference's -= after this += must give back the same sum
        // (grouping.cpp:184-198); a new group (push_back) cannot drift
        const double yp = g.gp[k] + up, ym = g.gm[k] + um;
        g.drift = g.drift || (yp - up) != g.gp[k] || (ym - um) != g.gm[k];
      }
      g.gp[k] += up;
      g.gm[k] += um;
      g.gc[k] += 1;
#ifdef HPK_FCACHE
      g.f0[k] = g.f1[k];
      g.f1[k] = P.f[g.gc[k] + 1];
#endif
    }
  }
}

template <int NS = 2>
__device__ __forceinline__ void remove_unit(const PView& P, Groups& g, int lane, int grp,
                                            double up, double um) {
  const int ks = grp >> 5;
  const bool me = (grp & 31) == lane;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    if (k == ks && me) {
      g.gp[k] -= up;
      g.gm[k] -= um;
      g.gc[k] -= 1;
#ifdef HPK_FCACHE
      g.f1[k] = g.f0[k];
      g.f0[k] = P.f[g.gc[k]];
#endif
    }
  }
}
#else
template <bool DRIFT>
__device__ __forceinline__ void add_unit(const PView& P, Groups& g, int lane, int grp, double up,
                                         double um) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const bool o = grp == lane + 32 * k;
    if (DRIFT && o && g.gc[k] > 0) {
      // the reference's -= after this += must give back the same sum
      // (grouping.cpp:184-198); a new group (push_back) cannot drift
      const double yp = g.gp[k] + up, ym = g.gm[k] + um;
      g.drift = g.drift || (yp - up) != g.gp[k] || (ym - um) != g.gm[k];
    }
    g.gp[k] += o ? up : 0.0;
    g.gm[k] += o ? um : 0.0;
    g.gc[k] += o ? 1 : 0;
    const double fn = P.f[g.gc[k] + 1];
#ifdef HPK_FCACHE
    g.f0[k] = o ? g.f1[k] : g.f0[k];
    g.f1[k] = o ? fn : g.f1[k];
#else
    (void)fn;
#endif
  }
}

__device__ __forceinline__ void remove_unit(const PView& P, Groups& g, int lane, int grp,
                                            double up, double um) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const bool o = grp == lane + 32 * k;
    g.gp[k] -= o ? up : 0.0;
    g.gm[k] -= o ? um : 0.0;
    g.gc[k] -= o ? 1 : 0;
    const double fp = P.f[g.gc[k]];
#ifdef HPK_FCACHE
    g.f1[k] = o ? g.f0[k] : g.f1[k];
    g.f0[k] = o ? fp : g.f0[k];
#else
    (void)fp;
#endif
  }
}

#endif

__device__ __forceinline__ void groups_init(const PView& P, Groups& g) {
  g.drift = false;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    g.gp[k] = 0;
    g.gm[k] = 0;
    g.gc[k] = 0;
#ifdef HPK_FCACHE
    g.f0[k] = P.f[0];
    g.f1[k] = P.f[1];
#endif
  }
}

// eff of this lane's slot k: f0 = f[gc] is the reference's (1 - rho) for the
// group (grouping.cpp:103-108); an empty slot has gp = 0 and f[0] = 0.
__device__ __forceinline__ double slot_eff(const PView& P, const Groups& g, int k) {
  (void)P;
  return g.gp[k] * HPK_F0(P, g, k);
}
__device__ __forceinline__ double slot_def(const PView& P, const Groups& g, int k) {
  const double d = P.min_mem - g.gm[k];
  return (g.gc[k] > 0 && d > 0.0) ? d : 0.0;  // std::max(0.0, d) over existing groups
}

// Exact node check in the reference's serial order (grouping.cpp:154-169) for
// the node whose units 0..next-1 are applied. Warp-uniform result.
__device__ bool exact_passes(const PView& P, const Groups& g, int G, int next, double cut) {
  double bound = 0;
  for (int gi = 0; gi < G; ++gi) {
    const int k = gi >> 5;
    const double e = shfl(k == 0 ? slot_eff(P, g, 0) : slot_eff(P, g, 1), gi & 31);
    bound += e;
  }
  for (int i = next; i < P.n; ++i) bound += P.p[i];
  if (cut >= 0 && bound < cut) return false;
  double deficit = 0;
  for (int gi = 0; gi < G; ++gi) {
    const int k = gi >> 5;
    const double dv = shfl(k == 0 ? slot_def(P, g, 0) : slot_def(P, g, 1), gi & 31);
    deficit += dv;
  }
  return !(deficit > P.RM[next]);
}

// Filter decision for a node given approximate sums (incrementally maintained
// along the path). P.mb_abs / P.md_abs bound the gap between the
// approximations and the reference's serial fp64 sums; only a
// cutoff inside that margin needs the exact serial evaluation.
// NOTE: written as early returns on purpose. The equivalent if/else-chain
// formulation (db/dd codes combined at the end) is miscompiled by nvcc 12.9 for
// sm_100a at -O3 — it never returns PASS (found with the HPK_TRACE=2 counters:
// 44% of child checks fell to the exact path); tools/ubench/decide_test2.cu
// and hpk_selftest_decide() pin the correct behaviour on the device.
__device__ __noinline__ int decide_core(double A, double D, double rem, double cut,
                                       double mb_abs, double md_abs) {
  const bool has_cut = cut >= 0;
  const bool b_prune = has_cut && (A + mb_abs < cut);
  const bool d_prune = D - md_abs > rem;
  if (b_prune || d_prune) return DEC_PRUNE;
  const bool b_pass = !has_cut || (A - mb_abs >= cut);
  const bool d_pass = D + md_abs <= rem;
  return (b_pass && d_pass) ? DEC_PASS : DEC_EXACT;
}
__device__ __forceinline__ int decide(const PView& P, double A, double D, int next, double cut) {
  return decide_core(A, D, P.RM[next], cut, P.mb_abs, P.md_abs);
}

// Device self-test of the filter decision on a grid of cases (see note above).
__global__ void hpk_selftest_decide_kernel(const double* in, int n, const double* rm,
                                           double mb, double md, int* out) {
  __shared__ double sRM[4];
  if (threadIdx.x < 4) sRM[threadIdx.x] = rm[threadIdx.x];
  __syncthreads();
  PView P;
  P.RM = sRM;
  P.mb_abs = mb;
  P.md_abs = md;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int r = -1;
    if ((threadIdx.x & 31) == (i & 31)) r = decide(P, in[3 * i], in[3 * i + 1], 2, in[3 * i + 2]);
    out[i] = r;
  }
}

struct RunOut {
  long long visits;
  double m;
  bool finished, has_best;
  double best_obj;
  int best_G, a_star;
  int dstop;   // unfinished: the stop node is path[0..dstop-1) + [stop_c]
  int exact;   // child checks resolved by the exact serial check
  int stop_c;
  bool overflow;  // reached an internal node with more than 63 groups (lanes own
                  // groups g, g+32): the problem goes to the serial replica
  bool drift;     // check_drift problems: some group sum would not round-trip
  bool retry;     // NS == 1 run met an internal node with 32 groups: rerun with NS == 2
  double hi;      // k = 1: every entering cutoff in [C, hi] gives this same run
};

// DFS of subtree(E.u) in preorder (PREFIX: stopping before E.end), cap visits.
//
// The current level's state — next child c, group count G, the approximate
// level sums Sd/Dd, the unit (up, um) its children assign, the children's
// pass/prune bitmasks and the cutoff they were computed with — is held in
// warp-uniform registers. A level is spilled to the per-warp smem stack only
// when the DFS descends below it and reloaded when it pops back, so a child
// check is register-only. A run of children the masks prune is consumed in
// O(1): each still counts one visit (grouping.cpp:178, the check happens on
// entry :161-169) and none is entered.
//
// stopf (optional): set once the wave's run queue has drained; a capped run
// then stops at its next check after the time slice and is split like a run
// that hit its cap, so no warp idles behind the wave's longest run.
//
// TOPK (top_k = tk > 1): the cutoff follows the state vector sm->T (entering
// state loaded by the caller; cut = its cutoff) — a feasible leaf above the
// cutoff joins it — and the run keeps its own top_k candidates in sm->r*,
// written to rec at the end (grouping.cpp:117-132).
// NS: group slots per lane in use — 1 when the problem has at most 32 units
// (every child index and group then fits lane slot 0, so slot 1 stays empty
// and its work compiles out), else 2.
template <bool TOPK, bool DRIFT, bool PFX, int NS, bool CI>
__device__ RunOut run_segment(const PView& P, const Entry* E, Entry* Eout, double C,
                              long long cap, WarpSmem* sm, int lane, int* err,
                              const unsigned long long* deadline_slot,
                              unsigned long long* prof, const int* stopf, int tk, double floor_,
                              CandRec* rec) {
  // (the watchdog deadline and the wave's time slice end, sm->wave_end, are
  // read where they are checked — every 1024 / 32 iterations — instead of
  // occupying registers through the hot loop)
  // prof (trace >= 2): [0] run cycles [1] leaf batches [2] leaves [3] loop iterations
  //   [4] single checks [5] descends [6] pops [7] prune skips [8] children skipped
  //   [9] exact fallbacks [10] mask computations
  long long pc0 = 0;
  unsigned long long pcnt[11];  // per-warp counters, flushed once per run (no atomics in the loop)
#pragma unroll
  for (int k = 0; k < 11; ++k) pcnt[k] = 0;
#ifdef HPK_RUNNER_PROF  // per-warp counters (trace >= 2), compiled out by default
#define HPK_PC(k, v) \
  do {               \
    if (prof) pcnt[k] += (v); \
  } while (0)
#else
#define HPK_PC(k, v) \
  do {               \
  } while (0)
#endif
  if (prof) pc0 = clock64();
  const int n = P.n;
  const int du = E->du;
  const bool prefix = PFX;  // E->kind == KIND_PREFIX (the caller dispatches)
  RunOut o;
  o.visits = 0;
  o.m = -1.0;
  o.finished = false;
  o.has_best = false;
  o.best_obj = 0;
  o.best_G = 0;
  o.a_star = -1;
  o.dstop = 0;
  o.stop_c = 0;
  o.exact = 0;
  o.overflow = false;
  o.retry = false;
  o.drift = false;
  o.hi = INFINITY;
  // Cutoff interval (k = 1, and top_k > 1 runs that find no leaf above their
  // entering cutoff: their cutoff stays that scalar). A larger entering cutoff C' only changes a run
  // through a child or node check that PASSED: a prune stays a prune, leaves
  // are not pruned and the run's own improvements raise both cutoffs alike. So
  // the run is the same for every C' <= each passed check's value — hl keeps
  // this lane's minimum of the filter's lower bound A - mb over its passed
  // children (the value the filter compared with the cutoff), or the cutoff
  // itself for a check resolved exactly; the commit walk then accepts the run
  // for an exact cutoff anywhere in [C, min over lanes].
  double hl = INFINITY;
  if (TOPK && lane == 0) sm->rn = 0;
  if (cap <= 0) {  // budget already exhausted: the reference aborts before entering u
    if (TOPK && lane == 0) rec->n = 0;
    return o;
  }
  const int dend = prefix ? E->dend : 0;
  for (int i = lane; i < du; i += 32) sm->path[i] = E->u[i];
  if (prefix)
    for (int i = lane; i < dend; i += 32) sm->endp[i] = E->end[i];
  __syncwarp();

  Groups g;
  groups_init(P, g);
  int G = 0;
  if (lane == 0) sm->lvl[0] = 0;
  for (int i = 0; i + 1 < du; ++i) {  // the range's parent node: units 0..du-2
    const int grp = sm->path[i];
    add_unit<DRIFT, NS>(P, g, lane, grp, P.p[i], P.m[i]);
    if (grp == G) ++G;
    if (lane == 0) sm->lvl[i + 1] = (unsigned)G << 16;
  }
  __syncwarp();
  // the segment is the children [u[dpar], hi] of the parent (each with its
  // subtree). A range is visited, checked and entered by the loop below like
  // the children of any other node (grouping.cpp:171-201); a single child is
  // entered directly (one visit, one node check) and the loop starts inside it.
  const int dpar = du - 1;
  const int hi = E->hi;
  const bool single = hi == sm->path[dpar];
  const int dtop = single ? du : dpar;  // the loop ends when this level is exhausted
  int d = dtop;
  double cut = C;
  double Sd, Dd;
  if (!single && G > 63) {  // the range's parent has 64 groups (65 children)
    o.overflow = true;
    o.finished = true;
    goto done;
  }
  if (NS == 1 && G > 31) {  // the parent's children would need lane slot 1
    o.retry = true;
    o.finished = true;
    goto done;
  }
  if (single) {  // enter the segment root u
    const int i = du - 1;
    const int grp = sm->path[i];
    add_unit<DRIFT, NS>(P, g, lane, grp, P.p[i], P.m[i]);
    if (grp == G) ++G;
    if (lane == 0) sm->lvl[du] = (unsigned)G << 16;
    o.visits = 1;
    __syncwarp();
    if (d < n && G > 63) {  // its children would need group slot 64
      o.overflow = true;
      o.finished = true;
      goto done;
    }
    if (NS == 1 && d < n && G > 31) {
      o.retry = true;
      o.finished = true;
      goto done;
    }
    if (d == n) {  // the root is a leaf (grouping.cpp:138-149)
      bool infeas = false;
      double z = INFINITY;
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        if (g.gc[k] > 0) {
          if (g.gm[k] < P.min_mem) infeas = true;
          const double e = slot_eff(P, g, k);
          z = e < z ? e : z;
        }
      }
      const bool any_infeas = __any_sync(HPK_FULL_MASK, infeas);
      z = warp_min(z);
      if (!any_infeas) {
        const double obj = (double)G * z;
        o.has_best = true;
        o.best_obj = obj;
        o.best_G = G;
        o.m = obj;
        if (TOPK) {
          if (lane == 0) {
            if (obj > cut) state_insert(sm->T, &sm->nT, tk, obj);
          }
          cand_insert(sm->robj, sm->rG, rec->rgs, &sm->rn, tk, n, obj, G,
                      [&](int i) { return sm->path[i]; }, lane);
        } else {
          for (int i = lane; i < n; i += 32) sm->best[i] = sm->path[i];
        }
      }
      o.finished = true;
      goto done;
    }
  }
  {
    const double le = NS == 2 ? slot_eff(P, g, 0) + slot_eff(P, g, 1) : slot_eff(P, g, 0);
    const double ld = NS == 2 ? slot_def(P, g, 0) + slot_def(P, g, 1) : slot_def(P, g, 0);
    Sd = warp_sum_approx(le);
    Dd = warp_sum_approx(ld);
  }
  if (single) {  // node check of u itself
    int dec = decide(P, Sd + P.R[d], Dd, d, cut);
    if (CI && dec == DEC_PASS) {
      const double lb = (Sd + P.R[d]) - P.mb_abs;
      hl = lb < hl ? lb : hl;
    } else if (dec == DEC_EXACT) {
      dec = exact_passes(P, g, G, d, cut) ? DEC_PASS : DEC_PRUNE;
      if (CI && dec == DEC_PASS) hl = cut < hl ? cut : hl;
    }
    if (dec == DEC_PRUNE) {
      if (prefix) o.a_star = du;
      o.finished = true;
      goto done;
    }
  }
  {
    const double kNaN = __longlong_as_double(0x7ff8000000000000LL);
    const double mm_ = P.min_mem, mb = P.mb_abs, md = P.md_abs;
    const int hil = single ? 255 : hi;  // last child at level dtop (single: all of them)
    int c = single ? 0 : (int)sm->path[dpar];  // next child of the current node
    double up = P.p[d], um = P.m[d];  // unit d: assigned by the children
    unsigned long long mp = 0, mr = 0;
    double mc = kNaN;                 // cutoff of mp/mr (NaN: not computed)
    double lS[2] = {0, 0}, lD[2] = {0, 0};  // this lane's children's level sums
    bool sums_ok = false;             // lS/lD belong to the current node
    int match = prefix ? dtop : -1;   // path == end marker on levels < match
    int ec = (prefix && dtop < dend) ? sm->endp[dtop] : -1;  // end child at level `match`
    unsigned it = 0;
    int stop_pending = 0;  // stop flag loaded 32 iterations ago (latency off the chain)

    while (true) {
      HPK_PC(3, 1);
      if ((++it & (HPK_CHECK_EVERY - 1)) == 0) {  // stop flag / time slice
        if ((it & (32 * HPK_CHECK_EVERY - 1)) == 0) {  // wall-clock watchdog (lane 0's clock)
          unsigned long long now;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          now = __shfl_sync(HPK_FULL_MASK, now, 0);
          if (now > *((volatile const unsigned long long*)deadline_slot)) {
            if (lane == 0) atomicOr(err, 2);
            o.finished = true;
            break;
          }
        }
        if (stopf != nullptr) {
          const int s = shfl(stop_pending, 0);  // the queue has drained
          if (lane == 0) stop_pending = *((volatile const int*)stopf);
          if (s) {
            const unsigned long long wave_end = sm->wave_end;
            if (wave_end != 0) {  // ... and the wave's time slice is over: stop
              unsigned long long now;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
              now = __shfl_sync(HPK_FULL_MASK, now, 0);
              if (now > wave_end && o.visits < cap && o.visits > 0) cap = o.visits;
            }
          }
        }
      }
      if (d == n - 1) {
        // ---- leaf batch: children c0..G are leaves (unit n-1) ----
        const int c0 = c;
        const int lim = d == dtop && hil < G ? hil : G;  // last child of this node in the segment
        int count = lim + 1 - c0;
        bool end_hit = false;
        if ((PFX && match == d)) {  // dend == n here
          if (ec - c0 < count) {
            count = ec - c0 > 0 ? ec - c0 : 0;
            end_hit = true;
          }
        }
        bool cap_hit = false;
        if ((long long)count > cap - o.visits) {
          count = (int)(cap - o.visits);
          cap_hit = true;
          end_hit = false;
        }
        if (count > 0) {
          bool inf_k[2] = {false, false};
          double eff_k[2] = {INFINITY, INFINITY};
#pragma unroll
          for (int k = 0; k < NS; ++k) {
            const bool valid = g.gc[k] > 0;
            inf_k[k] = valid && g.gm[k] < mm_;
            eff_k[k] = valid ? slot_eff(P, g, k) : INFINITY;
          }
          const int n_inf = __popc(__ballot_sync(HPK_FULL_MASK, inf_k[0])) +
                            (NS == 2 ? __popc(__ballot_sync(HPK_FULL_MASK, inf_k[1])) : 0);
          // min1 / idx1 / min2 over existing groups. Effective powers are
          // non-negative doubles (empty slots: +inf), whose bit patterns order
          // like the values: two 32-bit redux.sync per 64-bit min, exact.
          const unsigned long long eb0 = (unsigned long long)__double_as_longlong(eff_k[0]);
          const unsigned long long eb1 = (unsigned long long)__double_as_longlong(eff_k[1]);
          const unsigned long long m1b = warp_min_u64(eb0 < eb1 ? eb0 : eb1);
          const double m1 = __longlong_as_double((long long)m1b);
          const unsigned bz0 = __ballot_sync(HPK_FULL_MASK, eb0 == m1b);
          const unsigned bz1 = NS == 2 ? __ballot_sync(HPK_FULL_MASK, eb1 == m1b) : 0u;
          const int i1 = bz0 ? __ffs(bz0) - 1 : 31 + __ffs(bz1);  // lowest index attaining it
          const unsigned long long x0 = lane == i1 ? ~0ull : eb0;
          const unsigned long long x1 = lane + 32 == i1 ? ~0ull : eb1;
          const double m2 = __longlong_as_double((long long)warp_min_u64(x0 < x1 ? x0 : x1));
          if (DRIFT) {  // every visited leaf child does += / -= on its group
#pragma unroll
            for (int k = 0; k < NS; ++k) {
              const int ch = lane + 32 * k;
              if (ch >= c0 && ch < c0 + count && ch < G &&
                  (((g.gp[k] + up) - up) != g.gp[k] || ((g.gm[k] + um) - um) != g.gm[k]))
                g.drift = true;
            }
          }
          // each lane evaluates the children it owns (c = lane, lane+32)
          double obj_s[2] = {-1.0, -1.0};
          int gc_s[2] = {0, 0};
          bool fe_s[2] = {false, false};
#pragma unroll
          for (int k = 0; k < NS; ++k) {
            const int ch = lane + 32 * k;
            const bool isnew = ch == G;  // new singleton group (the slot is empty)
            const double eff_new = (g.gp[k] + up) * HPK_F1(P, g, k);
            const double mem_new = g.gm[k] + um;
            const int others_inf = n_inf - (inf_k[k] ? 1 : 0);
            const double other_min = (!isnew && ch == i1) ? m2 : m1;
            gc_s[k] = isnew ? G + 1 : G;
            fe_s[k] = ch >= c0 && ch < c0 + count && others_inf == 0 && !(mem_new < mm_);
            const double z = eff_new < other_min ? eff_new : other_min;
            obj_s[k] = fe_s[k] ? (double)gc_s[k] * z : -1.0;
          }
          o.visits += count;
          if (TOPK) {
            // max objective of the batch (objectives >= 0; none feasible: -1)
            const bool anyf = __any_sync(HPK_FULL_MASK, fe_s[0] || fe_s[1]);
            double mx = -1.0;
            if (anyf) {
              const double lm = obj_s[0] > obj_s[1] ? obj_s[0] : obj_s[1];
              const unsigned long long lb =
                  lm >= 0 ? (unsigned long long)__double_as_longlong(lm) : 0ull;
              mx = __longlong_as_double((long long)warp_max_u64(lb));
            }
            if (mx >= 0) {
              o.m = mx > o.m ? mx : o.m;
              if (mx > cut) {  // the cutoff state takes every leaf above the cutoff
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                  unsigned b = __ballot_sync(HPK_FULL_MASK, fe_s[k] && obj_s[k] > cut);
                  while (b) {
                    const int l = __ffs(b) - 1;
                    b &= b - 1;
                    const double v = shfl(obj_s[k], l);
                    if (lane == 0) state_insert(sm->T, &sm->nT, tk, v);
                  }
                }
                __syncwarp();
                cut = state_cut(sm->T, sm->nT, tk, floor_);
              }
              // the run's own list: offers in enumeration (child) order
              const int rn = sm->rn;
              const double ko = rn >= tk ? sm->robj[tk - 1] : -1.0;
              const int kg = rn >= tk ? sm->rG[tk - 1] : 0;
              bool any = false;
#pragma unroll
              for (int k = 0; k < NS; ++k) {
                unsigned b = __ballot_sync(HPK_FULL_MASK, fe_s[k] && (rn < tk || rank_better(obj_s[k], gc_s[k], ko, kg)));
                if (b && !any) {
                  __syncwarp();  // lane 0's path spills are visible
                  any = true;
                }
                while (b) {
                  const int l = __ffs(b) - 1;
                  b &= b - 1;
                  const double v = shfl(obj_s[k], l);
                  const int gv = shfl(gc_s[k], l);
                  const int ch = l + 32 * k;
                  cand_insert(sm->robj, sm->rG, rec->rgs, &sm->rn, tk, n, v, gv,
                              [&](int i) { return i < n - 1 ? sm->path[i] : (uint8_t)ch; }, lane);
                }
              }
            }
          } else {
          // the batch's best leaf by the reference ranking (objective desc,
          // #groups asc, enumeration = child order asc): the lane's better child,
          // then a 64-bit max of the objective bits and a min of (G, child)
          // among the lanes attaining it; mx (max objective) is its objective
          double best_o = -1.0;
          int best_Gc = 0, best_c = 1 << 30;
          {
            const bool t0 = fe_s[0] && (!fe_s[1] || key_better(obj_s[0], gc_s[0], lane, obj_s[1],
                                                               gc_s[1], lane + 32));
            const bool has = fe_s[0] || fe_s[1];
            const double lo_ = t0 ? obj_s[0] : obj_s[1];
            const int lg = t0 ? gc_s[0] : gc_s[1];
            const int lc = t0 ? lane : lane + 32;
            if (__any_sync(HPK_FULL_MASK, has)) {
              const unsigned long long lb = has ? (unsigned long long)__double_as_longlong(lo_) : 0ull;
              const unsigned long long bb = warp_max_u64(lb);
              const unsigned key = (has && lb == bb) ? (unsigned)(lg << 7 | lc) : 0xffffffffu;
              const unsigned kmin = __reduce_min_sync(HPK_FULL_MASK, key);
              best_o = __longlong_as_double((long long)bb);
              best_Gc = (int)(kmin >> 7);
              best_c = (int)(kmin & 127);
            }
          }
          const double mx = best_o;
          if (best_o >= 0) {
            if (!o.has_best || best_o > o.best_obj ||
                (best_o == o.best_obj && best_Gc < o.best_G)) {
              o.has_best = true;
              o.best_obj = best_o;
              o.best_G = best_Gc;
              __syncwarp();  // lane 0's path spills are visible
              for (int i = lane; i < n - 1; i += 32) sm->best[i] = sm->path[i];
              if (lane == 0) sm->best[n - 1] = (uint8_t)best_c;
              __syncwarp();
            }
            o.m = mx > o.m ? mx : o.m;
            cut = mx > cut ? mx : cut;
          }
          }
        }
        HPK_PC(1, 1);
        HPK_PC(2, count > 0 ? count : 0);
        if (cap_hit) {
          if (lane == 0) sm->lvl[d] = (unsigned)G << 16;
          o.dstop = d + 1;
          o.stop_c = c0 + count;
          o.finished = false;
          break;
        }
        if (end_hit) {
          o.finished = true;
          break;
        }
        c = lim + 1;
      }
      if (c > (d == dtop && hil < G ? hil : G)) {  // node exhausted: pop unit d-1
        if (d == dtop) {
          o.finished = true;
          break;
        }
        __syncwarp();  // lane 0's spills of this level are visible
        --d;
        const unsigned w0 = sm->lvl[d];  // path | next child << 8 | G << 16
        up = P.p[d];
        um = P.m[d];
        Sd = sm->S[d];
        Dd = sm->DEF[d];
        mp = sm->mpass[d];
        mr = sm->mprune[d];
        mc = sm->mcut[d];
        const int grp = w0 & 255;
        c = (w0 >> 8) & 255;
        G = (w0 >> 16) & 255;
        remove_unit<NS>(P, g, lane, grp, up, um);
        sums_ok = false;
        if (PFX && match > d) match = d;
        if ((PFX && match == d)) ec = sm->endp[d];
        HPK_PC(6, 1);
        continue;
      }
      if ((PFX && match == d)) {
        if (c > ec || (c == ec && d + 1 == dend)) {
          o.finished = true;
          break;
        }
      }
      if (o.visits >= cap) {
        if (lane == 0) sm->lvl[d] = (unsigned)G << 16;
        o.dstop = d + 1;
        o.stop_c = c;
        o.finished = false;
        break;
      }
      // ---- child decisions of this node, lane-parallel (lane ci decides
      // children ci and ci+32), recomputed only when the cutoff moved. The
      // child's level sums follow from the parent's in O(1):
      //   S' = S - eff(ci) + eff'(ci),  DEF' = DEF - def(ci) + def'(ci)
      // (an empty slot ci == G gives eff = 0, eff' = up * f[1]). A child is
      // PRUNE / PASS when the approximate bound and deficit clear the cutoff by
      // more than the error margins mb / md; else it is checked exactly.
      if (mc != cut) {
        const double Rn = P.R[d + 1], RMn = P.RM[d + 1];
        const bool hc = cut >= 0;
        bool pr[2] = {true, true}, ps[2] = {false, false};  // slot 1 unused when NS == 1
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const int ci = lane + 32 * k;
          const double eff_old = g.gp[k] * HPK_F0(P, g, k);
          const double eff_new = (g.gp[k] + up) * HPK_F1(P, g, k);
          const double d0 = mm_ - g.gm[k];
          const double def_old = (g.gc[k] > 0 && d0 > 0.0) ? d0 : 0.0;
          const double d1 = mm_ - (g.gm[k] + um);
          const double def_new = d1 > 0.0 ? d1 : 0.0;
          lS[k] = (Sd - eff_old) + eff_new;
          lD[k] = (Dd - def_old) + def_new;
          const double A = lS[k] + Rn;
          const bool valid = ci <= (d == dtop && hil < G ? hil : G);
          // every visited child, pruned or entered, does += / -= on its group
          // (grouping.cpp:178-199): a round trip that does not restore the sum
          // makes the reference's later sums path dependent
          if (DRIFT && valid && ci < G &&
              (((g.gp[k] + up) - up) != g.gp[k] || ((g.gm[k] + um) - um) != g.gm[k]))
            g.drift = true;
          pr[k] = !valid || (hc && A + mb < cut) || (lD[k] - md > RMn);
          ps[k] = !pr[k] && (!hc || A - mb >= cut) && (lD[k] + md <= RMn);
          if (CI && ps[k]) {
            const double lb = A - mb;
            hl = lb < hl ? lb : hl;
          }
        }
        mp = (unsigned long long)__ballot_sync(HPK_FULL_MASK, ps[0]) |
             (NS == 2 ? ((unsigned long long)__ballot_sync(HPK_FULL_MASK, ps[1]) << 32) : 0ull);
        mr = (unsigned long long)__ballot_sync(HPK_FULL_MASK, pr[0]) |
             (NS == 2 ? ((unsigned long long)__ballot_sync(HPK_FULL_MASK, pr[1]) << 32)
                      : 0xffffffff00000000ull);
        mc = cut;
        sums_ok = true;
        HPK_PC(10, 1);
      }
      const unsigned long long bit = 1ull << c;
      if (mr & bit) {
        // children c .. c+k-1 are all pruned: k visits, nothing entered
        const unsigned long long rest = ~(mr >> c);
        int k = rest ? __ffsll((long long)rest) - 1 : 64 - c;
        const int lim = d == dtop && hil < G ? hil : G;
        if (k > lim + 1 - c) k = lim + 1 - c;
        if ((long long)k > cap - o.visits) k = (int)(cap - o.visits);
        if ((PFX && match == d)) {
          // the end node (d+1 == dend) is not visited; the end path's child is,
          // and its prune is the ancestor prune a* (grouping.cpp:162,169)
          const int kl = (d + 1 == dend) ? ec - c : ec - c + 1;
          if (k > kl) k = kl;
          if (d + 1 < dend && c + k - 1 == ec && o.a_star < 0) o.a_star = d + 1;
        }
        o.visits += k;
        c += k;
        HPK_PC(7, 1);
        HPK_PC(8, k);
        continue;
      }
      o.visits += 1;
      HPK_PC(4, 1);
      if (!(mp & bit)) {  // inside the error margin: the exact serial check
        o.exact += 1;
        add_unit<DRIFT, NS>(P, g, lane, c, up, um);
        const int Gc = c == G ? G + 1 : G;
        const bool pass = exact_passes(P, g, Gc, d + 1, cut);
        remove_unit<NS>(P, g, lane, c, up, um);
        if (!pass) {
          if ((PFX && match == d) && c == ec && o.a_star < 0) o.a_star = d + 1;
          ++c;
          continue;
        }
        if (CI) hl = cut < hl ? cut : hl;
      }
      // ---- PASS: descend into child c
      if (!sums_ok) {  // (after a pop) the lanes recompute their children's sums
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const double eff_old = g.gp[k] * HPK_F0(P, g, k);
          const double eff_new = (g.gp[k] + up) * HPK_F1(P, g, k);
          const double d0 = mm_ - g.gm[k];
          const double def_old = (g.gc[k] > 0 && d0 > 0.0) ? d0 : 0.0;
          const double d1 = mm_ - (g.gm[k] + um);
          const double def_new = d1 > 0.0 ? d1 : 0.0;
          lS[k] = (Sd - eff_old) + eff_new;
          lD[k] = (Dd - def_old) + def_new;
        }
        sums_ok = true;
      }
      const double Sn = shfl((NS == 1 || c < 32) ? lS[0] : lS[1], c & 31);
      const double Dn = shfl((NS == 1 || c < 32) ? lD[0] : lD[1], c & 31);
      if (lane == 0) {  // spill this level
        sm->lvl[d] = (unsigned)c | ((unsigned)(c + 1) << 8) | ((unsigned)G << 16);
        sm->path[d] = (uint8_t)c;
        sm->S[d] = Sd;
        sm->DEF[d] = Dd;
        sm->mpass[d] = mp;
        sm->mprune[d] = mr;
        sm->mcut[d] = mc;
      }
      add_unit<DRIFT, NS>(P, g, lane, c, up, um);
      if (c == G) ++G;
      if ((PFX && match == d) && c == ec) match = d + 1;
      ++d;
      if (MAXN > 64 && G > 63 && d < n) {  // an internal node with 64 groups: 65 children
        o.overflow = true;
        o.finished = true;
        break;
      }
      if (NS == 1 && G > 31 && d < n) {  // 33 children: slot 1 needed, rerun with NS == 2
        o.retry = true;
        o.finished = true;
        break;
      }
      Sd = Sn;
      Dd = Dn;
      c = 0;
      mc = kNaN;
      sums_ok = false;
      up = P.p[d];
      um = P.m[d];
      if ((PFX && match == d)) ec = sm->endp[d];
      HPK_PC(5, 1);
    }
  }
done:
  __syncwarp();
  if (DRIFT) o.drift = __any_sync(HPK_FULL_MASK, g.drift);
  o.hi = CI ? warp_min(hl) : C;
  if (TOPK) {
    const int rn = sm->rn;
    o.has_best = rn > 0;
    if (rn > 0) {
      o.best_obj = sm->robj[0];
      o.best_G = sm->rG[0];
    }
    if (lane < rn) {
      rec->obj[lane] = sm->robj[lane];
      rec->G[lane] = sm->rG[lane];
    }
    if (lane == 0) rec->n = rn;
  } else if (o.has_best) {
    for (int i = lane; i < n; i += 32) Eout->best_rgs[i] = sm->best[i];
  }
  __syncwarp();
  if (prof && lane == 0) {
    pcnt[0] = (unsigned long long)(clock64() - pc0);
#pragma unroll
    for (int k = 0; k < 11; ++k) atomicAdd(prof + k, pcnt[k]);
  }
#undef HPK_PC
  return o;
}

// --------------------------------------------------------------- scheduler

__device__ __forceinline__ bool is_prefix_of(const uint8_t* a, int la, const uint8_t* b, int lb) {
  if (la > lb) return false;
  for (int i = 0; i < la; ++i)
    if (a[i] != b[i]) return false;
  return true;
}

// Split of an unfinished run (warp-level, right after the run): the entry
// becomes the PREFIX record [u, stop) and the remainder of subtree(u) becomes
// new FULL pieces in preorder — subtree(stop), then the right siblings of stop
// and of each of its ancestors down to u's children. Pieces are allocated from
// the problem's entry pool; returns the piece count (0: pool full, run dropped).
__device__ int split_run(const KParams& kp, int p, GState& S, Entry* E, const RunOut& o,
                         WarpSmem* sm, int lane, bool front, int* first_out) {
  const int dpar = E->du - 1;
  const int d = o.dstop - 1;  // the stop node is child stop_c of path[0..d)
  // one range piece per level: lev = d (children stop_c..), then each ancestor
  // level d-1 .. dpar (the children after the path's child), deepest first
  const auto lim = [&](int lev) {
    return lev == dpar ? (int)E->hi : (int)((sm->lvl[lev] >> 16) & 255);
  };
  // kp.ranges == 0: one piece per sibling instead (more, smaller pieces: more
  // parallelism for a few problems; ranges keep big batches' lists short)
  const bool rng = kp.ranges != 0;
  int count = rng ? 1 : 1 + lim(d) - o.stop_c;
  for (int lev = d - 1; lev >= dpar; --lev) {
    const int w = lim(lev) - (int)sm->path[lev];
    count += rng ? (w > 0 ? 1 : 0) : w;
  }
  int first = 0;
  if (lane == 0) {  // CAS bump allocation: a failed attempt leaves no hole, and the
    // list head alone may use the last `reserve` slots (progress guarantee)
    const int limit = kp.pcap - (front ? 0 : kp.reserve);
    int old = *((volatile int*)&S.pool_top);
    while (true) {
      if (old + count > limit) {
        first = -1;
        break;
      }
      const int prev = atomicCAS(&S.pool_top, old, old + count);
      if (prev == old) {
        first = old;
        break;
      }
      old = prev;
    }
  }
  first = shfl(first, 0);
  if (first < 0) return 0;
  Entry* pool = pool_ptr(kp, p, S.pool_cur);
  for (int k = lane; k < count; k += 32) {
    Entry& qe = pool[first + k];
    int lev = d, child = o.stop_c, last;
    if (rng) {
      for (int idx = k; idx > 0;) {  // the k-th non-empty level below d
        --lev;
        if ((int)sm->path[lev] < lim(lev)) {
          --idx;
          child = sm->path[lev] + 1;
        }
      }
      last = lim(lev);
    } else {  // the k-th sibling piece, level by level (deepest first)
      int idx = k, base = o.stop_c - 1, cnt = lim(d) - base;
      while (idx >= cnt) {
        idx -= cnt;
        --lev;
        base = sm->path[lev];
        cnt = lim(lev) - base;
      }
      child = base + 1 + idx;
      last = child;
    }
    Entry& q = pool[first + k];
    for (int i = 0; i < lev; ++i) q.u[i] = sm->path[i];
    q.u[lev] = (uint8_t)child;
    q.du = (uint8_t)(lev + 1);
    q.hi = (uint8_t)last;
    q.kind = KIND_FULL;
    q.cver = -1;
    q.finished = 0;
    q.capped = 0;
    q.uncapped = 0;
    q.has_best = 0;
    q.a_star = -1;
  }
  // the entry itself becomes the prefix record [u, stop)
  for (int i = lane; i < d; i += 32) E->end[i] = sm->path[i];
  if (lane == 0) {
    E->end[d] = (uint8_t)o.stop_c;
    E->dend = (uint8_t)(d + 1);
    E->kind = KIND_PREFIX;
  }
  *first_out = first;
  return count;
}

// Block-wide exclusive scan of src[0..len) into dst (may alias) over tiles of
// blockDim.x * 8 elements: each thread owns 8 consecutive elements, so every
// thread keeps 8 independent loads in flight (the scheduler's passes are
// latency-bound on L2); warp shuffles + one smem round per tile. Returns the total.
template <typename T>
__device__ T block_scan8(const T* src, T* dst, int len, T* sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  T carry = 0;
  for (int base = 0; base < len; base += blockDim.x * 8) {
    const int i0 = base + tid * 8;
    T v[8];
    T sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = i0 + k < len ? src[i0 + k] : (T)0;
      sum += v[k];
    }
    T x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T t = __shfl_up_sync(HPK_FULL_MASK, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    if (warp == 0) {
      T w = lane < nw ? sh[lane] : (T)0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(HPK_FULL_MASK, w, o);
        if (lane >= o) w += t;
      }
      if (lane < nw) sh[lane] = w;
    }
    __syncthreads();
    T run = carry + (warp == 0 ? (T)0 : sh[warp - 1]) + x - sum;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (i0 + k < len) dst[i0 + k] = run;
      run += v[k];
    }
    carry += sh[nw - 1];
    __syncthreads();
  }
  return carry;
}

// TOPK: offer a committed run's own candidates to the global list (one warp;
// the run is later in the enumeration than everything already listed).
__device__ void merge_run_cands(GState& S, const CandRec& r, int tk, int n, int lane) {
  const int rn = r.n;
  for (int t = 0; t < rn; ++t) {
    const double o = r.obj[t];
    const int g = r.G[t];
    const int nb = S.nbest;
    if (nb >= tk && !rank_better(o, g, S.bl_obj[tk - 1], S.bl_G[tk - 1])) break;  // ranked list
    cand_insert(S.bl_obj, S.bl_G, S.bl_rgs, &S.nbest, tk, n, o, g,
                [&](int i) { return r.rgs[t][i]; }, lane);
  }
}
// TOPK: the committed run's leaves join the front's cutoff state (one thread).
__device__ void merge_run_state(GState& S, const CandRec& r, int tk) {
  for (int t = 0; t < r.n; ++t) {
    const double v = r.obj[t];
    if (v > S.seed_obj && v > state_cut(S.T, S.nT, tk, S.seed_obj)) state_insert(S.T, &S.nT, tk, v);
  }
}
__device__ __forceinline__ bool same_state(const CandRec& r, const GState& S) {
  if (r.ntin != S.nT) return false;
  for (int t = 0; t < KW; ++t)
    if (r.tin[t] != S.T[t]) return false;
  return true;
}

__device__ void finish_problem(const KParams& kp, GState& S) {
  S.done = 1;
  atomicSub(kp.active, 1);
  atomicSub(kp.active + 62, S.n_units);  // units of the active problems (queue weights)
}

// Queue the first qmax positions (list order) whose run is missing or used a
// cutoff other than the PREDICTED entering cutoff
//     c^_j = max(C_front, max objective found by the runs before j),
// which equals the exact cutoff whenever those runs are exact (the commit walk
// checks the equality exactly, so a wrong prediction only costs a re-run).
// Positions provably past the budget's abort point are never queued: the
// visits of the exact runs before them (others count 1, a lower bound — a
// higher cutoff only prunes more) already exhaust the budget.
template <typename T, typename Op>
__device__ __forceinline__ T block_excl_scan_1(T x, T ident, T* sh, Op op, T* total) {
  // exclusive scan of one value per thread (thread order), returns the prefix
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  T inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T t = __shfl_up_sync(HPK_FULL_MASK, inc, o);
    if (lane >= o) inc = op(inc, t);
  }
  if (lane == 31) sh[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nw ? sh[lane] : ident;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T t = __shfl_up_sync(HPK_FULL_MASK, w, o);
      if (lane >= o) w = op(w, t);
    }
    if (lane < nw) sh[lane] = w;
  }
  __syncthreads();
  T ex = __shfl_up_sync(HPK_FULL_MASK, inc, 1);
  if (lane == 0) ex = ident;
  if (warp > 0) ex = op(sh[warp - 1], ex);
  *total = sh[nw - 1];
  __syncthreads();
  return ex;
}

struct OpMax {
  __device__ double operator()(double a, double b) const { return a > b ? a : b; }
};
struct OpAddL {
  __device__ long long operator()(long long a, long long b) const { return a + b; }
};
struct OpAddI {
  __device__ int operator()(int a, int b) const { return a + b; }
};

//
// TOPK (tk > 1): the predicted state is a vector (SchedSmem::tv). It is
// constant up to the first position whose run found a leaf above the
// predicted cutoff (an improver); the tile is cut right after it, the
// improver's own candidates are merged into the prediction, and the scan
// resumes. An improver is exact only if it entered with the predicted VECTOR
// (any other run only depends on the cutoff). At most 16 improvers per pass.
__device__ void push_items(const KParams& kp, int queue, int p, const int* ids, const int* pran,
                           const long long* pvis, const double* pcut, const double* pm,
                           const int* pchi,
                           const Entry* pool, int head, int len, double C, int qmax,
                           long long budget_left, long long* shl, double* shd, int* shi,
                           const TileAgg* ag, int nagg, int ashift, SchedSmem* sh, int tk,
                           double floor_, const CandRec* crec, const GState& S) {
  const int tid = threadIdx.x;
  RunQueue* q = kp.queues + queue;
  RunItem* items = kp.items + (size_t)queue * kp.qcap;
  long long before = 0;  // lower bound of visits before the tile
  double cmax = C;       // predicted cutoff entering the tile
  int pushed = 0;
  int ta = 0;  // tile-summary cursor (summaries are at buffer offset -ashift)
  int base = 0;
  const bool topk = tk > 1;
  int n_imp = 0;
  // ramp-up: short runs while the list is young (they split the tree into
  // runnable pieces quickly), the full segment cap after a few waves
  const long long wave_cap = kp.ramp > 0 ? min(kp.seg_cap, (long long)kp.ramp << min(S.waves, 30))
                                         : kp.seg_cap;
  if (topk) {
    if (tid < KW) sh->tv[tid] = S.T[tid];
    if (tid == 0) sh->ntv = S.nT;
    __syncthreads();
  }
  while (base < len) {
    if (nagg) {
      // a summarised tile whose runs are all exact under the predicted cutoff
      // queues nothing: pass it in O(1)
      const int at = head + base;
      while (ta < nagg && ag[ta].ob - ashift + ag[ta].n <= at) ++ta;
      if (ta < nagg && ag[ta].ob - ashift == at) {
        const TileAgg a = ag[ta];
        if (a.nrun == a.n && a.mmax <= cmax &&
            (a.cutc == cmax || (!topk && a.cutx <= cmax && cmax <= a.chimin))) {
          before += a.sumvis;
          base += a.n;
          ++ta;
          if (kp.trace >= 5 && tid == 0) atomicAdd(kp.prof + 19, 1ull);
          if (budget_left >= 0 && before >= budget_left) break;
          continue;
        }
      }
    }
    const int lim = (nagg && ta < nagg) ? min(len, ag[ta].ob - ashift + ag[ta].n - head) : len;
    int jend = base + min(lim - base, (int)blockDim.x * 8);
    const int j0 = base + tid * 8;  // this thread's 8 consecutive positions
    if (kp.trace >= 5 && tid == 0) {
      atomicAdd(kp.prof + 20, 1ull);
      atomicAdd(kp.prof + 21, (unsigned long long)(jend - base));
    }
    bool ran[8];
    double mj[8], cj[8];
    long long vj[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int j = j0 + k;
      ran[k] = j < jend && pran[head + j] == 1;
      mj[k] = ran[k] ? pm[head + j] : -1.0;
      cj[k] = ran[k] ? pcut[head + j] : -2.0;
      vj[k] = ran[k] ? pvis[head + j] : 0;
    }
    int fi_rel = -1;  // TOPK: the tile's first improver (relative to base), -1: none
    if (topk) {
      if (tid == 0) sh->fi = 1 << 30;
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (ran[k] && mj[k] > cmax) {
          atomicMin(&sh->fi, j0 + k - base);
          break;
        }
      __syncthreads();
      if (sh->fi < (1 << 30)) {
        fi_rel = sh->fi;
        jend = base + fi_rel + 1;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (j0 + k >= jend) {
            ran[k] = false;
            mj[k] = -1.0;
          }
      }
      __syncthreads();
    }
    double tmax = -1.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) tmax = mj[k] > tmax ? mj[k] : tmax;
    double tile_max;
    const double exm = block_excl_scan_1<double>(tmax, -1.0, shd, OpMax(), &tile_max);
    double chat[8];
    bool need[8];
    long long vsum = 0;
    {
      double run = cmax > exm ? cmax : exm;
      if (topk) run = cmax;  // constant up to (and including) the improver
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        chat[k] = run;
        if (!topk) run = mj[k] > run ? mj[k] : run;
        bool exact = ran[k] && (cj[k] == chat[k] ||
                                (cj[k] < chat[k] && (!topk || mj[k] <= cj[k]) &&
                                 chat[k] <= __int_as_float(pchi[head + j0 + k])));
        if (topk && exact && j0 + k - base == fi_rel) {  // the improver: compare the vectors
          const CandRec& r = crec[ids[head + j0 + k]];
          bool same = r.ntin == sh->ntv;
          for (int t = 0; t < KW && same; ++t) same = r.tin[t] == sh->tv[t];
          exact = same;
        }
        vj[k] = (j0 + k < jend) ? (exact ? vj[k] : 1) : 0;
        need[k] = (j0 + k < jend) && !exact;
        vsum += vj[k];
      }
    }
    long long tile_vis;
    const long long exv = block_excl_scan_1<long long>(vsum, 0, shl, OpAddL(), &tile_vis);
    int nneed = 0;
    {
      long long run = before + exv;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        need[k] = need[k] && (budget_left < 0 || run < budget_left);
        run += vj[k];
        nneed += need[k] ? 1 : 0;
      }
    }
    int tile_need;
    const int exn = block_excl_scan_1<int>(nneed, 0, shi, OpAddI(), &tile_need);
    if (tid == 0) {
      const int take = min(tile_need, qmax - pushed);
      shi[40] = take;
      shi[41] = take > 0 ? atomicAdd(&q->len, take) : 0;
    }
    __syncthreads();
    const int take = shi[40], slot0 = shi[41];
    int rank = exn;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (need[k]) {
        if (rank < take) {
          if (slot0 + rank >= kp.qcap) {
            atomicOr(kp.err, 4);  // must not happen
          } else {
            const int j = j0 + k;
            RunItem& it = items[slot0 + rank];
            const int id = ids[head + j];
            it.problem = p;
            it.pos = head + j;
            it.id = id;
            it.front = (j == 0);
            // an uncapped (list-full) run is the head's: under a budget it
            // needs at most budget_left + 1 visits to show the overflow
            // the list head is the commit front's critical path: only the time
            // slice bounds its run (kp.front_cap), the others take the segment cap
            it.cap = !pool[id].uncapped ? (j == 0 ? kp.front_cap : wave_cap)
                     : budget_left < 0  ? 0x3fffffffffffffffLL
                                        : budget_left + 1;
            it.cut = chat[k];
            if (topk) {
              it.ntv = sh->ntv;
              for (int t = 0; t < KW; ++t) it.tv[t] = sh->tv[t];
            } else {
              it.ntv = 0;
            }
          }
        }
        ++rank;
      }
    }
    pushed += take;
    before += tile_vis;
    if (!topk) cmax = tile_max > cmax ? tile_max : cmax;
    base = jend;
    __syncthreads();
    if (topk && fi_rel >= 0) {
      // the improver's candidates join the predicted state (a stale run's
      // values are still the best prediction available)
      if (tid == 0) {
        const CandRec& r = crec[ids[head + base - 1]];
        int nt = sh->ntv;
        for (int t = 0; t < r.n; ++t) {
          const double v = r.obj[t];
          if (v > floor_ && v > state_cut(sh->tv, nt, tk, floor_)) state_insert(sh->tv, &nt, tk, v);
        }
        sh->ntv = nt;
      }
      __syncthreads();
      cmax = state_cut(sh->tv, sh->ntv, tk, floor_);
      __syncthreads();
      if (++n_imp >= 16) break;
    }
    if (pushed >= qmax || (budget_left >= 0 && before >= budget_left)) break;
  }
}

// ---- S4: the queue step of the commit CTAs (push_items, k = 1) spread over
// every CTA, one item per list tile (the S2 expansion tiles). The predicted
// cutoff entering tile t is max(C, max objective of the runs in earlier tiles)
// — from the tile summaries alone, so every tile scans itself independently;
// the budget window and the queue share (lower-bound visits and needs before
// the tile) come from the earlier tiles' published aggregates. Items are the
// sequential push's, in per-tile order.
__device__ void push_tile(const KParams& kp, int p, int t, int queue, int wave, SchedSmem* sh) {
  GState& S = kp.states[p];
  const int tid = threadIdx.x;
  if (tid == 0) {
    unsigned ns = 32;
    while (*((volatile int*)&S.pp_wave) != wave) {
      __nanosleep(ns);
      ns = ns < 256 ? ns * 2 : 256;
    }
    __threadfence();
  }
  __syncthreads();
  if (*((volatile int*)&S.pp_mode) != 1 || t >= S.pp_ntile) {
    __syncthreads();
    return;
  }
  const int head = S.pp_head, len = S.pp_len, ashift = S.pp_ashift, qmax = S.pp_qmax;
  const long long bl = S.pp_bl;
  const double C = S.pp_C;
  const TileAgg* ag = kp.agg + (size_t)p * kp.xtn;
  PushAgg* pa = kp.pagg + (size_t)p * kp.xtn;
  const TileAgg a = ag[t];
  const int tlo = a.ob - ashift;
  const int lo = max(tlo, head), hi = min(tlo + a.n, head + len);
  double cin = C;
  for (int u = 0; u < t; ++u) cin = ag[u].mmax > cin ? ag[u].mmax : cin;
  const int cur = S.cur;
  const int* ids = list_arr(kp, p, cur, 0);
  const int* pran = list_arr(kp, p, cur, 1);
  const long long* pvis = list_vis(kp, p, cur);
  const double* pcut = list_dbl(kp, p, cur, 0);
  const double* pm = list_dbl(kp, p, cur, 1);
  const int* pchi = list_arr(kp, p, cur, 5);
  const Entry* pool = pool_ptr(kp, p, S.pool_cur);
  // pass 1: needs and lower-bound visits of the tile
  long long tvis = 0;
  int tneed = 0;
  const bool whole = lo == tlo && hi == tlo + a.n;
  if (whole && a.nrun == a.n && a.mmax <= cin &&
      (a.cutc == cin || (a.cutx <= cin && cin <= a.chimin))) {
    tvis = a.sumvis;  // every run exact under the predicted cutoff
  } else {
    double cmax = cin;
    for (int base = lo; base < hi; base += blockDim.x * 8) {
      const int j0 = base + threadIdx.x * 8;
      bool ran[8];
      double mj[8], cj[8];
      long long vj[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = j0 + k;
        ran[k] = j < hi && pran[j] == 1;
        mj[k] = ran[k] ? pm[j] : -1.0;
        cj[k] = ran[k] ? pcut[j] : -2.0;
        vj[k] = ran[k] ? pvis[j] : 0;
      }
      double tmax = -1.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) tmax = mj[k] > tmax ? mj[k] : tmax;
      double chunk_max;
      const double exm = block_excl_scan_1<double>(tmax, -1.0, sh->d, OpMax(), &chunk_max);
      double run = cmax > exm ? cmax : exm;
      long long v = 0;
      int nn = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (j0 + k < hi) {
          const bool exact =
              ran[k] && (cj[k] == run || (cj[k] < run && run <= __int_as_float(pchi[j0 + k])));
          v += exact ? vj[k] : 1;
          nn += exact ? 0 : 1;
        }
        run = mj[k] > run ? mj[k] : run;
      }
      long long vt;
      int nt;
      block_excl_scan_1<long long>(v, 0, sh->l, OpAddL(), &vt);
      block_excl_scan_1<int>(nn, 0, sh->i, OpAddI(), &nt);
      tvis += vt;
      tneed += nt;
      cmax = chunk_max > cmax ? chunk_max : cmax;
    }
  }
  if (tid == 0) {
    pa[t].nneed = tneed;
    pa[t].vis = tvis;
    __threadfence();
    *((volatile int*)&pa[t].stamp) = wave;
  }
  if (tneed == 0) return;
  // look-back: needs and visits of the earlier tiles
  if (tid < 32) {
    long long bv = 0;
    int bn = 0;
    for (int u = tid; u < t; u += 32) {
      unsigned ns = 32;
      while (*((volatile int*)&pa[u].stamp) != wave) {
        __nanosleep(ns);
        ns = ns < 256 ? ns * 2 : 256;
      }
      __threadfence();
      bv += *((volatile long long*)&pa[u].vis);
      bn += *((volatile int*)&pa[u].nneed);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bv += __shfl_xor_sync(HPK_FULL_MASK, bv, o);
      bn += __shfl_xor_sync(HPK_FULL_MASK, bn, o);
    }
    if (tid == 0) {
      sh->v_before = bv;
      sh->i[50] = bn;
    }
  }
  __syncthreads();
  long long before = sh->v_before;
  int rank0 = sh->i[50];
  __syncthreads();
  if (rank0 >= qmax || (bl >= 0 && before >= bl)) return;
  // pass 2: queue the needing positions inside the budget window, in order
  RunQueue* q = kp.queues + queue;
  RunItem* items = kp.items + (size_t)queue * kp.qcap;
  double cmax = cin;
  for (int base = lo; base < hi; base += blockDim.x * 8) {
    const int j0 = base + threadIdx.x * 8;
    bool ran[8];
    double mj[8], cj[8];
    long long vj[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int j = j0 + k;
      ran[k] = j < hi && pran[j] == 1;
      mj[k] = ran[k] ? pm[j] : -1.0;
      cj[k] = ran[k] ? pcut[j] : -2.0;
      vj[k] = ran[k] ? pvis[j] : 0;
    }
    double tmax = -1.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) tmax = mj[k] > tmax ? mj[k] : tmax;
    double chunk_max;
    const double exm = block_excl_scan_1<double>(tmax, -1.0, sh->d, OpMax(), &chunk_max);
    double chat[8];
    bool need[8];
    long long vsum = 0;
    {
      double run = cmax > exm ? cmax : exm;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        chat[k] = run;
        run = mj[k] > run ? mj[k] : run;
        const bool exact =
            ran[k] &&
            (cj[k] == chat[k] || (cj[k] < chat[k] && chat[k] <= __int_as_float(pchi[j0 + k])));
        vj[k] = (j0 + k < hi) ? (exact ? vj[k] : 1) : 0;
        need[k] = (j0 + k < hi) && !exact;
        vsum += vj[k];
      }
    }
    long long chunk_vis;
    const long long exv = block_excl_scan_1<long long>(vsum, 0, sh->l, OpAddL(), &chunk_vis);
    int nneed = 0;
    {
      long long run = before + exv;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        need[k] = need[k] && (bl < 0 || run < bl);
        run += vj[k];
        nneed += need[k] ? 1 : 0;
      }
    }
    int chunk_need;
    const int exn = block_excl_scan_1<int>(nneed, 0, sh->i, OpAddI(), &chunk_need);
    if (tid == 0) {
      const int take = max(0, min(chunk_need, qmax - rank0));
      sh->i[40] = take;
      sh->i[41] = take > 0 ? atomicAdd(&q->len, take) : 0;
    }
    __syncthreads();
    const int take = sh->i[40], slot0 = sh->i[41];
    int r = exn;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (need[k]) {
        if (r < take) {
          if (slot0 + r >= kp.qcap) {
            atomicOr(kp.err, 4);  // must not happen
          } else {
            const int j = j0 + k;
            RunItem& it = items[slot0 + r];
            const int id = ids[j];
            it.problem = p;
            it.pos = j;
            it.id = id;
            it.front = (j == head);
            it.cap = !pool[id].uncapped ? (j == head ? kp.front_cap : kp.seg_cap)
                     : bl < 0           ? 0x3fffffffffffffffLL
                                        : bl + 1;
            it.cut = chat[k];
            it.ntv = 0;
          }
        }
        ++r;
      }
    }
    rank0 += take;
    before += chunk_vis;
    cmax = chunk_max > cmax ? chunk_max : cmax;
    __syncthreads();
    if (rank0 >= qmax || (bl >= 0 && before >= bl)) break;
  }
}

// ---- list expansion, spread over every CTA (schedule step S2). The list of a
// problem is cut into tiles of TILE positions; the runners added the piece
// counts of their splits to xt[tile] (atomic), so a tile's output offset is
// known from the tile counts alone: tiles without splits are shifted copies,
// the others scan their expansion counts. A nearly full list (the revert rule
// needs the whole list in order) is left to the problem's own CTA (S3).
__device__ __forceinline__ int xt_sums(const int* xt, int ntile, int t, SchedSmem* sh, int* before) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    int b = 0, a = 0;
    for (int k = tid; k < ntile; k += 32) {
      const int x = xt[k];
      a += x;
      if (k < t) b += x;
    }
    b = warp_sum_int(b);
    a = warp_sum_int(a);
    if (tid == 0) {
      sh->i[60] = b;
      sh->i[61] = a;
    }
  }
  __syncthreads();
  *before = sh->i[60];
  const int all = sh->i[61];
  __syncthreads();
  return all;
}

// Per-thread accumulator of a TileAgg, reduced over the CTA.
struct AggAcc {
  int nrun, ndel;
  long long sumvis;
  double mmax, cmin, cmax, bo;
  float chimin;
  int bg, bi;
  __device__ void init() {
    chimin = INFINITY;
    nrun = 0;
    ndel = 0;
    sumvis = 0;
    mmax = -1.0;
    cmin = INFINITY;
    cmax = -INFINITY;
    bo = -1.0;
    bg = 0;
    bi = 0x7fffffff;
  }
  __device__ void add(int pc, int inf, long long vis, double cut, double m, double bobj, int pos,
                      float chi) {
    if (pc != 1) return;
    chimin = chi < chimin ? chi : chimin;
    ++nrun;
    ndel += (inf & 512) ? 1 : 0;
    sumvis += vis;
    mmax = m > mmax ? m : mmax;
    cmin = cut < cmin ? cut : cmin;
    cmax = cut > cmax ? cut : cmax;
    if (inf & 256) {
      const int g = inf & 255;
      if (bo < 0 || key_better(bobj, g, pos, bo, bg, bi)) {
        bo = bobj;
        bg = g;
        bi = pos;
      }
    }
  }
  __device__ void merge(const AggAcc& o) {
    nrun += o.nrun;
    ndel += o.ndel;
    sumvis += o.sumvis;
    mmax = o.mmax > mmax ? o.mmax : mmax;
    cmin = o.cmin < cmin ? o.cmin : cmin;
    cmax = o.cmax > cmax ? o.cmax : cmax;
    chimin = o.chimin < chimin ? o.chimin : chimin;
    if (o.bo >= 0 && (bo < 0 || key_better(o.bo, o.bg, o.bi, bo, bg, bi))) {
      bo = o.bo;
      bg = o.bg;
      bi = o.bi;
    }
  }
  __device__ void shfl_merge(int off) {
    AggAcc o;
    o.nrun = __shfl_xor_sync(HPK_FULL_MASK, nrun, off);
    o.ndel = __shfl_xor_sync(HPK_FULL_MASK, ndel, off);
    o.sumvis = __shfl_xor_sync(HPK_FULL_MASK, sumvis, off);
    o.mmax = __shfl_xor_sync(HPK_FULL_MASK, mmax, off);
    o.cmin = __shfl_xor_sync(HPK_FULL_MASK, cmin, off);
    o.cmax = __shfl_xor_sync(HPK_FULL_MASK, cmax, off);
    o.chimin = __shfl_xor_sync(HPK_FULL_MASK, chimin, off);
    o.bo = __shfl_xor_sync(HPK_FULL_MASK, bo, off);
    o.bg = __shfl_xor_sync(HPK_FULL_MASK, bg, off);
    o.bi = __shfl_xor_sync(HPK_FULL_MASK, bi, off);
    merge(o);
  }
};

// CTA reduction of the accumulators; thread 0 writes the tile summary.
__device__ void write_tile_agg(AggAcc acc, TileAgg* out, int ob, int n, SchedSmem* sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc.shfl_merge(off);
  AggAcc* part = reinterpret_cast<AggAcc*>(sh->part);
  if (lane == 0) part[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) acc.merge(part[w]);
    TileAgg a;
    a.ob = ob;
    a.n = n;
    a.nrun = acc.nrun;
    a.ndel = acc.ndel;
    a.mmax = acc.mmax;
    a.cutc = (acc.nrun > 0 && acc.cmin == acc.cmax) ? acc.cmin
                                                     : __longlong_as_double(0x7ff8000000000000LL);
    a.cutx = acc.nrun > 0 ? acc.cmax : __longlong_as_double(0x7ff8000000000000LL);
    a.chimin = (double)acc.chimin;
    a.sumvis = acc.sumvis;
    a.bobj = acc.bo;
    a.bG = acc.bg;
    a.bidx = acc.bi;
    *out = a;
  }
  __syncthreads();
}

__device__ void expand_tile(const KParams& kp, int p, int t, SchedSmem* sh) {
  const GState& S = kp.states[p];
  const int tid = threadIdx.x;
  if (S.done || S.rerun_pending) return;
  const int cur = S.cur, head = S.head, len = S.len;
  const int ntile = (len + TILE - 1) / TILE;
  const int* xt = kp.xt + (size_t)p * kp.xtn;
  int ebase = 0;
  const int etot = xt_sums(xt, ntile, t, sh, &ebase);
  if (len + etot > kp.lcap - kp.reserve) return;
  const int lo = t * TILE, n = min(TILE, len - lo);
  const int* __restrict__ ids_i = list_arr(kp, p, cur, 0) + head + lo;
  const int* __restrict__ pcv_i = list_arr(kp, p, cur, 1) + head + lo;
  const int* __restrict__ cnt_i = list_arr(kp, p, cur, 2) + head + lo;
  const int* __restrict__ pf_i = list_arr(kp, p, cur, 3) + head + lo;
  const int* __restrict__ inf_i = list_arr(kp, p, cur, 4) + head + lo;
  const int* __restrict__ chi_i = list_arr(kp, p, cur, 5) + head + lo;
  const long long* __restrict__ vis_i = list_vis(kp, p, cur) + head + lo;
  const double* __restrict__ cut_i = list_dbl(kp, p, cur, 0) + head + lo;
  const double* __restrict__ m_i = list_dbl(kp, p, cur, 1) + head + lo;
  const double* __restrict__ bo_i = list_dbl(kp, p, cur, 2) + head + lo;
  const int ob = lo + ebase;  // output position of the tile's first entry
  int* __restrict__ ids_o = list_arr(kp, p, cur ^ 1, 0) + ob;
  int* __restrict__ pcv_o = list_arr(kp, p, cur ^ 1, 1) + ob;
  int* __restrict__ cnt_o = list_arr(kp, p, cur ^ 1, 2) + ob;
  int* __restrict__ inf_o = list_arr(kp, p, cur ^ 1, 4) + ob;
  int* __restrict__ chi_o = list_arr(kp, p, cur ^ 1, 5) + ob;
  long long* __restrict__ vis_o = list_vis(kp, p, cur ^ 1) + ob;
  double* __restrict__ cut_o = list_dbl(kp, p, cur ^ 1, 0) + ob;
  double* __restrict__ m_o = list_dbl(kp, p, cur ^ 1, 1) + ob;
  double* __restrict__ bo_o = list_dbl(kp, p, cur ^ 1, 2) + ob;
  AggAcc acc;
  acc.init();
  const int xtt = xt[t];
  if (xtt == 0) {  // no split in this tile: shifted copy
#pragma unroll 4
    for (int i = tid; i < n; i += blockDim.x) {
      const int id = ids_i[i], pc = pcv_i[i], inf = inf_i[i], ch = chi_i[i];
      const long long vv = vis_i[i];
      const double cu = cut_i[i], mm = m_i[i], bb = bo_i[i];
      ids_o[i] = id;
      pcv_o[i] = pc;
      inf_o[i] = inf;
      chi_o[i] = ch;
      vis_o[i] = vv;
      cut_o[i] = cu;
      m_o[i] = mm;
      bo_o[i] = bb;
      cnt_o[i] = 1;
      acc.add(pc, inf, vv, cu, mm, bb, ob + i, __int_as_float(ch));
    }
    write_tile_agg(acc, kp.agg + (size_t)p * kp.xtn + t, ob, n, sh);
    return;
  }
  int* off = kp.scratch + (size_t)p * (kp.lcap + 1) + lo;
  const int tsum = block_scan8<int>(cnt_i, off, n, sh->i);
  __syncthreads();
  const int* __restrict__ o_ = off;
  // 4 consecutive inputs per thread, all loads issued before the stores
  for (int i0 = tid * 4; i0 < n; i0 += blockDim.x * 4) {
    int o[5], id[4], pc[4], inf[4], ch[4];
    long long vv[4];
    double cu[4], mm[4], bb[4];
#pragma unroll
    for (int k = 0; k < 5; ++k) o[k] = i0 + k < n ? o_[i0 + k] : tsum;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + k < n ? i0 + k : i0;
      id[k] = ids_i[i];
      pc[k] = pcv_i[i];
      inf[k] = inf_i[i];
      ch[k] = chi_i[i];
      vv[k] = vis_i[i];
      cu[k] = cut_i[i];
      mm[k] = m_i[i];
      bb[k] = bo_i[i];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (i0 + k < n) {
        const int q = o[k];
        ids_o[q] = id[k];
        pcv_o[q] = pc[k];
        inf_o[q] = inf[k];
        chi_o[q] = ch[k];
        vis_o[q] = vv[k];
        cut_o[q] = cu[k];
        m_o[q] = mm[k];
        bo_o[q] = bb[k];
        cnt_o[q] = 1;
        acc.add(pc[k], inf[k], vv[k], cu[k], mm[k], bb[k], ob + q, __int_as_float(ch[k]));
        const int c = o[k + 1] - q;
        if (c > 1) {
          const int pf = pf_i[i0 + k];
          for (int tt = 1; tt < c; ++tt) {
            ids_o[q + tt] = pf + tt - 1;
            pcv_o[q + tt] = -1;
            inf_o[q + tt] = 0;
            chi_o[q + tt] = 0;
            vis_o[q + tt] = 0;
            cut_o[q + tt] = -1.0;
            m_o[q + tt] = -1.0;
            bo_o[q + tt] = -1.0;
            cnt_o[q + tt] = 1;
          }
        }
      }
    }
  }
  write_tile_agg(acc, kp.agg + (size_t)p * kp.xtn + t, ob, tsum, sh);
}

// Per-problem scheduler (one CTA): expand splits, ordered commit, compaction,
// queue the next wave.
__device__ void publish_push(GState& S, int mode, int wave) {
  S.pp_mode = mode;
  __threadfence();
  *((volatile int*)&S.pp_wave) = wave;
}

__device__ void schedule_problem(const KParams& kp, int p, int next_queue, void* smem_tmp,
                                 int wnext, int wave) {
  GState& S = kp.states[p];
  const GProb& P = kp.probs[p];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (S.done) {
    if (tid == 0) publish_push(S, 0, wave);
    return;
  }
  const int cur = S.cur, head = S.head, len = S.len;
  int* ids_in = list_arr(kp, p, cur, 0);
  int* pcv_in = list_arr(kp, p, cur, 1);
  int* cnt_in = list_arr(kp, p, cur, 2);
  int* pf_in = list_arr(kp, p, cur, 3);
  int* ids_out = list_arr(kp, p, cur ^ 1, 0);
  int* pcv_out = list_arr(kp, p, cur ^ 1, 1);
  int* cnt_out = list_arr(kp, p, cur ^ 1, 2);
  long long* vis_in = list_vis(kp, p, cur);
  long long* vis_out = list_vis(kp, p, cur ^ 1);
  double* cut_in = list_dbl(kp, p, cur, 0);
  double* m_in = list_dbl(kp, p, cur, 1);
  double* cut_out = list_dbl(kp, p, cur ^ 1, 0);
  double* m_out = list_dbl(kp, p, cur ^ 1, 1);
  int* inf_in = list_arr(kp, p, cur, 4);
  int* inf_out = list_arr(kp, p, cur ^ 1, 4);
  int* chi_in = list_arr(kp, p, cur, 5);
  int* chi_out = list_arr(kp, p, cur ^ 1, 5);
  double* bo_in = list_dbl(kp, p, cur, 2);
  double* bo_out = list_dbl(kp, p, cur ^ 1, 2);
  Entry* pool = pool_ptr(kp, p, S.pool_cur);

  const int tk = P.top_k;
  const bool topk = tk > 1;
  const CandRec* crec = topk ? cand_ptr(kp, p, S.pool_cur) : nullptr;
  if (S.rerun_pending) {
    // the capped re-run of the overflow segment (at the head) is back
    if (topk) {
      if (warp == 0) merge_run_cands(S, crec[ids_in[head]], tk, P.n, lane);
      __syncthreads();
    }
    if (tid == 0) {
      const Entry& e = pool[ids_in[head]];
      if (!topk && e.has_best && (!S.has_best || e.best_obj > S.best_obj ||
                         (e.best_obj == S.best_obj && e.best_G < S.best_G))) {
        S.has_best = 1;
        S.best_obj = e.best_obj;
        S.best_G = e.best_G;
        for (int i = 0; i < P.n; ++i) S.best_rgs[i] = e.best_rgs[i];
      }
      S.V = P.budget;
      S.aborted = 1;
      S.rerun_pending = 0;
      finish_problem(kp, S);
      publish_push(S, 0, wave);
    }
    __syncthreads();
    return;
  }

  unsigned long long _tprev = 0;
  if (kp.trace >= 5 && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_tprev));
  // ---- A. expand the splits made by this wave's runs (cnt = 1 + pieces).
  // Normally done by expand_tile() over every CTA (S2); a nearly full list is
  // expanded here, in order, with the revert rule.
  SchedSmem* sh = reinterpret_cast<SchedSmem*>(smem_tmp);
  int* xt = kp.xt + (size_t)p * kp.xtn;
  const int ntile = (len + TILE - 1) / TILE;
  int xt_before;
  const int etot = xt_sums(xt, ntile, 0, sh, &xt_before);
  for (int k = tid; k < ntile; k += blockDim.x) xt[k] = 0;  // re-armed for the next wave
  int total;
  int nagg = 0;  // tile summaries of the new list (valid when expand_tile() expanded it)
  const TileAgg* ag = kp.agg + (size_t)p * kp.xtn;
  if (len + etot <= kp.lcap - kp.reserve) {
    total = len + etot;  // expanded by expand_tile()
    nagg = ntile;
  } else {
    const int mr = len;
    int* off = kp.scratch + (size_t)p * (kp.lcap + 1);
    int total_run = block_scan8<int>(cnt_in + head, off, mr, sh->i);
    if (total_run + (len - mr) > kp.lcap - kp.reserve) {
      // List nearly full: expansions are kept in list order while the list still
      // leaves the head's reserve free (the inclusive count of extra entries is
      // monotone, so the kept ones form a prefix); the others are reverted to
      // unrun FULL segments (their pieces become garbage). If even the head cannot
      // expand it re-runs uncapped (finishes in one run) — progress is guaranteed.
      for (int i = tid; i < mr; i += blockDim.x) {
        const int nx = i + 1 < mr ? off[i + 1] : total_run;
        int c = nx - off[i];
        if (c > 1) {
          const int incl_extra = nx - (i + 1);
          const int limit = (i == 0 ? kp.lcap : kp.lcap - kp.reserve) - len;
          if (incl_extra > limit) {
            c = 1;
            Entry& e = pool[ids_in[head + i]];
            e.kind = KIND_FULL;
            e.cver = -1;
            e.finished = 0;
            if (i == 0) e.uncapped = 1;
            pcv_in[head + i] = -1;
          }
        }
        cnt_in[head + i] = c;
      }
      __syncthreads();
      total_run = block_scan8<int>(cnt_in + head, off, mr, sh->i);
    }
    total = total_run + (len - mr);
    if (tid == 0) off[mr] = total_run;
    __syncthreads();
    {
      const int* __restrict__ o_ = off;
      const int* __restrict__ ids_i = ids_in + head;
      const int* __restrict__ pcv_i = pcv_in + head;
      const int* __restrict__ inf_i = inf_in + head;
      const int* __restrict__ chi_i = chi_in + head;
      const int* __restrict__ pf_i = pf_in + head;
      const long long* __restrict__ vis_i = vis_in + head;
      const double* __restrict__ cut_i = cut_in + head;
      const double* __restrict__ m_i = m_in + head;
      const double* __restrict__ bo_i = bo_in + head;
      int* __restrict__ ids_o = ids_out;
      int* __restrict__ pcv_o = pcv_out;
      int* __restrict__ inf_o = inf_out;
      int* __restrict__ chi_o = chi_out;
      int* __restrict__ cnt_o = cnt_out;
      long long* __restrict__ vis_o = vis_out;
      double* __restrict__ cut_o = cut_out;
      double* __restrict__ m_o = m_out;
      double* __restrict__ bo_o = bo_out;
      // run region: 4 consecutive inputs per thread, all loads issued before the stores
      for (int i0 = tid * 4; i0 < mr; i0 += blockDim.x * 4) {
        int o[5], id[4], pc[4], inf[4], ch[4];
        long long vv[4];
        double cu[4], mm[4], bb[4];
  #pragma unroll
        for (int k = 0; k < 5; ++k) o[k] = i0 + k <= mr ? o_[i0 + k] : 0;
  #pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = i0 + k < mr ? i0 + k : i0;
          id[k] = ids_i[i];
          pc[k] = pcv_i[i];
          inf[k] = inf_i[i];
          ch[k] = chi_i[i];
          vv[k] = vis_i[i];
          cu[k] = cut_i[i];
          mm[k] = m_i[i];
          bb[k] = bo_i[i];
        }
  #pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (i0 + k < mr) {
            const int q = o[k];
            ids_o[q] = id[k];
            pcv_o[q] = pc[k];
            inf_o[q] = inf[k];
            chi_o[q] = ch[k];
            vis_o[q] = vv[k];
            cut_o[q] = cu[k];
            m_o[q] = mm[k];
            bo_o[q] = bb[k];
            cnt_o[q] = 1;
            const int c = o[k + 1] - q;
            if (c > 1) {
              const int pf = pf_i[i0 + k];
              for (int t = 1; t < c; ++t) {
                ids_o[q + t] = pf + t - 1;
                pcv_o[q + t] = -1;
                inf_o[q + t] = 0;
                chi_o[q + t] = 0;
                vis_o[q + t] = 0;
                cut_o[q + t] = -1.0;
                m_o[q + t] = -1.0;
                bo_o[q + t] = -1.0;
                cnt_o[q + t] = 1;
              }
            }
          }
        }
      }
      // tail: shifted copy
      const int delta = total_run - mr;
  #pragma unroll 4
      for (int i = mr + tid; i < len; i += blockDim.x) {
        const int q = i + delta;
        ids_o[q] = ids_i[i];
        pcv_o[q] = pcv_i[i];
        inf_o[q] = inf_i[i];
        chi_o[q] = chi_i[i];
        vis_o[q] = vis_i[i];
        cut_o[q] = cut_i[i];
        m_o[q] = m_i[i];
        bo_o[q] = bo_i[i];
        cnt_o[q] = 1;
      }
    }
    __syncthreads();
  }
  if (kp.trace >= 5 && tid == 0) {
    unsigned long long _t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));
    atomicAdd(kp.prof + 12, _t - _tprev);
    _tprev = _t;
  }
  // ---- B. ordered commit walk, block-parallel over tiles of 8 positions per
  // thread. Walking the list in order, position j commits iff its run is
  // exact: it ran with the cutoff the serial DFS has on entering it,
  //     C_j = max(C_front, max m over the committed positions before j)
  // (a prefix max — improvements need no stop). A tile stops at the first
  // position that is not exact, or right after a PREFIX whose re-run pruned an
  // ancestor (it deletes the pieces under that ancestor) or the position where
  // the budget runs out (grouping.cpp:174-177).
  double C = S.C;
  int cver = S.cver;
  long long V = S.V;
  const long long B = P.budget;
  int i = 0;
  int done = 0, aborted = 0, rerun = 0;
  long long rerun_cap = 0;
  int ta = 0;  // tile-summary cursor
  while (i < total) {
    if (nagg) {
      // whole summarised tiles commit in O(1) when every position ran with the
      // cutoff C, none improves on it, none deletes and the budget is not reached
      while (ta < nagg && ag[ta].ob + ag[ta].n <= i) ++ta;
      if (ta < nagg && ag[ta].ob == i) {
        const TileAgg a = ag[ta];
        if (a.nrun == a.n && a.ndel == 0 && a.mmax <= C &&
            (a.cutc == C || (!topk && a.cutx <= C && C <= a.chimin)) &&
            (B < 0 || V + a.sumvis < B) &&
            (!topk || a.bobj < 0 ||
             (S.nbest >= tk && !rank_better(a.bobj, a.bG, S.bl_obj[tk - 1], S.bl_G[tk - 1])))) {
          if (!topk && a.bobj >= 0 && tid < 32) {
            const int gh = S.has_best;
            const double gbo = S.best_obj;
            const int gbg = S.best_G;
            if (!gh || a.bobj > gbo || (a.bobj == gbo && a.bG < gbg)) {
              const Entry& w = pool[ids_out[a.bidx]];
              for (int t = lane; t < P.n; t += 32) S.best_rgs[t] = w.best_rgs[t];
              if (lane == 0) {
                S.has_best = 1;
                S.best_obj = a.bobj;
                S.best_G = a.bG;
              }
            }
          }
          V += a.sumvis;
          i += a.n;
          ++ta;
          if (kp.trace >= 5 && tid == 0) atomicAdd(kp.prof + 22, 1ull);
          __syncthreads();
          continue;
        }
      }
    }
    const int lim = (nagg && ta < nagg) ? ag[ta].ob + ag[ta].n : total;
    const int tile = min(lim - i, (int)blockDim.x * 8);
    if (kp.trace >= 5 && tid == 0) atomicAdd(kp.prof + 23, 1ull);
    const int r0 = tid * 8;  // this thread's positions, relative to i
    int pc[8], inf[8];
    double cu[8], mm[8];
    float ch[8];
    long long vv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = r0 + k;
      const int j = i + (r < tile ? r : 0);
      pc[k] = r < tile ? pcv_out[j] : 0;
      cu[k] = cut_out[j];
      ch[k] = __int_as_float(chi_out[j]);
      mm[k] = m_out[j];
      vv[k] = vis_out[j];
      inf[k] = inf_out[j];
    }
    double tmax = -1.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (pc[k] == 1) tmax = mm[k] > tmax ? mm[k] : tmax;
    double dummy_d;
    const double exm = block_excl_scan_1<double>(tmax, -1.0, sh->d, OpMax(), &dummy_d);
    bool ok[8];
    double cafter[8];
    long long vsum = 0;
    {
      double run = C > exm ? C : exm;
      if (topk) run = C;  // improvers end the tile (below)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        // (top_k > 1: only a run that found no leaf above its entering cutoff
        // depends on that scalar alone; an improver needs the front's vector)
        ok[k] = pc[k] == 1 &&
                (cu[k] == run || (cu[k] < run && run <= ch[k] && (!topk || mm[k] <= cu[k])));
        if (topk && ok[k] && mm[k] > C)  // an improver is exact only with the front's vector
          ok[k] = same_state(crec[ids_out[i + r0 + k]], S);
        if (pc[k] == 1 && !topk) run = mm[k] > run ? mm[k] : run;
        cafter[k] = run;
        vsum += ok[k] ? vv[k] : 0;
      }
    }
    long long dummy_l;
    const long long exv = block_excl_scan_1<long long>(vsum, 0, sh->l, OpAddL(), &dummy_l);
    int fb = 1 << 30, fs = 1 << 30;
    long long cum[8];
    {
      long long run = V + exv;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        run += ok[k] ? vv[k] : 0;
        cum[k] = run;
        const int r = r0 + k;
        if (!ok[k] && r < fb) fb = r;
        const bool del = (inf[k] & 512) != 0;
        const bool over = B >= 0 && run >= B;
        const bool imp = topk && mm[k] > C;
        if (ok[k] && (del || over || imp) && r < fs) fs = r;
      }
    }
    if (fb > tile) fb = tile;
    if (tid == 0) {
      sh->fb = 1 << 30;
      sh->fs = 1 << 30;
    }
    __syncthreads();
    atomicMin(&sh->fb, fb);
    atomicMin(&sh->fs, fs);
    __syncthreads();
    const int FB = sh->fb, FS = sh->fs;
    const bool special_last = FS < FB;
    const int kc = special_last ? FS + 1 : FB;  // relative positions [0, kc) are processed
    // the thread owning position kc-1 publishes the state after it
    if (kc > 0 && (kc - 1) >> 3 == tid) {
      const int k = (kc - 1) & 7;
      sh->v_after = cum[k];
      sh->c_after = cafter[k];
      sh->v_before = cum[k] - vv[k];
      sh->c_before = k > 0 ? cafter[k - 1] : (C > exm ? C : exm);
      sh->sp_del = (inf[k] & 512) != 0;
      sh->sp_imp = topk && mm[k] > C;
    }
    __syncthreads();
    bool overflow = false;  // budget runs out INSIDE the special position: re-run it capped
    if (special_last && B >= 0 && sh->v_after > B) overflow = true;
    const int kcommit = overflow ? kc - 1 : kc;
    // best over the committed positions: (obj desc, G asc, position asc)
    if (topk) {
      // positions whose best candidate could enter the global list, in order
      const int nb = S.nbest;
      const double ko = nb >= tk ? S.bl_obj[tk - 1] : -1.0;
      const int kg = nb >= tk ? S.bl_G[tk - 1] : 0;
      bool qk[8];
      int nql = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = r0 + k;
        qk[k] = r < kcommit && (inf[k] & 256) &&
                (nb < tk || rank_better(bo_out[i + r], inf[k] & 255, ko, kg));
        nql += qk[k] ? 1 : 0;
      }
      int nqt;
      int qo = block_excl_scan_1<int>(nql, 0, sh->i, OpAddI(), &nqt);
      if (nqt > 0) {
        // (the problem's scan scratch is free during the commit walk)
        int* qpos = kp.scratch + (size_t)p * (kp.lcap + 1);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (qk[k]) qpos[qo++] = r0 + k;
        __syncthreads();
        if (warp == 0)
          for (int t = 0; t < nqt; ++t)
            merge_run_cands(S, crec[ids_out[i + qpos[t]]], tk, P.n, lane);
        __syncthreads();
      }
    } else {
      double ko = -1;
      int kg = 0, ki = 1 << 30;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = r0 + k;
        if (r < kcommit && (inf[k] & 256)) {
          const double bo = bo_out[i + r];
          const int bg = inf[k] & 255;
          if (ko < 0 || key_better(bo, bg, r, ko, kg, ki)) {
            ko = bo;
            kg = bg;
            ki = r;
          }
        }
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) {
        const double oo = __shfl_xor_sync(HPK_FULL_MASK, ko, o2);
        const int og = __shfl_xor_sync(HPK_FULL_MASK, kg, o2);
        const int oi = __shfl_xor_sync(HPK_FULL_MASK, ki, o2);
        if (oo >= 0 && (ko < 0 || key_better(oo, og, oi, ko, kg, ki))) {
          ko = oo;
          kg = og;
          ki = oi;
        }
      }
      if (lane == 0) {
        sh->bo[warp] = ko;
        sh->bg[warp] = kg;
        sh->bi[warp] = ki;
      }
      __syncthreads();
      if (warp == 0) {
        const int nw = blockDim.x >> 5;
        ko = lane < nw ? sh->bo[lane] : -1.0;
        kg = lane < nw ? sh->bg[lane] : 0;
        ki = lane < nw ? sh->bi[lane] : (1 << 30);
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) {
          const double oo = __shfl_xor_sync(HPK_FULL_MASK, ko, o2);
          const int og = __shfl_xor_sync(HPK_FULL_MASK, kg, o2);
          const int oi = __shfl_xor_sync(HPK_FULL_MASK, ki, o2);
          if (oo >= 0 && (ko < 0 || key_better(oo, og, oi, ko, kg, ki))) {
            ko = oo;
            kg = og;
            ki = oi;
          }
        }
        const int gh = S.has_best;
        const double gbo = S.best_obj;
        const int gbg = S.best_G;
        if (ko >= 0 && (!gh || ko > gbo || (ko == gbo && kg < gbg))) {
          const Entry& w = pool[ids_out[i + ki]];
          for (int t = lane; t < P.n; t += 32) S.best_rgs[t] = w.best_rgs[t];
          if (lane == 0) {
            S.has_best = 1;
            S.best_obj = ko;
            S.best_G = kg;
          }
        }
      }
    }
    if (topk && special_last && kcommit == kc && sh->sp_imp) {
      // the committed improver's leaves raise the front's cutoff state
      if (tid == 0) {
        merge_run_state(S, crec[ids_out[i + kc - 1]], tk);
        sh->c_after = state_cut(S.T, S.nT, tk, S.seed_obj);
      }
      __syncthreads();
    }
    if (kcommit > 0) {
      const double cn = (kcommit == kc) ? sh->c_after : sh->c_before;
      V = (kcommit == kc) ? sh->v_after : sh->v_before;
      if (cn > C) {
        C = cn;
        ++cver;
      }
    }
    i += kcommit;
    if (overflow) {
      rerun = 1;
      rerun_cap = B - V;
      __syncthreads();
      break;
    }
    if (special_last) {
      const int jl = i - 1;  // the special entry, now committed
      if (sh->sp_del) {
        if (warp == 0) {
          const Entry& e = pool[ids_out[jl]];
          const int la = e.a_star;
          int ndel = 0;
          for (int base = jl + 1; base < total; base += 32) {
            const int t = base + lane;
            bool inside = false;
            if (t < total) {
              const Entry& f = pool[ids_out[t]];
              inside = is_prefix_of(e.end, la, f.u, f.du);
            }
            const unsigned bin = __ballot_sync(HPK_FULL_MASK, inside);
            const int firstout = (~bin) ? __ffs(~bin) - 1 : 32;
            ndel += firstout;
            if (firstout < 32) break;
          }
          if (lane == 0) sh->ndel = ndel;
        }
        __syncthreads();
        i += sh->ndel;
      }
      __syncthreads();
      if (B >= 0 && V == B) {
        done = 1;
        aborted = i < total ? 1 : 0;
        break;
      }
      continue;  // every later position is re-checked against the updated C
    }
    __syncthreads();
    if (kc < tile) break;  // reached a position that still needs a run
  }
  if (tid == 0) {
    if (kp.trace && kp.trace < 5 && (kp.trace_p < 0 || kp.trace_p == p) && S.waves < 200000)
      printf("[hpk] wave %d p %d len %d total %d extra %d commit %d V %lld C %.17g pool %d "
             "head-pcv %d head-cut %.17g head-uncapped %d\n",
             S.waves, p, len, total, etot, i, V, C, S.pool_top, total > i ? pcv_out[i] : -9,
             total > i ? cut_out[i] : -9.0, total > i ? (int)pool[ids_out[i]].uncapped : -9);
    S.C = C;
    S.cver = cver;
    S.V = V;
    S.cur = cur ^ 1;
    S.head = i;
    S.len = total - i;
    S.waves += 1;
    S.max_list = max(S.max_list, total);
    if (rerun) {
      S.rerun_pending = 1;
      S.rerun_cap = rerun_cap;
    }
    if (done) {
      S.aborted = aborted;
      finish_problem(kp, S);
    } else if (!rerun && S.len == 0) {
      S.aborted = 0;
      finish_problem(kp, S);
    }
    sh->head = i;
    sh->flag = (S.done ? 0 : 1) | (rerun ? 2 : 0);
    sh->cap = rerun_cap;
  }
  __syncthreads();
  if (kp.trace >= 5 && tid == 0) {
    unsigned long long _t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));
    atomicAdd(kp.prof + 13, _t - _tprev);
    _tprev = _t;
  }
  const int flag = sh->flag;
  int nhead = sh->head;
  const int nlen = total - nhead;
  // ---- C. pool compaction when the bump allocator is nearly exhausted
  int ashift = 0;  // the list moves from [nhead, total) to [0, nlen)
  if ((flag & 1) && S.pool_top > kp.pcap - 2 * kp.reserve - 64 * 32) {
    ashift = nhead;
    Entry* np = pool_ptr(kp, p, S.pool_cur ^ 1);
    CandRec* ncr = topk ? cand_ptr(kp, p, S.pool_cur ^ 1) : nullptr;
    int* pcv_tmp = list_arr(kp, p, cur, 1);  // the input buffer is free now
    long long* vis_tmp = vis_in;
    for (int k = tid; k < nlen; k += blockDim.x) {
      np[k] = pool[ids_out[nhead + k]];
      if (topk) ncr[k] = crec[ids_out[nhead + k]];
      pcv_tmp[k] = pcv_out[nhead + k];
      vis_tmp[k] = vis_out[nhead + k];
      cut_in[k] = cut_out[nhead + k];
      m_in[k] = m_out[nhead + k];
      inf_in[k] = inf_out[nhead + k];
      chi_in[k] = chi_out[nhead + k];
      bo_in[k] = bo_out[nhead + k];
    }
    __syncthreads();
    for (int k = tid; k < nlen; k += blockDim.x) {
      ids_out[k] = k;
      pcv_out[k] = pcv_tmp[k];
      vis_out[k] = vis_tmp[k];
      cut_out[k] = cut_in[k];
      m_out[k] = m_in[k];
      inf_out[k] = inf_in[k];
      chi_out[k] = chi_in[k];
      bo_out[k] = bo_in[k];
      cnt_out[k] = 1;
    }
    __syncthreads();
    if (tid == 0) {
      S.pool_cur ^= 1;
      S.pool_top = nlen;
      S.head = 0;
    }
    nhead = 0;
    __syncthreads();
  }
  if (kp.trace >= 5 && tid == 0) {
    unsigned long long _t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));
    atomicAdd(kp.prof + 14, _t - _tprev);
    _tprev = _t;
  }
  // ---- D. queue the next wave
  if (!(flag & 2) && (flag & 1)) {
    // share of the run slots: from the active count SNAPSHOT taken before this
    // schedule phase (the live count drops as problems finish mid-phase; using it
    // let late schedulers over-push past qcap, starving problems)
    const int act = max(1, *((volatile int*)kp.active + 6));
    // ... throttled by the list's headroom: each queued run may split, adding
    // about as many pieces as this wave's runs did on average; a full list
    // would revert splits (wasted runs) every wave
    const long long runs_now = S.runs;
    const long long dr = runs_now - S.runs_prev;
    const int est = (int)min((long long)kp.reserve, max(1LL, (etot + dr - 1) / max(1LL, dr)));
    const int headroom = kp.lcap - kp.reserve - nlen;
    // an equal share of the run slots per active problem
    const int fair = kp.qmax / act;
    const int qmax = max(1, min(min(max(32, fair), kp.qmax_one), headroom / est));
    const long long bl = P.budget < 0 ? -1 : P.budget - S.V;
    if (kp.par_push && P.top_k <= 1 && nagg > 0) {
      // the tiles of the list are pushed by every CTA after the commits (S4)
      if (tid == 0) {
        S.pp_head = nhead;
        S.pp_len = nlen;
        S.pp_ashift = ashift;
        S.pp_qmax = qmax;
        S.pp_ntile = nagg;
        S.pp_bl = bl;
        S.pp_C = S.C;
        S.runs_prev = runs_now;
        publish_push(S, 1, wave);
      }
    } else {
      push_items(kp, next_queue, p, ids_out, pcv_out, vis_out, cut_out, m_out, chi_out,
                 pool_ptr(kp, p, S.pool_cur), nhead, nlen, S.C, qmax, bl, sh->l, sh->d, sh->i,
                 ag, nagg, ashift, sh, P.top_k, S.seed_obj,
                 P.top_k > 1 ? cand_ptr(kp, p, S.pool_cur) : nullptr, S);
      if (tid == 0) S.runs_prev = runs_now;
    }
  }
  if (tid == 0 && *((volatile int*)&S.pp_wave) != wave) publish_push(S, 0, wave);
  if (warp == 0) {
    if (flag & 2) {
      if (lane == 0) {
        Entry& e = pool_ptr(kp, p, S.pool_cur)[ids_out[nhead]];
        e.capped = 1;
        RunQueue* q = kp.queues + next_queue;
        const int slot = atomicAdd(&q->len, 1);
        if (slot >= kp.qcap) {
          atomicOr(kp.err, 4);  // never: qcap covers every problem's share
        } else {
        RunItem& it = kp.items[(size_t)next_queue * kp.qcap + slot];
        it.problem = p;
        it.pos = nhead;
        it.id = ids_out[nhead];
        it.front = 1;
        it.cap = sh->cap;
        it.cut = S.C;
        it.ntv = S.nT;
        for (int t = 0; t < KW; ++t) it.tv[t] = S.T[t];
        }
      }
    }
  }
  __syncthreads();
  if (kp.trace >= 5 && tid == 0) {
    unsigned long long _t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));
    atomicAdd(kp.prof + 15, _t - _tprev);
    _tprev = _t;
  }
  // expansion work items of the next wave: one per list tile
  if (tid == 0 && !S.done && !(flag & 2)) {
    const int nt = (S.len + TILE - 1) / TILE;
    const int base = atomicAdd(kp.wcount + wnext, nt);
    for (int t = 0; t < nt; ++t) kp.work[(size_t)wnext * kp.wcap + base + t] = make_int2(p, t);
  }
}

// ---------------------------------------------------------------- init

__device__ void first_occurrence(const int* key, int n, uint8_t* out) {
  int seen[MAXN];
  int ns = 0;
  for (int i = 0; i < n; ++i) {
    int ix = -1;
    for (int j = 0; j < ns; ++j)
      if (seen[j] == key[i]) {
        ix = j;
        break;
      }
    if (ix < 0) {
      seen[ns] = key[i];
      ix = ns++;
    }
    out[i] = (uint8_t)ix;
  }
}

// evaluate_partition (grouping.cpp:227-247): fresh sums in unit order
__device__ double evaluate_partition(const GProb& P, const uint8_t* rgs, double* z_out) {
  int m = 0;
  for (int i = 0; i < P.n; ++i) m = max(m, (int)rgs[i] + 1);
  double pw[MAXN], me[MAXN];
  int cnt[MAXN];
  for (int g = 0; g < m; ++g) {
    pw[g] = 0;
    me[g] = 0;
    cnt[g] = 0;
  }
  for (int i = 0; i < P.n; ++i) {
    pw[rgs[i]] += P.p[i];
    me[rgs[i]] += P.m[i];
    cnt[rgs[i]] += 1;
  }
  double z = 0;
  for (int gi = 0; gi < m; ++gi) {
    if (cnt[gi] == 0 || me[gi] < P.min_mem) return -1;
    const double rho = (double)(cnt[gi] - 1) / (double)(P.K + cnt[gi] - 1);
    const double gv = pw[gi] * (1.0 - rho);
    z = gi == 0 ? gv : (gv < z ? gv : z);
  }
  *z_out = z;
  return (double)m * z;
}

__device__ void init_problem(const KParams& kp, int p) {
  GProb& P = kp.probs[p];
  GState& S = kp.states[p];
  const int tid = threadIdx.x;
  const int n = P.n;
  for (int d = tid; d <= n + 1; d += blockDim.x) {
    if (d >= 1) P.f[d] = 1.0 - (double)(d - 1) / (double)(P.K + d - 1);
    else P.f[0] = 0.0;
  }
  for (int d = tid; d <= n; d += blockDim.x) {
    double rm = 0;
    for (int i = d; i < n; ++i) rm += P.m[i];
    P.RM[d] = rm;
  }
  __syncthreads();
  if (tid == 0) {
    double r = 0;
    P.R[n] = 0;
    for (int d = n - 1; d >= 0; --d) {
      r += P.p[d];
      P.R[d] = r;
    }
    // Error budget of the incremental sums (<= ~4 roundings per level on
    // quantities <= 2x the total power) plus the reference's own serial sum
    // (<= n roundings): (8n + 64) ulps of the largest magnitude, doubled.
    P.mb_abs = (double)(8 * n + 64) * kEps52 * 2.0 * (P.R[0] > 0 ? P.R[0] : 1.0);
    if (P.check_drift) P.mb_abs *= 4.0;  // inexact unit sums: a wider filter margin
    if (P.exact_mem) {
      P.md_abs = 0.0;
    } else {
      double mt = 0;
      for (int i = 0; i < n; ++i) mt += fabs(P.m[i]);
      P.md_abs = (double)(8 * n + 64) * kEps52 * 2.0 * ((double)n * fabs(P.min_mem) + mt);
    }
    // seeds: one group, singletons, by type, by node (grouping.cpp:206-225)
    uint8_t seeds[4][MAXN];
    for (int i = 0; i < n; ++i) {
      seeds[0][i] = 0;
      seeds[1][i] = (uint8_t)i;
    }
    first_occurrence(P.tkey, n, seeds[2]);
    first_occurrence(P.nkey, n, seeds[3]);
    double seed_obj = -1, seed_z = 0;
    int seed_ix = -1;
    for (int k = 0; k < 4; ++k) {
      double z = 0;
      const double obj = evaluate_partition(P, seeds[k], &z);
      if (obj > seed_obj) {  // strict: the first seed wins ties (:304)
        seed_obj = obj;
        seed_z = z;
        seed_ix = k;
      }
    }
    S.seed_obj = seed_obj;
    S.seed_z = seed_z;
    S.seed_ix = seed_ix;
    if (seed_ix >= 0)
      for (int i = 0; i < n; ++i) S.seed_rgs[i] = seeds[seed_ix][i];
    S.C = seed_obj;  // prune_floor (:312)
    S.nT = 0;
    S.nbest = 0;
    S.pp_wave = -1;
    S.pp_mode = 0;
    S.n_units = n;
    for (int t = 0; t < KW; ++t) S.T[t] = -1.0;
    S.V = 0;
    S.has_best = 0;
    S.best_obj = 0;
    S.best_G = 0;
    S.cur = 0;
    S.head = 0;
    S.done = 0;
    S.aborted = 0;
    S.rerun_pending = 0;
    S.waves = 0;
    S.runs = 0;
    S.runs_prev = 0;
    S.run_visits = 0;
    S.exact_checks = 0;
    S.max_list = 1;
    S.error = 0;
    // root node (not a visit): bound = sum of all powers, serially (:154-160)
    double bound = 0;
    for (int i = 0; i < n; ++i) bound += P.p[i];
    const bool pruned = (S.C >= 0 && bound < S.C) || (0.0 > P.RM[0]);
    S.cver = 0;
    S.pool_cur = 0;
    S.pool_top = 1;
    if (pruned) {
      S.len = 0;
      S.done = 1;
      atomicSub(kp.active, 1);
      atomicSub(kp.active + 62, n);
    } else {
      Entry& e = pool_ptr(kp, p, 0)[0];
      e.u[0] = 0;  // root has no groups: its only child is [0]
      e.du = 1;
      e.hi = 0;
      e.kind = KIND_FULL;
      e.cver = -1;
      e.finished = 0;
      e.capped = 0;
      e.uncapped = 0;
      e.has_best = 0;
      e.a_star = -1;
      list_vis(kp, p, 0)[0] = 0;
      list_dbl(kp, p, 0, 0)[0] = -1.0;
      list_dbl(kp, p, 0, 1)[0] = -1.0;
      list_dbl(kp, p, 0, 2)[0] = -1.0;
      list_arr(kp, p, 0, 4)[0] = 0;
      list_arr(kp, p, 0, 5)[0] = 0;
      list_arr(kp, p, 0, 0)[0] = 0;   // id
      list_arr(kp, p, 0, 1)[0] = -1;  // needs a run
      list_arr(kp, p, 0, 2)[0] = 1;
      S.len = 1;
      const int wi = atomicAdd(kp.wcount + 0, 1);
      kp.work[wi] = make_int2(p, 0);
      RunQueue* q = kp.queues + 0;
      const int slot = atomicAdd(&q->len, 1);
      kp.items[slot].problem = p;
      kp.items[slot].pos = 0;
      kp.items[slot].id = 0;
      kp.items[slot].front = 1;
      kp.items[slot].cap = kp.ramp > 0 ? min(kp.seg_cap, (long long)kp.ramp) : kp.seg_cap;
      kp.items[slot].cut = S.C;
      kp.items[slot].ntv = 0;
      for (int t = 0; t < KW; ++t) kp.items[slot].tv[t] = -1.0;
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------ the kernel

// Grid barrier (all blocks are co-resident: cooperative launch). One thread
// per block arrives and waits with __nanosleep; other warps wait on the block
// barrier. cooperative_groups' grid.sync() spins with an L1 invalidation per
// iteration (CCTL.IVALL in the loop, seen in the ncu source page), which wiped
// the L1 of the warps still searching; here the invalidation happens once, in
// the acquire fence after the release is observed.
__device__ __forceinline__ void gsync(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = bar + 1;
    const unsigned int gen = *vgen;
    __threadfence();  // release this block's writes
    const unsigned int arrived = atomicAdd(bar, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      unsigned int ns = 32;
      while (*vgen == gen) {
        __nanosleep(ns);
        ns = ns < 256 ? ns * 2 : 256;
      }
    }
    __threadfence();  // acquire: later reads see every block's writes
  }
  __syncthreads();
}

// 2 CTAs (16 warps) per SM: <= 128 registers per thread (HPK_REG_FREE=1 lifts the
// bound: ~200 registers, 1 CTA per SM — an experiment knob)
#ifdef HPK_REG_FREE
#define HPK_WAVE_BOUNDS __launch_bounds__(BLOCK_THREADS)
#else
#define HPK_WAVE_BOUNDS __launch_bounds__(BLOCK_THREADS, 2)
#endif
__global__ void HPK_WAVE_BOUNDS hpk_wave_kernel(KParams kp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem* wsm = reinterpret_cast<WarpSmem*>(smem_raw);
  void* smem_tmp = smem_raw + sizeof(WarpSmem) * WARPS_PER_BLOCK;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wsm[warp].staged = -1;

  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (kp.deadline_ns != ~0ull) kp.deadline_ns += now;  // relative budget -> absolute
    *kp.deadline_slot = kp.deadline_ns;
  }
  if (kp.trace >= 4 && blockIdx.x == 0 && threadIdx.x == 0) kp.prof[11] = 4;  // per-decision trace
  if (HPK_TRACE_LEVEL == 1 && blockIdx.x == 0 && threadIdx.x == 0) {
    kp.prof[24] = ~0ull;
    kp.prof[25] = ~0ull;
    kp.prof[32] = 0;
    for (int k = 0; k < 4; ++k) kp.prof[28 + k] = 0;
  }
  for (int p = blockIdx.x; p < kp.n_problems; p += gridDim.x) init_problem(kp, p);
  gsync(kp.bar);
  kp.deadline_ns = *((volatile unsigned long long*)kp.deadline_slot);

  int cur = 0;
  for (int wave = 0; wave < kp.max_waves; ++wave) {
    // ---- run phase
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      kp.queues[cur ^ 1].len = 0;
      kp.queues[cur ^ 1].head = 0;
      kp.active[6] = *((volatile int*)kp.active);  // active-count snapshot for the schedule
      kp.active[63] = *((volatile int*)kp.active + 62);  // ... and of their units
    }
    RunQueue* q = kp.queues + cur;
    RunItem* items = kp.items + (size_t)cur * kp.qcap;
    const int qlen = min(*((volatile int*)&q->len), kp.qcap);
    unsigned long long wave_t0 = 0;  // this warp's view of the run phase start
    if (kp.wave_ns) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(wave_t0));
      wave_t0 = __shfl_sync(HPK_FULL_MASK, wave_t0, 0);
    }
    unsigned long long t_w0 = 0, t_dr = 0, t_x[4] = {0, 0, 0, 0}, t_x0 = 0;
    if (kp.trace && blockIdx.x == 0 && threadIdx.x == 0)
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_w0));
    while (warp < kp.runners) {
      int it = 0;
      if (lane == 0) it = atomicAdd(&q->head, 1);
      it = shfl(it, 0);
      if (it >= qlen) {  // queue drained: tell the runs still going to wrap up
        if (lane == 0) *((volatile int*)kp.stop) = 1;
        if (HPK_TRACE_LEVEL == 1 && lane == 0) {  // trace: when the queue drained
          unsigned long long now;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          atomicMin(kp.prof + 24, now);
        }
        break;
      }
      const RunItem item = items[it];
      unsigned long long t_start = 0;
      if (HPK_TRACE_LEVEL == 1) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
        if (lane == 0) atomicMin(kp.prof + 25, wave_t0);
      }
      const int p = item.problem;
      const GProb& P = kp.probs[p];
      GState& S = kp.states[p];
      Entry* E = pool_ptr(kp, p, S.pool_cur) + item.id;
      const double C = item.cut;
      const int cver = 1;
      const PView PV = stage_problem(P, wsm + warp, lane, p);
      // (a PREFIX re-run must end at its end marker: it is never split)
      const bool stoppable = !E->capped && !E->uncapped && E->kind != KIND_PREFIX;
      if (lane == 0)
        wsm[warp].wave_end = stoppable && kp.wave_ns ? wave_t0 + kp.wave_ns : 0ull;
      __syncwarp();
      const int tk = P.top_k;
      RunOut o;
      if (tk > 1) {
        // the entering cutoff state travels with the item; the record keeps it
        // for the commit walk's exactness check
        CandRec* rec = cand_ptr(kp, p, S.pool_cur) + item.id;
        WarpSmem* ws = wsm + warp;
        if (lane < KW) {
          ws->T[lane] = item.tv[lane];
          rec->tin[lane] = lane < item.ntv ? item.tv[lane] : -1.0;
        }
        if (lane == 0) {
          ws->nT = item.ntv;
          rec->ntin = item.ntv;
        }
        __syncwarp();
#define HPK_RUN4(TK, DR, PF, NS, CI_, WS, TKV, FL, REC)                                      \
  run_segment<TK, DR, PF, NS, CI_>(PV, E, E, C, item.cap, WS, lane, kp.err, kp.deadline_slot,   \
                              (kp.trace >= 2 && kp.trace < 5) ? kp.prof : nullptr,          \
                              stoppable ? kp.stop : nullptr, TKV, FL, REC)
// one lane slot while every node holds <= 32 groups (always for <= 32 units;
// a run that meets more is redone with two slots)
#define HPK_RUN3(TK, DR, PF, CI_, WS, TKV, FL, REC)                                        \
  [&]() {                                                                                  \
    if (MAXN <= 64) {                                                                      \
      RunOut r1 = HPK_RUN4(TK, DR, PF, 1, CI_, WS, TKV, FL, REC);                          \
      if (!r1.retry) return r1;                                                            \
      if (TK) { /* the entering top-k state again: the first try moved it */               \
        if (lane < KW) (WS)->T[lane] = item.tv[lane];                                      \
        if (lane == 0) (WS)->nT = item.ntv;                                                \
        __syncwarp();                                                                      \
      }                                                                                    \
    }                                                                                      \
    return HPK_RUN4(TK, DR, PF, 2, CI_, WS, TKV, FL, REC);                                 \
  }()
#define HPK_RUN(TK, DR, CI_, WS, TKV, FL, REC)                                             \
  (E->kind == KIND_PREFIX ? HPK_RUN3(TK, DR, true, CI_, WS, TKV, FL, REC)                  \
                          : HPK_RUN3(TK, DR, false, CI_, WS, TKV, FL, REC))
        // the drift-checking instantiation only for problems outside the
        // exact-sum contract: the common case carries no extra instructions
#if HPK_CUT_IV_MAX > 0
        o = PV.check_drift ? HPK_RUN(true, true, false, ws, tk, S.seed_obj, rec)
            : kp.cut_iv    ? HPK_RUN(true, false, true, ws, tk, S.seed_obj, rec)
                           : HPK_RUN(true, false, false, ws, tk, S.seed_obj, rec);
#else
        o = PV.check_drift ? HPK_RUN(true, true, false, ws, tk, S.seed_obj, rec)
                           : HPK_RUN(true, false, false, ws, tk, S.seed_obj, rec);
#endif
      } else {
        // k = 1 runs of a latency-bound launch (few problems) record their
        // cutoff interval; drift-checked problems keep the exact-cutoff rule
#if HPK_CUT_IV_MAX > 0
        o = PV.check_drift ? HPK_RUN(false, true, false, wsm + warp, 1, 0.0, nullptr)
            : kp.cut_iv    ? HPK_RUN(false, false, true, wsm + warp, 1, 0.0, nullptr)
                           : HPK_RUN(false, false, false, wsm + warp, 1, 0.0, nullptr);
#else
        o = PV.check_drift ? HPK_RUN(false, true, false, wsm + warp, 1, 0.0, nullptr)
                           : HPK_RUN(false, false, false, wsm + warp, 1, 0.0, nullptr);
#endif
#undef HPK_RUN
#undef HPK_RUN3
#undef HPK_RUN4
      }
      int* pcv = list_arr(kp, p, S.cur, 1);
      int* cnt = list_arr(kp, p, S.cur, 2);
      int* pfirst = list_arr(kp, p, S.cur, 3);
      int pieces = 0, first = 0;
      bool keep = true;
      if (!o.finished && E->uncapped) {
        // the head ran past the remaining budget: keep it as a finished run
        // with budget_left + 1 visits; the commit walk re-runs it capped
        o.finished = true;
      } else if (!o.finished && !E->capped) {
        pieces = split_run(kp, p, S, E, o, wsm + warp, lane, item.front != 0, &first);
        keep = pieces > 0;  // pool full: drop the run, it re-runs later
      }
      if (lane == 0) {
        E->visits = o.visits;
        E->finished = 1;
        E->has_best = o.has_best ? 1 : 0;
        E->best_obj = o.best_obj;
        E->best_G = o.best_G;
        E->m = o.m;
        E->a_star = o.a_star;
        if (E->capped) {
          E->cver = cver;  // budget re-run: consumed directly by the scheduler
        } else if (keep) {
          E->cver = cver;
          E->uncapped = 0;
          pcv[item.pos] = 1;
          cnt[item.pos] = 1 + pieces;
          pfirst[item.pos] = first;
          list_vis(kp, p, S.cur)[item.pos] = o.visits;
          list_dbl(kp, p, S.cur, 0)[item.pos] = C;
          list_dbl(kp, p, S.cur, 1)[item.pos] = o.m;
          list_dbl(kp, p, S.cur, 2)[item.pos] = o.best_obj;
          list_arr(kp, p, S.cur, 5)[item.pos] = __float_as_int(__double2float_rd(o.hi));
          list_arr(kp, p, S.cur, 4)[item.pos] =
              o.best_G | (o.has_best ? 256 : 0) |
              ((E->kind == KIND_PREFIX && o.a_star >= 0) ? 512 : 0);
          if (pieces > 0)
            atomicAdd(kp.xt + (size_t)p * kp.xtn + (item.pos - S.head) / TILE, pieces);
        } else {
          E->cver = -1;
          E->finished = 0;
          pcv[item.pos] = -1;
          cnt[item.pos] = 1;
        }
        if (HPK_TRACE_LEVEL == 1) {  // trace: end of the wave's stoppable / other runs
          unsigned long long now;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          atomicMax(kp.prof + (stoppable ? 29 : 28), now);
          if (now > wave_t0 + kp.wave_ns + 60000ull && atomicAdd(kp.prof + 32, 1ull) < 6)
            printf("[hpk-late] wave %d item %d/%d: start %.1f us end %.1f us (own slice start), "
                   "visits %lld cap %lld finished %d pieces %d stoppable %d kind %d retry-free\n",
                   wave, it, qlen, (t_start - wave_t0) * 1e-3, (now - wave_t0) * 1e-3,
                   o.visits, item.cap, (int)o.finished, pieces, (int)stoppable, (int)E->kind);
          if (!stoppable) {
            atomicMax(kp.prof + 30, (unsigned long long)o.visits);
            atomicAdd(kp.prof + 31, 1ull);
          }
        }
        atomicAdd((unsigned long long*)&S.runs, 1ull);
        atomicAdd((unsigned long long*)&S.run_visits, (unsigned long long)o.visits);
        if (o.exact) atomicAdd((unsigned long long*)&S.exact_checks, (unsigned long long)o.exact);
        if (o.overflow) atomicOr(&S.error, 8);  // > 63 groups: the serial replica redoes it
        if (o.drift) atomicOr(&S.error, 16);    // path-dependent sums: the serial replica
      }
      __syncwarp();
    }
    gsync(kp.bar);
    unsigned long long t_w1 = 0;
    if (kp.trace && blockIdx.x == 0 && threadIdx.x == 0)
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_w1));
    // ---- schedule phase. S2: list expansion, every CTA takes tiles
    {
      const int wb = wave & 1;
      if (blockIdx.x == 0 && threadIdx.x == 0) kp.wcount[wb ^ 1] = 0;
      const int nwk = *((volatile int*)(kp.wcount + wb));
      SchedSmem* sh = reinterpret_cast<SchedSmem*>(smem_tmp);
      for (int w = blockIdx.x; w < nwk; w += gridDim.x) {
        const int2 wk = kp.work[(size_t)wb * kp.wcap + w];
        expand_tile(kp, wk.x, wk.y, sh);
        __syncthreads();
      }
    }
    gsync(kp.bar);
    if (kp.trace >= 5 && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t_x;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_x));
      atomicAdd(kp.prof + 18, t_x - t_w1);
    }
    // S3: commit, compaction, queue the next wave (one CTA per problem)
    for (int p = blockIdx.x; p < kp.n_problems; p += gridDim.x)
      schedule_problem(kp, p, cur ^ 1, smem_tmp, (wave & 1) ^ 1, wave);
    // S4: the queue step, one item per list tile (the S2 items), every CTA;
    // each item waits for its problem's commit (done before by its own CTA)
    if (kp.par_push) {
      const int wb = wave & 1;
      const int nwk = *((volatile int*)(kp.wcount + wb));
      SchedSmem* sh = reinterpret_cast<SchedSmem*>(smem_tmp);
      for (int w = blockIdx.x; w < nwk; w += gridDim.x) {
        const int2 wk = kp.work[(size_t)wb * kp.wcap + w];
        push_tile(kp, wk.x, wk.y, cur ^ 1, wave, sh);
        __syncthreads();
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *((volatile int*)kp.stop) = 0;  // re-armed for the next run phase
      if (HPK_TRACE_LEVEL == 1) {
        t_dr = *((volatile unsigned long long*)kp.prof + 24);
        for (int k = 0; k < 4; ++k) t_x[k] = *((volatile unsigned long long*)kp.prof + 28 + k);
        kp.prof[24] = ~0ull;
        for (int k = 0; k < 4; ++k) kp.prof[28 + k] = 0;
        t_x0 = *((volatile unsigned long long*)kp.prof + 25);
        kp.prof[25] = ~0ull;
        kp.prof[32] = 0;
      }
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now > kp.deadline_ns) {  // wall-clock watchdog: stop every block
        atomicOr(kp.err, 2);
        atomicExch(kp.active, -1000000);
      }
    }
    gsync(kp.bar);
    if (kp.trace >= 5 && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t_w2;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_w2));
      atomicAdd(kp.prof + 16, t_w1 - t_w0);
      atomicAdd(kp.prof + 17, t_w2 - t_w1);
    }
    if (kp.trace && kp.trace < 5 && kp.trace_p < 0 && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t_w2;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_w2));
      const unsigned long long t_b = t_x0 < t_w0 ? t_x0 : t_w0;  // first warp's start
      auto rel = [&](unsigned long long t) {
        return t >= t_b && t != ~0ull ? (double)(t - t_b) * 1e-3 : -1.0;
      };
      printf("[hpk] wave %d: %d runs, run %.1f us (queue drained at %.1f us, last sliced run "
             "%.1f us, last other run %.1f us: %llu of them, max %llu visits), schedule %.1f us "
             "(active %d)\n", wave, qlen, (t_w1 - t_b) * 1e-3, rel(t_dr), rel(t_x[1]),
             rel(t_x[0]), t_x[3], t_x[2], (t_w2 - t_w1) * 1e-3, *((volatile int*)kp.active));
    }
    if (*((volatile int*)kp.active) <= 0) break;
    cur ^= 1;
  }
  if (kp.trace >= 5 && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long* q = kp.prof;
    printf("[hpk-sched] totals over all waves/problems (us): expand+scatter %.1f commit %.1f "
           "compaction %.1f push %.1f | run phases %.1f schedule phases %.1f (S2 expansion %.1f)\n",
           q[12] * 1e-3, q[13] * 1e-3, q[14] * 1e-3, q[15] * 1e-3, q[16] * 1e-3, q[17] * 1e-3,
           q[18] * 1e-3);
    printf("[hpk-sched] push: %llu tiles skipped, %llu chunks scanned (%llu positions) | commit: "
           "%llu tiles skipped, %llu chunks\n", q[19], q[20], q[21], q[22], q[23]);
  }
  if (kp.trace >= 2 && kp.trace < 5 && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long* q = kp.prof;
    const unsigned long long vis = q[2] + q[4] + q[8];
    printf("[hpk-prof] run cycles %llu, iterations %llu (%.1f cyc/iter), visits %llu (%.1f "
           "cyc/visit) | leaf batches %llu (leaves %llu) | single checks %llu | prune skips %llu "
           "(children %llu) | descends %llu pops %llu masks %llu exact %llu\n",
           q[0], q[3], q[3] ? (double)q[0] / q[3] : 0.0, vis, vis ? (double)q[0] / vis : 0.0,
           q[1], q[2], q[4], q[7], q[8], q[5], q[6], q[10], q[9]);
  }
}

// ------------------------------------------------------- serial replica

struct SerialCand {
  double obj, z;
  int G;
  uint8_t rgs[256];
};

// One thread replays dfs() of grouping.cpp:135-202 for one problem, with the
// reference's exact state updates (+= / -=) and top_k bookkeeping.
struct SerialProb {
  int n, K, top_k;
  long long budget;
  double min_mem;
  const double* p;
  const double* m;
  const int* tkey;
  const int* nkey;
  // outputs
  int status, count, optimal;
  long long visited;
  double* obj_out;   // device [top_k]
  double* z_out;     // device [top_k]
  SerialCand* cand;  // device [top_k + 1]: the best-first candidate list
  int* rgs_out;  // device [top_k * n]
};

__device__ void seed_rgs(const SerialProb& pb, int k, int* rgs) {
  int distinct = 0;
  for (int i = 0; i < pb.n; ++i) {
    if (k == 0) {
      rgs[i] = 0;
    } else if (k == 1) {
      rgs[i] = i;
    } else {
      const int* key = k == 2 ? pb.tkey : pb.nkey;
      int j = 0;
      while (key[j] != key[i]) ++j;
      rgs[i] = j == i ? distinct++ : rgs[j];
    }
  }
}

__device__ bool s_better(double ao, int ag, double bo, int bg) {
  if (ao != bo) return ao > bo;
  return ag < bg;
}

__global__ void hpk_serial_kernel(SerialProb* probs, int n_probs, SerialCand* cands,
                                  double* scratch, int* iscratch, int max_n) {
  const int pi = blockIdx.x * blockDim.x + threadIdx.x;
  if (pi >= n_probs) return;
  SerialProb& pb = probs[pi];
  const int n = pb.n;
  double* gp = scratch + (size_t)pi * 2 * (max_n + 1);
  double* gm = gp + (max_n + 1);
  int* gc = iscratch + (size_t)pi * 4 * (max_n + 1);
  int* rgs = gc + (max_n + 1);
  int* fr_G = rgs + (max_n + 1);
  int* fr_gi = fr_G + (max_n + 1);
  SerialCand* best = pb.cand;
  (void)cands;
  int n_best = 0;
  const int top_k = pb.top_k < 1 ? 1 : pb.top_k;

  // seeds (:206-225, :299-312)
  double seed_obj = -1, seed_z = 0;
  int seed_ix = -1;
  {
    for (int k = 0; k < 4; ++k) {
      // build seed k into rgs (first-occurrence numbering, :213-221)
      seed_rgs(pb, k, rgs);
      int mg = 0;
      for (int i = 0; i < n; ++i) mg = max(mg, rgs[i] + 1);
      for (int g = 0; g < mg; ++g) { gp[g] = 0; gm[g] = 0; gc[g] = 0; }
      for (int i = 0; i < n; ++i) { gp[rgs[i]] += pb.p[i]; gm[rgs[i]] += pb.m[i]; gc[rgs[i]] += 1; }
      double z = 0, obj = 0;
      bool ok = true;
      for (int gi = 0; gi < mg; ++gi) {
        if (gc[gi] == 0 || gm[gi] < pb.min_mem) { ok = false; break; }
        const double rho = (double)(gc[gi] - 1) / (double)(pb.K + gc[gi] - 1);
        const double gv = gp[gi] * (1.0 - rho);
        z = gi == 0 ? gv : (gv < z ? gv : z);
      }
      obj = ok ? (double)mg * z : -1;
      if (obj > seed_obj) {
        seed_obj = obj;
        seed_z = z;
        seed_ix = k;
      }
    }
  }
  const double prune_floor = seed_obj;
  long long visited = 0;
  bool aborted = false;
  int G = 0;
  // iterative dfs: node at depth `next`
  int next = 0;
  int phase = 0;  // 0: process node at `next`; 1: iterate children of frame next; 2: return to parent
  while (true) {
    if (phase == 0) {
      if (next == n) {  // leaf
        double z = 0;
        bool first = true, feas = true;
        for (int gi = 0; gi < G; ++gi) {
          if (gm[gi] < pb.min_mem) { feas = false; break; }
          const double rho = (double)(gc[gi] - 1) / (double)(pb.K + gc[gi] - 1);
          const double gv = gp[gi] * (1.0 - rho);
          z = first ? gv : (gv < z ? gv : z);
          first = false;
        }
        if (feas) {
          const double objective = (double)G * z;
          int pos = n_best;
          for (int i = 0; i < n_best; ++i)
            if (s_better(objective, G, best[i].obj, best[i].G)) { pos = i; break; }
          bool dup = false;
          for (int i = 0; i < n_best && !dup; ++i) {
            bool same = true;
            for (int t = 0; t < n; ++t)
              if (best[i].rgs[t] != rgs[t]) { same = false; break; }
            dup = same;
          }
          if (!dup) {
            for (int i = n_best; i > pos; --i) best[i] = best[i - 1];
            best[pos].obj = objective;
            best[pos].z = z;
            best[pos].G = G;
            for (int t = 0; t < n; ++t) best[pos].rgs[t] = (uint8_t)rgs[t];
            n_best = n_best + 1 > top_k ? top_k : n_best + 1;
          }
        }
        phase = 2;
        continue;
      }
      double bound = 0;
      for (int gi = 0; gi < G; ++gi) {
        const double rho = (double)(gc[gi] - 1) / (double)(pb.K + gc[gi] - 1);
        bound += gp[gi] * (1.0 - rho);
      }
      double remaining_mem = 0;
      for (int i = next; i < n; ++i) {
        bound += pb.p[i];
        remaining_mem += pb.m[i];
      }
      double cutoff = prune_floor;
      if (n_best >= top_k) cutoff = prune_floor > best[n_best - 1].obj ? prune_floor : best[n_best - 1].obj;
      if (cutoff >= 0 && bound < cutoff) { phase = 2; continue; }
      double deficit = 0;
      for (int gi = 0; gi < G; ++gi) {
        const double d = pb.min_mem - gm[gi];
        deficit += d > 0.0 ? d : 0.0;
      }
      if (deficit > remaining_mem) { phase = 2; continue; }
      fr_G[next] = G;
      fr_gi[next] = 0;
      phase = 1;
      continue;
    }
    if (phase == 1) {
      const int gi = fr_gi[next];
      const int ng = fr_G[next];
      if (gi > ng) { phase = 2; continue; }
      if (pb.budget >= 0 && visited >= pb.budget) { aborted = true; break; }
      ++visited;
      if (gi == ng) { gp[G] = pb.p[next]; gm[G] = pb.m[next]; gc[G] = 1; ++G; }
      else { gp[gi] += pb.p[next]; gm[gi] += pb.m[next]; gc[gi] += 1; }
      rgs[next] = gi;
      ++next;
      phase = 0;
      continue;
    }
    // phase 2: return from node at `next` to its parent frame
    if (next == 0) break;  // root finished
    --next;
    {
      const int gi = fr_gi[next];
      const int ng = fr_G[next];
      if (gi == ng) { --G; }
      else { gp[gi] -= pb.p[next]; gm[gi] -= pb.m[next]; gc[gi] -= 1; }
      fr_gi[next] = gi + 1;
    }
    phase = 1;
  }
  // result rules (:316-334)
  const bool optimal = !aborted;
  pb.visited = visited;
  pb.status = 0;
  if (n_best == 0) {
    if (seed_obj < 0) { pb.status = 3; return; }
  }
  if (n_best == 0 || (!optimal && seed_obj > best[0].obj)) {
    // rebuild the winning seed
    seed_rgs(pb, seed_ix, rgs);
    for (int i = 0; i < n; ++i) pb.rgs_out[i] = rgs[i];
    pb.count = 1;
    pb.obj_out[0] = seed_obj;
    pb.z_out[0] = seed_z;
    pb.optimal = 0;
    return;
  }
  pb.count = n_best;
  for (int k = 0; k < n_best; ++k) {
    pb.obj_out[k] = best[k].obj;
    pb.z_out[k] = best[k].z;
    for (int i = 0; i < n; ++i) pb.rgs_out[(size_t)k * n + i] = best[k].rgs[i];
  }
  pb.optimal = optimal ? 1 : 0;
}

// ------------------------------------------------------ enumeration engine
// Exhaustive searches (n <= exact_threshold) with top_k = 1 on the planner
// path: the reference's winner is the global maximum of the key (objective
// desc, #groups asc, enumeration order asc) over every feasible leaf — the
// prune floor is a seed's objective and that seed is itself a leaf, so bound
// pruning never removes a leaf that could win.
// Every restricted-growth string is unranked in lexicographic (= DFS preorder)
// order and evaluated with fresh sums, which equal the DFS's incremental
// sums under the value contract. Visits are not counted (the plan does not
// report them), so the search config opts in (hpk_search_config::enumerate).
constexpr int ENUM_MAXN = 12;  // Bell(12) = 4,213,597 leaves

struct EnumProb {
  int n, K, top_k, out0;  // out0: this problem's first output slot
  double floor_;  // the best seed's objective (the DFS's prune floor)
  double min_mem;
  double p[ENUM_MAXN], m[ENUM_MAXN];
  long long total;  // Bell(n)
  int block0, nblocks;
};
struct EnumBest {
  double obj;
  int G;
  long long rank;
};

// D[r][g]: completions of an RGS prefix with r positions left and g groups used
struct EnumTable {
  long long D[ENUM_MAXN + 1][ENUM_MAXN + 2];
};

__device__ __forceinline__ bool enum_better(double ao, int ag, long long ar, double bo, int bg,
                                            long long br) {
  if (ao != bo) return ao > bo;
  if (ag != bg) return ag < bg;
  return ar < br;
}

// top_k = k > 1: the DFS's list is the global top k by key whenever at least k
// feasible leaves reach the floor (every such leaf's ancestors then pass the
// cutoff, which never exceeds the global k-th objective); each block reports
// its k best and its count of leaves at or above the floor, and the host falls
// back to the wave engine when the count is short.
__global__ void __launch_bounds__(256) hpk_enum_kernel(const EnumProb* probs, int n_probs,
                                                       const EnumTable* tab, EnumBest* out,
                                                       int* nabove, int per_block) {
  // block -> (problem, chunk of ranks)
  int pi = 0;
  while (pi + 1 < n_probs && probs[pi + 1].block0 <= (int)blockIdx.x) ++pi;
  const EnumProb& P = probs[pi];
  const int n = P.n;
  const long long lo = (long long)(blockIdx.x - P.block0) * per_block;
  const long long hi = min(P.total, lo + per_block);
  const int tk = P.top_k;
  // this thread's k best, best first
  double lo_[KW];
  int lg_[KW];
  long long lr_[KW];
  int ln = 0, above = 0;
  for (long long rk = lo + threadIdx.x; rk < hi; rk += blockDim.x) {
    // unrank (lexicographic RGS): digit 0 is 0; each later digit is an
    // existing group (D[r][g] completions each) or the new group g
    int a[ENUM_MAXN];
    a[0] = 0;
    int g = 1;
    unsigned k = (unsigned)rk;  // Bell(12) < 2^32: 32-bit unranking
#pragma unroll
    for (int i = 1; i < ENUM_MAXN; ++i) {
      if (i < n) {
        const int r = n - 1 - i;
        const unsigned w = (unsigned)tab->D[r][g];
        const unsigned q = k / w;
        if (q < (unsigned)g) {
          a[i] = (int)q;
          k -= q * w;
        } else {
          a[i] = g;
          k -= (unsigned)g * w;
          ++g;
        }
      }
    }
    // leaf (grouping.cpp:138-149): every group's memory >= MIN_mem, z = the
    // running min of the groups' Eq. (2) effective powers in group order
    bool ok = true;
    double z = 0;
    for (int gi = 0; gi < g; ++gi) {
      double pw = 0, me = 0;
      int cnt = 0;
#pragma unroll
      for (int i = 0; i < ENUM_MAXN; ++i) {
        if (i < n && a[i] == gi) {
          pw += P.p[i];
          me += P.m[i];
          ++cnt;
        }
      }
      if (me < P.min_mem) {
        ok = false;
        break;
      }
      const double rho = (double)(cnt - 1) / (double)(P.K + cnt - 1);
      const double e = pw * (1.0 - rho);
      z = gi == 0 ? e : (e < z ? e : z);
    }
    if (!ok) continue;
    const double obj = (double)g * z;
    above += obj >= P.floor_ ? 1 : 0;
    if (ln < tk || enum_better(obj, g, rk, lo_[ln - 1], lg_[ln - 1], lr_[ln - 1])) {
      int pos = ln < tk ? ln : tk - 1;
      while (pos > 0 && enum_better(obj, g, rk, lo_[pos - 1], lg_[pos - 1], lr_[pos - 1])) {
        lo_[pos] = lo_[pos - 1];
        lg_[pos] = lg_[pos - 1];
        lr_[pos] = lr_[pos - 1];
        --pos;
      }
      lo_[pos] = obj;
      lg_[pos] = g;
      lr_[pos] = rk;
      ln = ln < tk ? ln + 1 : tk;
    }
  }
  // the block's k best: k rounds of a block argmax over the threads' heads
  __shared__ double so[8];
  __shared__ int sg[8];
  __shared__ long long sr[8];
  __shared__ int sa[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int head = 0;
  for (int round = 0; round < tk; ++round) {
    double bo = head < ln ? lo_[head] : -1.0;
    int bg = head < ln ? lg_[head] : 0;
    long long br = head < ln ? lr_[head] : 0x7fffffffffffffffLL;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double oo = __shfl_xor_sync(HPK_FULL_MASK, bo, o);
      const int og = __shfl_xor_sync(HPK_FULL_MASK, bg, o);
      const long long orr = __shfl_xor_sync(HPK_FULL_MASK, br, o);
      if (oo >= 0 && (bo < 0 || enum_better(oo, og, orr, bo, bg, br))) {
        bo = oo;
        bg = og;
        br = orr;
      }
    }
    if (lane == 0) {
      so[warp] = bo;
      sg[warp] = bg;
      sr[warp] = br;
    }
    __syncthreads();
    bo = so[0];
    bg = sg[0];
    br = sr[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (so[w] >= 0 && (bo < 0 || enum_better(so[w], sg[w], sr[w], bo, bg, br))) {
        bo = so[w];
        bg = sg[w];
        br = sr[w];
      }
    // every thread now holds the block winner (ranks are unique): its owner pops it
    if (head < ln && lr_[head] == br && bo >= 0) ++head;
    if (threadIdx.x == 0) {
      EnumBest& e = out[(size_t)P.out0 + (size_t)(blockIdx.x - P.block0) * tk + round];
      e.obj = bo;
      e.G = bg;
      e.rank = br;
    }
    __syncthreads();
  }
  // leaves at or above the floor
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) above += __shfl_xor_sync(HPK_FULL_MASK, above, o);
  if (lane == 0) sa[warp] = above;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sa[w];
    nabove[blockIdx.x] = t;
  }
}

}  // namespace hpk

// ================================================================== host

namespace {

using namespace hpk;

struct DeviceCtx {
  int device = -1;
  int sms = 0;
  int blocks_per_sm = 0;
  size_t cap_probs = 0, cap_pools = 0, cap_lists = 0, cap_items = 0, cap_states = 0,
         cap_scratch = 0;
  GProb* probs = nullptr;
  GState* states = nullptr;
  Entry* pools = nullptr;
  CandRec* cands = nullptr;
  size_t cap_cands = 0;
  int* lists = nullptr;
  long long* lvis = nullptr;
  size_t cap_lvis = 0;
  double* ldbl = nullptr;
  size_t cap_ldbl = 0;
  int* scratch = nullptr;
  int* xt = nullptr;
  size_t cap_xt = 0;
  int2* work = nullptr;
  size_t cap_work = 0;
  TileAgg* agg = nullptr;
  size_t cap_agg = 0;
  PushAgg* pagg = nullptr;
  size_t cap_pagg = 0;
  RunQueue* queues = nullptr;
  RunItem* items = nullptr;
  int* active = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  HpkArena arena;  // enumeration engine's inputs / outputs
  std::mutex mu;
};

DeviceCtx g_ctx[16 * HPK_SPLIT_MAX];  // [device + 16 * slot]: slots 1.. = concurrent partitions (split_device)

thread_local std::string t_err;
thread_local hpk_timing t_timing;

int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

#define HPK_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(5, std::string("hetplan_b200 CUDA error: ") + cudaGetErrorString(_e) + \
                         " at " #call);                                                   \
  } while (0)

int ensure_ctx(DeviceCtx& c, int device) {
  if (c.device == device) return 0;
  HPK_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  HPK_CUDA(cudaGetDeviceProperties(&prop, device));
  c.sms = prop.multiProcessorCount;
  const size_t smem = sizeof(WarpSmem) * WARPS_PER_BLOCK + sizeof(SchedSmem);
  HPK_CUDA(cudaFuncSetAttribute(hpk_wave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  int bps = 0;
  HPK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, hpk_wave_kernel, BLOCK_THREADS,
                                                         smem));
  if (bps < 1) return fail(5, "hetplan_b200: wave kernel cannot be resident");
  c.blocks_per_sm = bps;
  HPK_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  HPK_CUDA(cudaEventCreate(&c.ev0));
  HPK_CUDA(cudaEventCreate(&c.ev1));
  HPK_CUDA(cudaMalloc(&c.active, sizeof(int) * 128));  // [64, 128): trace slots
  HPK_CUDA(cudaMalloc(&c.queues, sizeof(RunQueue) * 2));
  c.device = device;
  return 0;
}

template <typename T>
int grow(T*& ptr, size_t& cap, size_t need) {
  if (need <= cap) return 0;
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  size_t want = std::max(need, cap * 2);
  HPK_CUDA(cudaMalloc(&ptr, sizeof(T) * want));
  cap = want;
  return 0;
}

// Values exactly summable in fp64: all multiples of a common power of two with
// the total (in those units) below 2^53 -> every partial sum, in any order,
// is exact, so the reference's path-dependent += / -= sums equal ours.
bool exact_sums(const double* v, int n, double extra, bool include_extra) {
  int emin = 100000;
  double total = 0;
  auto lowexp = [](double x, int* e) -> bool {
    if (!(x >= 0) || std::isinf(x)) return false;
    if (x == 0) {
      *e = 100000;
      return true;
    }
    int ex;
    double mant = std::frexp(x, &ex);  // x = mant * 2^ex, mant in [0.5,1)
    // lowest set bit of the 53-bit significand
    long long sig = (long long)std::ldexp(mant, 53);
    int tz = 0;
    while ((sig & 1) == 0) {
      sig >>= 1;
      ++tz;
    }
    *e = ex - 53 + tz;
    return true;
  };
  for (int i = 0; i < n; ++i) {
    int e;
    if (!lowexp(v[i], &e)) return false;
    emin = std::min(emin, e);
    total += std::fabs(v[i]);
  }
  if (include_extra) {
    int e;
    if (!lowexp(extra, &e)) return false;
    emin = std::min(emin, e);
    total += std::fabs(extra);
  }
  if (emin == 100000) return true;
  // total in units of 2^emin must stay below 2^53
  return std::ldexp(total, -emin) < 9007199254740992.0 * 0.5;
}

// z of a DFS leaf as the reference computes it (grouping.cpp:140-147): the
// running min of the groups' effective powers, in group order.
double leaf_z(const hpk_grouping_problem& pr, const uint8_t* rgs, int G) {
  double pw[MAXN] = {0}, me[MAXN] = {0};
  int cn[MAXN] = {0};
  for (int u = 0; u < pr.n; ++u) {
    pw[rgs[u]] += pr.power[u];
    me[rgs[u]] += pr.memory[u];
    cn[rgs[u]] += 1;
  }
  double z = 0;
  for (int gi = 0; gi < G; ++gi) {
    const double rho = (double)(cn[gi] - 1) / (double)(pr.n_microbatches + cn[gi] - 1);
    const double gv = pw[gi] * (1.0 - rho);
    z = gi == 0 ? gv : (gv < z ? gv : z);
  }
  return z;
}

// The prune floor of solve_grouping_topk (grouping.cpp:299-312): the best of
// the four seed partitions (one group, singletons, by type, by node; first
// occurrence numbering), evaluated with fresh sums in unit order (:227-247),
// strict '>' so the first seed wins ties; -1 if none is feasible.
double seed_floor(const hpk_grouping_problem& pr) {
  const int n = pr.n;
  double best = -1;
  for (int k = 0; k < 4; ++k) {
    std::vector<int> rgs(n);
    std::vector<int> seen;
    for (int i = 0; i < n; ++i) {
      if (k == 0) {
        rgs[i] = 0;
      } else if (k == 1) {
        rgs[i] = i;
      } else {
        const int key = k == 2 ? pr.type_key[i] : pr.node_key[i];
        int ix = -1;
        for (size_t j = 0; j < seen.size(); ++j)
          if (seen[j] == key) ix = (int)j;
        if (ix < 0) {
          ix = (int)seen.size();
          seen.push_back(key);
        }
        rgs[i] = ix;
      }
    }
    const int m = *std::max_element(rgs.begin(), rgs.end()) + 1;
    std::vector<double> pw(m, 0), me(m, 0);
    std::vector<int> cnt(m, 0);
    for (int i = 0; i < n; ++i) {
      pw[rgs[i]] += pr.power[i];
      me[rgs[i]] += pr.memory[i];
      cnt[rgs[i]] += 1;
    }
    double z = 0, obj = -1;
    bool ok = true;
    for (int gi = 0; gi < m && ok; ++gi) {
      if (cnt[gi] == 0 || me[gi] < pr.min_mem) {
        ok = false;
        break;
      }
      const double rho = (double)(cnt[gi] - 1) / (double)(pr.n_microbatches + cnt[gi] - 1);
      const double gv = pw[gi] * (1.0 - rho);
      z = gi == 0 ? gv : (gv < z ? gv : z);
    }
    if (ok) obj = (double)m * z;
    if (obj > best) best = obj;
  }
  return best;
}

}  // namespace

#ifndef HPK_WIDE
// The wide (128-unit) build's entry points (hpk_grouping_wide.cu).
extern "C" int hpk_grouping_search_wide(const hpk_grouping_problem*, int, hpk_grouping_result*,
                                        const hpk_search_config*);
extern "C" void hpk_last_timing_wide(hpk_timing*);
extern "C" void hpk_reset_timing_wide(void);
extern "C" const char* hpk_last_error_wide(void);
#endif

// Hooks shared with hpk_partition.cu (same thread-local error / timing).
void hpkp_fail(const std::string& msg) { t_err = msg; }
namespace hpk_timing_bridge {
void add_pipeline(double ms, long long h2d, long long d2h) {
  t_timing.pipeline_ms += ms;
  t_timing.kernel_launches += 1;
  t_timing.h2d_bytes += h2d;
  t_timing.d2h_bytes += d2h;
}
void add_affinity(double ms, long long h2d, long long d2h) {
  t_timing.affinity_ms += ms;
  t_timing.kernel_launches += 1;
  t_timing.h2d_bytes += h2d;
  t_timing.d2h_bytes += d2h;
}
void add_partition(double ms, long long h2d, long long d2h) {
  t_timing.partition_ms += ms;
  t_timing.h2d_bytes += h2d;
  t_timing.d2h_bytes += d2h;
  t_timing.kernel_launches += 1;
}
void reset() { t_timing = hpk_timing{}; }
}  // namespace hpk_timing_bridge

extern "C" {

// Runs the device filter decision on n cases (A, D, cut triplets; rem = rm[2])
// and writes the codes; used by the GPU tests to pin decide() (see its note).
int hpk_selftest_decide(const double* cases, int n, const double* rm4, double mb_abs,
                        double md_abs, int* out_codes) {
  if (hpk_device_count() <= 0) return fail(5, "hetplan_b200: no CUDA device visible");
  double *din, *drm;
  int* dout;
  HPK_CUDA(cudaMalloc(&din, sizeof(double) * 3 * (size_t)n));
  HPK_CUDA(cudaMalloc(&drm, sizeof(double) * 4));
  HPK_CUDA(cudaMalloc(&dout, sizeof(int) * (size_t)n));
  HPK_CUDA(cudaMemcpy(din, cases, sizeof(double) * 3 * (size_t)n, cudaMemcpyHostToDevice));
  HPK_CUDA(cudaMemcpy(drm, rm4, sizeof(double) * 4, cudaMemcpyHostToDevice));
  hpk_selftest_decide_kernel<<<1, 32>>>(din, n, drm, mb_abs, md_abs, dout);
  HPK_CUDA(cudaGetLastError());
  HPK_CUDA(cudaMemcpy(out_codes, dout, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost));
  cudaFree(din);
  cudaFree(drm);
  cudaFree(dout);
  return 0;
}

const char* hpk_version(void) { return "hetplan-b200 0.1.0 (sm_100a)"; }
const char* hpk_last_error(void) { return t_err.c_str(); }

int hpk_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void hpk_search_config_init(hpk_search_config* cfg) {
  if (!cfg) return;
  cfg->device = -1;
  cfg->segment_cap = 0;
  cfg->max_list = 0;
  cfg->force_serial = 0;
  cfg->enumerate = 0;
  cfg->max_waves = 0;
  cfg->max_seconds = 0;
  cfg->max_ctas = 0;
  cfg->cut_intervals = -1;
}

void hpk_last_timing(hpk_timing* out) {
  if (out) *out = t_timing;
}

void hpk_reset_timing(void) { t_timing = hpk_timing{}; }

}  // extern "C"

namespace hpk {

int search_device(const hpk_grouping_problem* problems, int n_problems,
                  hpk_grouping_result* results, const hpk_search_config& cfg, int slot = 0);

// Relative cost of one search for the device assignment: a budgeted search
// runs node_budget visits, an exhaustive one Bell(n); deeper searches cost more
// per visit (more groups per node check), hence the unit-count weight.
double search_cost(const hpk_grouping_problem& pr) {
  double bell = 1;  // Bell(n) by the Bell triangle, capped
  {
    std::vector<double> row{1.0};
    for (int i = 1; i < pr.n && bell < 1e18; ++i) {
      std::vector<double> next{row.back()};
      for (double x : row) next.push_back(next.back() + x);
      row.swap(next);
      bell = row.back();
    }
  }
  const bool budgeted = pr.n > pr.exact_threshold && pr.node_budget >= 0;
  const double visits = budgeted ? std::min<double>((double)pr.node_budget, bell) : bell;
  return visits * (double)(pr.n + 8);
}

// Longest-first (LPT) assignment of searches to devices: each problem, in
// decreasing search_cost (ties: caller order), to the device with the least
// assigned cost so far (ties: the lowest ordinal).
void assign_devices(const hpk_grouping_problem* problems, int n, int ndev, int* out) {
  std::vector<int> order(n);
  std::vector<double> cost(n);
  for (int i = 0; i < n; ++i) {
    order[i] = i;
    cost[i] = search_cost(problems[i]);
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  std::vector<double> load(std::max(1, ndev), 0.0);
  for (int i : order) {
    const int d = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    load[d] += cost[i];
    out[i] = d;
  }
}

// One device, concurrent partitions: each long budgeted search of a small launch
// (the single-plan, latency-bound case) runs alone as its own persistent
// cooperative kernel on an equal share of the CTA slots (at most HPK_SPLIT_MAX
// partitions; shorter searches join the cheapest one), each on its own context
// slot and stream, one host thread each. The searches are independent: the
// long pole no longer waits for the others' schedule phases.
int split_device(const hpk_grouping_problem* problems, int n_problems,
                 hpk_grouping_result* results, const hpk_search_config& cfg, int device,
                 bool* done) {
  *done = false;
  if (n_problems < 2 || n_problems > 16 || cfg.force_serial || cfg.max_ctas > 0) return 0;
  std::vector<std::pair<double, int>> big;
  for (int i = 0; i < n_problems; ++i) {
    const hpk_grouping_problem& pr = problems[i];
    if (pr.node_budget <= 0 || pr.n <= pr.exact_threshold || pr.n > MAXN || pr.top_k > KW)
      continue;  // budgeted wave-engine searches only
    const double c = search_cost(pr);
    if (c >= 1e6) big.push_back({-c, i});
  }
  if (big.size() < 2) return 0;  // one long search: nothing to isolate it from
  std::sort(big.begin(), big.end());
  const int K = std::min((int)big.size(), HPK_SPLIT_MAX);
  DeviceCtx& c0 = g_ctx[device];
  {
    std::lock_guard<std::mutex> lock(c0.mu);
    if (int rc = ensure_ctx(c0, device)) return rc;
  }
  const int slots = c0.sms * c0.blocks_per_sm;
  if (slots / K < 1) return 0;
  std::vector<std::vector<int>> part(K);
  std::vector<double> pcost(K, 0.0);
  std::vector<char> placed(n_problems, 0);
  for (int k = 0; k < K; ++k) {
    part[k].push_back(big[k].second);
    pcost[k] = -big[k].first;
    placed[big[k].second] = 1;
  }
  for (int i = 0; i < n_problems; ++i) {  // the rest: to the cheapest partition
    if (placed[i]) continue;
    const int k = (int)(std::min_element(pcost.begin(), pcost.end()) - pcost.begin());
    part[k].push_back(i);
    pcost[k] += search_cost(problems[i]);
  }
  std::vector<std::vector<hpk_grouping_problem>> pp(K);
  std::vector<std::vector<hpk_grouping_result>> rr(K);
  std::vector<hpk_timing> tt(K);
  std::vector<std::string> ee(K);
  std::vector<int> rc(K, 0);
  for (int k = 0; k < K; ++k)
    for (int i : part[k]) {
      pp[k].push_back(problems[i]);
      rr[k].push_back(results[i]);
    }
  auto run = [&](int k) {
    hpk_search_config ck = cfg;
    ck.device = device;
    ck.max_ctas = slots / K;
    t_timing = hpk_timing{};
    rc[k] = search_device(pp[k].data(), (int)pp[k].size(), rr[k].data(), ck, k);
    tt[k] = t_timing;
    ee[k] = t_err;
  };
  const hpk_timing before = t_timing;
  std::vector<std::thread> workers;
  for (int k = 1; k < K; ++k) workers.emplace_back(run, k);
  run(0);
  for (auto& w : workers) w.join();
  t_timing = before;
  double sm = 0, se = 0;
  for (int k = 0; k < K; ++k) {
    sm = std::max(sm, tt[k].search_ms);
    se = std::max(se, tt[k].serial_ms);
    t_timing.h2d_bytes += tt[k].h2d_bytes;
    t_timing.d2h_bytes += tt[k].d2h_bytes;
    t_timing.kernel_launches += tt[k].kernel_launches;
  }
  t_timing.search_ms += sm;
  t_timing.serial_ms += se;
  for (int k = 0; k < K; ++k)
    if (rc[k] != 0) {
      t_err = ee[k];
      return rc[k];
    }
  for (int k = 0; k < K; ++k)
    for (size_t m = 0; m < part[k].size(); ++m) results[part[k][m]] = rr[k][m];
  *done = true;
  return 0;
}

// hpk_grouping_search over every visible device: problems go longest-first to
// the least-loaded device (one host thread and one persistent kernel per
// device, each on its own context and stream); results land in the caller's
// slots. Device time is the max over devices (they run concurrently).
int search_all_devices(const hpk_grouping_problem* problems, int n_problems,
                       hpk_grouping_result* results, const hpk_search_config& cfg, int ndev) {
  const int D = std::min(ndev, 16);
  std::vector<int> dev(n_problems);
  assign_devices(problems, n_problems, D, dev.data());
  std::vector<std::vector<int>> mine(D);
  for (int i = 0; i < n_problems; ++i) mine[dev[i]].push_back(i);  // caller order
  std::vector<int> rc(D, 0);
  std::vector<hpk_timing> tim(D);
  std::vector<std::string> err(D);
  auto run = [&](int d) {
    if (mine[d].empty()) return;
    std::vector<hpk_grouping_problem> pb;
    std::vector<hpk_grouping_result> rs;
    for (int i : mine[d]) {
      pb.push_back(problems[i]);
      rs.push_back(results[i]);
    }
    hpk_search_config c = cfg;
    c.device = d;
    t_timing = hpk_timing{};
    rc[d] = search_device(pb.data(), (int)pb.size(), rs.data(), c);
    tim[d] = t_timing;
    err[d] = t_err;
    for (size_t k = 0; k < mine[d].size(); ++k) results[mine[d][k]] = rs[k];
  };
  std::vector<std::thread> workers;
  for (int d = 1; d < D; ++d) workers.emplace_back(run, d);
  const hpk_timing before = t_timing;
  run(0);
  for (auto& w : workers) w.join();
  t_timing = before;
  for (int d = 0; d < D; ++d) {
    t_timing.search_ms = std::max(t_timing.search_ms, before.search_ms + tim[d].search_ms);
    t_timing.serial_ms = std::max(t_timing.serial_ms, before.serial_ms + tim[d].serial_ms);
    t_timing.h2d_bytes += tim[d].h2d_bytes;
    t_timing.d2h_bytes += tim[d].d2h_bytes;
    t_timing.kernel_launches += tim[d].kernel_launches;
  }
  t_timing.devices_used = 0;
  for (int d = 0; d < D; ++d) t_timing.devices_used += mine[d].empty() ? 0 : 1;
  for (int d = 0; d < D; ++d)
    if (rc[d] != 0) {
      t_err = err[d];
      return rc[d];
    }
  return 0;
}

}  // namespace hpk

extern "C" {

int hpk_assign_devices(const hpk_grouping_problem* problems, int n_problems, int n_devices,
                       int* out_device) {
  if (n_problems < 0 || n_devices < 1 || (n_problems > 0 && (!problems || !out_device)))
    return 6;
  assign_devices(problems, n_problems, n_devices, out_device);
  return 0;
}

int hpk_grouping_search(const hpk_grouping_problem* problems, int n_problems,
                        hpk_grouping_result* results, const hpk_search_config* cfg_in) {
  t_err.clear();
  if (n_problems <= 0) return 0;
  hpk_search_config cfg;
  hpk_search_config_init(&cfg);
  if (cfg_in) cfg = *cfg_in;
  const int ndev = hpk_device_count();
  if (ndev <= 0)
    return fail(5, "hetplan_b200: no CUDA device visible; the B200 planner has no CPU "
                   "fallback");
  if (cfg.device == HPK_ALL_DEVICES) {
    // a batch worth less than ~100 K budgeted visits stays on one device: the
    // extra host threads and launches would cost more than the split saves
    double total = 0;
    for (int i = 0; i < n_problems; ++i) total += search_cost(problems[i]);
    if (ndev > 1 && total > 5e6) return search_all_devices(problems, n_problems, results, cfg, ndev);
    cfg.device = 0;
  }
  if (cfg.device < 0) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) d = 0;
    cfg.device = d;
  }
  if (HPK_SPLIT_ONE_DEVICE) {
    bool done = false;
    if (int rc = split_device(problems, n_problems, results, cfg, cfg.device, &done)) return rc;
    if (done) {
      t_timing.devices_used = std::max(t_timing.devices_used, 1);
      return 0;
    }
  }
  const int rc = search_device(problems, n_problems, results, cfg);
  t_timing.devices_used = std::max(t_timing.devices_used, 1);
  return rc;
}

}  // extern "C"

namespace hpk {

int search_device(const hpk_grouping_problem* problems, int n_problems,
                  hpk_grouping_result* results, const hpk_search_config& cfg, int slot) {
  const int ndev = hpk_device_count();
  int device = cfg.device;
  if (device < 0) {
    if (cudaGetDevice(&device) != cudaSuccess) device = 0;
  }
  if (device >= ndev || device >= 16) return fail(6, "hetplan_b200: bad device ordinal");
  DeviceCtx& c = g_ctx[device + 16 * slot];
  std::lock_guard<std::mutex> lock(c.mu);
  if (int rc = ensure_ctx(c, device)) return rc;
  HPK_CUDA(cudaSetDevice(device));

  // Partition problems between the engines.
  std::vector<int> wave_ix, serial_ix, enum_ix, wide_ix;
  for (int i = 0; i < n_problems; ++i) {
    const hpk_grouping_problem& pr = problems[i];
    results[i].status = 0;
    results[i].count = 0;
    results[i].optimal = 0;
    results[i].visited = 0;
    results[i].waves = 0;
    results[i].segment_runs = 0;
    results[i].segment_visits = 0;
    results[i].max_list = 0;
    results[i].exact_checks = 0;
    if (pr.n < 1) return fail(6, "grouping: no devices");
    const bool contract = exact_sums(pr.power, pr.n, 0, false) &&
                          exact_sums(pr.memory, pr.n, 0, false);
    // outside the exact-sum contract the wave engine still runs, checking every
    // += for drift; the enumeration engine (fresh sums only) needs the contract
    const bool wave_ok = !cfg.force_serial && pr.n <= MAXN && pr.top_k <= KW;
    const bool enum_ok = wave_ok && contract && cfg.enumerate && pr.n <= pr.exact_threshold &&
                         pr.n <= ENUM_MAXN;
#ifndef HPK_WIDE
    if (!cfg.force_serial && !wave_ok && pr.n <= HPK_MAX_UNITS && pr.top_k <= KW) {
      wide_ix.push_back(i);  // 65..128 units: the wide build's wave engine
      continue;
    }
#endif
    (enum_ok ? enum_ix : wave_ok ? wave_ix : serial_ix).push_back(i);
  }
#ifndef HPK_WIDE
  if (!wide_ix.empty()) {
    std::vector<hpk_grouping_problem> wp;
    std::vector<hpk_grouping_result> wr;
    for (int i : wide_ix) {
      wp.push_back(problems[i]);
      wr.push_back(results[i]);
    }
    hpk_search_config wc = cfg;
    wc.device = device;
    hpk_reset_timing_wide();
    const int rc = hpk_grouping_search_wide(wp.data(), (int)wp.size(), wr.data(), &wc);
    hpk_timing tw;
    hpk_last_timing_wide(&tw);
    t_timing.search_ms += tw.search_ms;
    t_timing.serial_ms += tw.serial_ms;
    t_timing.h2d_bytes += tw.h2d_bytes;
    t_timing.d2h_bytes += tw.d2h_bytes;
    t_timing.kernel_launches += tw.kernel_launches;
    if (rc != 0) return fail(rc, hpk_last_error_wide());
    for (size_t k = 0; k < wide_ix.size(); ++k) results[wide_ix[k]] = wr[k];
  }
#endif

  // ---------------- enumeration engine (exhaustive searches, planner path)
  if (!enum_ix.empty()) {
    EnumTable tab;
    std::memset(&tab, 0, sizeof(tab));
    for (int g = 0; g <= ENUM_MAXN + 1; ++g) tab.D[0][g] = 1;
    for (int r = 1; r <= ENUM_MAXN; ++r)
      for (int g = 0; g <= ENUM_MAXN; ++g) tab.D[r][g] = g * tab.D[r - 1][g] + tab.D[r - 1][g + 1];
    const int per_block = 512;  // spread even the 8-unit cases over several SMs
    const int E = (int)enum_ix.size();
    std::vector<EnumProb> ep(E);
    int nblocks = 0, nout = 0;
    for (int k = 0; k < E; ++k) {
      const hpk_grouping_problem& pr = problems[enum_ix[k]];
      EnumProb& e = ep[k];
      std::memset(&e, 0, sizeof(e));
      e.n = pr.n;
      e.K = pr.n_microbatches;
      e.top_k = std::max(1, pr.top_k);
      e.floor_ = seed_floor(pr);
      e.min_mem = pr.min_mem;
      for (int i = 0; i < pr.n; ++i) {
        e.p[i] = pr.power[i];
        e.m[i] = pr.memory[i];
      }
      e.total = tab.D[pr.n - 1][1];  // Bell(n): digit 0 is fixed
      e.block0 = nblocks;
      e.nblocks = (int)((e.total + per_block - 1) / per_block);
      e.out0 = nout;
      nblocks += e.nblocks;
      nout += e.nblocks * e.top_k;
    }
    HpkArena& ar = c.arena;
    ar.reset();
    const size_t o_p = ar.take(sizeof(EnumProb) * E);
    const size_t o_t = ar.take(sizeof(EnumTable));
    const size_t in_end = ar.used;
    const size_t o_b = ar.take(sizeof(EnumBest) * nout);
    const size_t o_a = ar.take(sizeof(int) * nblocks);
    const size_t out_end = ar.used;
    HPK_CUDA(ar.fit());
    std::memcpy(ar.h + o_p, ep.data(), sizeof(EnumProb) * E);
    std::memcpy(ar.h + o_t, &tab, sizeof(EnumTable));
    HPK_CUDA(cudaMemcpyAsync(ar.d, ar.h, in_end, cudaMemcpyHostToDevice, c.stream));
    HPK_CUDA(cudaEventRecord(c.ev0, c.stream));
    hpk_enum_kernel<<<nblocks, 256, 0, c.stream>>>(ar.dp<EnumProb>(o_p), E, ar.dp<EnumTable>(o_t),
                                                   ar.dp<EnumBest>(o_b), ar.dp<int>(o_a),
                                                   per_block);
    HPK_CUDA(cudaGetLastError());
    HPK_CUDA(cudaEventRecord(c.ev1, c.stream));
    HPK_CUDA(cudaMemcpyAsync(ar.h + o_b, ar.d + o_b, out_end - o_b, cudaMemcpyDeviceToHost,
                             c.stream));
    HPK_CUDA(cudaStreamSynchronize(c.stream));
    float ms = 0;
    HPK_CUDA(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
    t_timing.search_ms += ms;
    t_timing.kernel_launches += 1;
    t_timing.h2d_bytes += (long long)in_end;
    t_timing.d2h_bytes += (long long)(out_end - o_b);
    const EnumBest* eb = ar.hp<EnumBest>(o_b);
    const int* na = ar.hp<int>(o_a);
    auto key_less = [](const EnumBest& x, const EnumBest& y) {  // x ranks before y
      if (x.obj != y.obj) return x.obj > y.obj;
      if (x.G != y.G) return x.G < y.G;
      return x.rank < y.rank;
    };
    for (int k = 0; k < E; ++k) {
      const int i = enum_ix[k];
      const hpk_grouping_problem& pr = problems[i];
      hpk_grouping_result& r = results[i];
      const int tk = ep[k].top_k;
      std::vector<EnumBest> all;
      long long above = 0;
      for (int q = 0; q < ep[k].nblocks; ++q) {
        above += na[ep[k].block0 + q];
        for (int t = 0; t < tk; ++t) {
          const EnumBest& x = eb[(size_t)ep[k].out0 + (size_t)q * tk + t];
          if (x.obj >= 0) all.push_back(x);
        }
      }
      if (tk > 1 && above < tk) {  // the DFS's list depends on its pruning: wave engine
        wave_ix.push_back(i);
        continue;
      }
      std::sort(all.begin(), all.end(), key_less);
      r.engine = 2;
      r.visited = -1;  // not counted by this engine
      if (all.empty()) {  // no feasible leaf: no seed is feasible either (seeds are leaves)
        r.status = 3;
        continue;
      }
      const int cnt = std::min<int>(tk, (int)all.size());
      r.count = cnt;
      r.optimal = 1;
      for (int t = 0; t < cnt; ++t) {
        uint8_t rgs[ENUM_MAXN];
        rgs[0] = 0;
        int g = 1;
        long long kk = all[t].rank;
        for (int u = 1; u < pr.n; ++u) {
          const long long w = tab.D[pr.n - 1 - u][g];
          const long long q = kk / w;
          if (q < g) {
            rgs[u] = (uint8_t)q;
            kk -= q * w;
          } else {
            rgs[u] = (uint8_t)g;
            kk -= (long long)g * w;
            ++g;
          }
        }
        r.objective[t] = all[t].obj;
        r.z[t] = leaf_z(pr, rgs, all[t].G);
        for (int u = 0; u < pr.n; ++u) r.rgs[(size_t)t * pr.n + u] = rgs[u];
      }
    }
  }

  // ---------------- wave engine
  if (!wave_ix.empty()) {
    const int P = (int)wave_ix.size();
    // (big batches — a replanning sweep — run longer segments: fewer splits and
    // list positions for the same work; one plan's few searches need the
    // shorter cap to spread their fronts)
    const long long seg_cap = cfg.segment_cap > 0 ? cfg.segment_cap
                              : (P > 16 ? HPK_SEG_CAP_BATCH : HPK_SEG_CAP);
    // list capacity (ids) and entry-pool capacity per problem; large by default
    // (the list must hold the whole speculative frontier), scaled down so that
    // big batches (cfg5 sweeps) stay within ~4 GB of HBM.
    bool any_topk = false;
    for (int k = 0; k < P; ++k) any_topk = any_topk || problems[wave_ix[k]].top_k > 1;
    const size_t entry_bytes = sizeof(Entry) + (any_topk ? sizeof(CandRec) : 0);
    int lcap = cfg.max_list > 0 ? cfg.max_list : (1 << 17);
    int pcap = 2 * lcap;
    while (lcap > 4096 &&
           (size_t)P * ((size_t)pcap * 2 * entry_bytes + (size_t)lcap * 108) > ((size_t)4 << 30)) {
      lcap /= 2;
      pcap /= 2;
    }
    int max_n = 1;
    for (int k = 0; k < P; ++k) max_n = std::max(max_n, problems[wave_ix[k]].n);
    // piece shape: sibling ranges for big batches (cfg5: 1.3x faster, shorter
    // lists), single siblings for a few problems (cfg3: 1.9x faster — more
    // parallel pieces near one search's commit front)
    const int ranges = P > 16 ? 1 : 0;
    const int reserve = ranges ? max_n + 64                     // one piece per level
                               : max_n * (max_n + 1) / 2 + 98;  // one per sibling
    if (pcap < 4 * reserve) pcap = 4 * reserve;
    std::vector<GProb> hp(P);
    for (int k = 0; k < P; ++k) {
      const hpk_grouping_problem& pr = problems[wave_ix[k]];
      GProb& g = hp[k];
      std::memset(&g, 0, sizeof(GProb));
      g.n = pr.n;
      g.K = pr.n_microbatches;
      g.budget = pr.n <= pr.exact_threshold ? -1 : pr.node_budget;
      g.min_mem = pr.min_mem;
      g.top_k = std::max(1, pr.top_k);
      g.exact_mem = exact_sums(pr.memory, pr.n, pr.min_mem, true) ? 1 : 0;
      g.check_drift = exact_sums(pr.power, pr.n, 0, false) && exact_sums(pr.memory, pr.n, 0, false)
                          ? 0 : 1;
      for (int i = 0; i < pr.n; ++i) {
        g.p[i] = pr.power[i];
        g.m[i] = pr.memory[i];
        g.tkey[i] = pr.type_key[i];
        g.nkey[i] = pr.node_key[i];
      }
    }
    if (int rc = grow(c.probs, c.cap_probs, (size_t)P)) return rc;
    if (int rc = grow(c.states, c.cap_states, (size_t)P)) return rc;
    if (int rc = grow(c.pools, c.cap_pools, (size_t)P * 2 * pcap)) return rc;
    if (any_topk)
      if (int rc = grow(c.cands, c.cap_cands, (size_t)P * 2 * pcap)) return rc;
    if (int rc = grow(c.lists, c.cap_lists, (size_t)P * 2 * 6 * lcap)) return rc;
    if (int rc = grow(c.scratch, c.cap_scratch, (size_t)P * (lcap + 1))) return rc;
    if (int rc = grow(c.lvis, c.cap_lvis, (size_t)P * 2 * lcap)) return rc;
    if (int rc = grow(c.ldbl, c.cap_ldbl, (size_t)P * 6 * lcap)) return rc;
    const int xtn = lcap / TILE + 2;
    if (int rc = grow(c.xt, c.cap_xt, (size_t)P * xtn)) return rc;
    if (int rc = grow(c.work, c.cap_work, (size_t)2 * P * xtn)) return rc;
    if (int rc = grow(c.agg, c.cap_agg, (size_t)P * xtn)) return rc;
    if (int rc = grow(c.pagg, c.cap_pagg, (size_t)P * xtn)) return rc;
    HPK_CUDA(cudaMemsetAsync(c.pagg, 0xff, sizeof(PushAgg) * P * xtn, c.stream));  // stamps -1
    HPK_CUDA(cudaMemsetAsync(c.xt, 0, sizeof(int) * P * xtn, c.stream));
    const int grid = cfg.max_ctas > 0 ? std::min(cfg.max_ctas, c.sms * c.blocks_per_sm)
                                      : c.sms * c.blocks_per_sm;
    const int nwarps = grid * WARPS_PER_BLOCK;
    // total run slots per wave, shared by the active problems (most segments are
    // small: several per warp keep the warps busy through the time slice)
    // (4 per warp and a 300 us slice: measured best on cfg4 / cfg3 after the
    // parallel queue step; HPK_QMUL / HPK_WAVE_US override)
    const int qmax = HPK_QMUL * (HPK_SPLIT_ONE_DEVICE ? c.sms * c.blocks_per_sm * WARPS_PER_BLOCK
                                                      : nwarps);
    const int qcap = qmax + 33 * P + 64;
    if (int rc = grow(c.items, c.cap_items, (size_t)2 * qcap)) return rc;

    HPK_CUDA(cudaMemcpyAsync(c.probs, hp.data(), sizeof(GProb) * P, cudaMemcpyHostToDevice,
                             c.stream));
    HPK_CUDA(cudaMemsetAsync(c.queues, 0, sizeof(RunQueue) * 2, c.stream));
    int init_flags[64] = {0};  // [0] active [1] err [2:4) deadline [4:6) barrier
    init_flags[0] = P;         // [6] active snapshot [7] stop [8:60) trace counters
    {
      int units = 0;  // [62] units of the active problems, [63] its snapshot
      for (int k = 0; k < P; ++k) units += problems[wave_ix[k]].n;
      init_flags[62] = units;
      init_flags[63] = units;
    }
                               // [60:62) expansion work counts
    HPK_CUDA(cudaMemcpyAsync(c.active, init_flags, sizeof(int) * 64, cudaMemcpyHostToDevice,
                             c.stream));
    t_timing.h2d_bytes += sizeof(GProb) * P + sizeof(int);

    KParams kp;
    kp.probs = c.probs;
    kp.states = c.states;
    kp.pools = c.pools;
    kp.cands = any_topk ? c.cands : nullptr;
    kp.lists = c.lists;
    kp.lvis = c.lvis;
    kp.ldbl = c.ldbl;
    kp.scratch = c.scratch;
    kp.xt = c.xt;
    kp.xtn = xtn;
    kp.agg = c.agg;
    kp.pagg = c.pagg;
    kp.par_push = 1;
    kp.work = c.work;
    kp.wcap = P * xtn;
    kp.wcount = c.active + 60;
    kp.queues = c.queues;
    kp.items = c.items;
    kp.active = c.active;
    kp.err = c.active + 1;
    kp.stop = c.active + 7;
    kp.runners = WARPS_PER_BLOCK;
    kp.ranges = ranges;
    kp.cut_iv = cfg.cut_intervals < 0 ? (P <= HPK_CUT_IV_MAX ? 1 : 0) : (cfg.cut_intervals != 0);
    // run-phase time slice: 300 us (HPK_WAVE_US overrides; 0 = none)
    kp.wave_ns = HPK_WAVE_NS;
    kp.n_problems = P;
    kp.lcap = lcap;
    kp.pcap = pcap;
    kp.reserve = reserve;
    kp.qcap = qcap;
    kp.qmax = qmax;
    // (a lone search's share is sized by the whole device: a launch on part of
    // the SMs still runs its long runs side by side, the tiny ones fill in)
    kp.qmax_one = (int)(HPK_QONE * (HPK_SPLIT_ONE_DEVICE ? c.sms * c.blocks_per_sm * WARPS_PER_BLOCK
                                                         : nwarps));
    kp.seg_cap = seg_cap;
    kp.front_cap = seg_cap;
    kp.ramp = 64;  // measured: -0.7 ms cfg4, -1.3 ms tp1 alone
    kp.max_waves = cfg.max_waves > 0 ? cfg.max_waves : 0x7fffffff;  // explicit watchdog only
    // watchdog: an explicit max_seconds, else derived from the budgets (a
    // visit rate 100x below the slowest measured, plus 60 s); searches with no
    // budget (exhaustive mode) have no deadline, like the reference
    double secs = cfg.max_seconds;
    if (secs <= 0) {
      long long tot = 0;
      bool unbounded = false;
      for (int k = 0; k < P; ++k) {
        const hpk_grouping_problem& pr = problems[wave_ix[k]];
        if (pr.n <= pr.exact_threshold || pr.node_budget < 0) unbounded = pr.n > 12 || unbounded;
        else tot += pr.node_budget;
      }
      secs = unbounded ? 0.0 : 60.0 + (double)tot / 1e6;
    }
    kp.deadline_ns = secs > 0 ? (unsigned long long)(secs * 1e9) : ~0ull;
    kp.deadline_slot = reinterpret_cast<unsigned long long*>(c.active + 2);
    kp.bar = reinterpret_cast<unsigned int*>(c.active + 4);
    kp.prof = reinterpret_cast<unsigned long long*>(c.active + 8);
    kp.trace = HPK_TRACE_LEVEL;  // build-time: -DHPK_TRACE_LEVEL=n
    kp.trace_p = -1;
    const size_t smem = sizeof(WarpSmem) * WARPS_PER_BLOCK + sizeof(SchedSmem);
    void* args[] = {&kp};
    HPK_CUDA(cudaEventRecord(c.ev0, c.stream));
    HPK_CUDA(cudaLaunchCooperativeKernel((void*)hpk_wave_kernel, dim3(grid),
                                         dim3(BLOCK_THREADS), args, smem, c.stream));
    HPK_CUDA(cudaEventRecord(c.ev1, c.stream));
    t_timing.kernel_launches += 1;
    std::vector<GState> hs(P);
    int flags_out[2] = {0, 0};
    HPK_CUDA(cudaMemcpyAsync(hs.data(), c.states, sizeof(GState) * P, cudaMemcpyDeviceToHost,
                             c.stream));
    HPK_CUDA(cudaMemcpyAsync(flags_out, c.active, sizeof(int) * 2, cudaMemcpyDeviceToHost,
                             c.stream));
    HPK_CUDA(cudaStreamSynchronize(c.stream));
    if (flags_out[1] & 1) return fail(5, "hetplan_b200: segment runner watchdog tripped");
    if (flags_out[1] & 2) return fail(5, "hetplan_b200: wave engine exceeded its time budget");
    if (flags_out[1] & 4) return fail(5, "hetplan_b200: run queue overflow (scheduler bug)");
    t_timing.d2h_bytes += sizeof(GState) * P;
    float ms = 0;
    HPK_CUDA(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
    t_timing.search_ms += ms;
    for (int k = 0; k < P; ++k) {
      const int i = wave_ix[k];
      const hpk_grouping_problem& pr = problems[i];
      hpk_grouping_result& r = results[i];
      const GState& s = hs[k];
      r.engine = 0;
      r.waves = s.waves;
      r.segment_runs = s.runs;
      r.segment_visits = s.run_visits;
      r.max_list = s.max_list;
      r.exact_checks = s.exact_checks;
      r.visited = s.V;
      if (s.error & (8 | 16)) {  // > 63 groups, or drifting sums: exact serial replay
        serial_ix.push_back(i);
        continue;
      }
      if (!s.done)
        return fail(5, "hetplan_b200: wave engine did not converge within " +
                           std::to_string(kp.max_waves) + " waves (problem " +
                           std::to_string(i) + ", waves " + std::to_string(s.waves) +
                           ", visits " + std::to_string(s.V) + ")");
      const bool optimal = !s.aborted;
      if (pr.top_k > 1) {
        // result rules, grouping.cpp:316-334, over the top_k list
        if (s.nbest == 0 && s.seed_obj < 0) {
          r.status = 3;
          continue;
        }
        if (s.nbest == 0 || (!optimal && s.seed_obj > s.bl_obj[0])) {
          r.count = 1;
          r.objective[0] = s.seed_obj;
          r.z[0] = s.seed_z;
          r.optimal = 0;
          for (int u = 0; u < pr.n; ++u) r.rgs[u] = s.seed_rgs[u];
          continue;
        }
        r.count = s.nbest;
        r.optimal = optimal ? 1 : 0;
        for (int t = 0; t < s.nbest; ++t) {
          r.objective[t] = s.bl_obj[t];
          r.z[t] = leaf_z(pr, s.bl_rgs[t], s.bl_G[t]);
          for (int u = 0; u < pr.n; ++u) r.rgs[(size_t)t * pr.n + u] = s.bl_rgs[t][u];
        }
        continue;
      }
      // result rules, grouping.cpp:316-334
      if (!s.has_best) {
        if (s.seed_obj < 0) {
          r.status = 3;
          continue;
        }
      }
      if (!s.has_best || (!optimal && s.seed_obj > s.best_obj)) {
        r.count = 1;
        r.objective[0] = s.seed_obj;
        r.z[0] = s.seed_z;
        r.optimal = 0;
        for (int u = 0; u < pr.n; ++u) r.rgs[u] = s.seed_rgs[u];
        continue;
      }
      r.count = 1;
      r.objective[0] = s.best_obj;
      // z = objective / G is not how the reference gets z; recompute it from
      // the partition exactly as the leaf did (min effective power).
      {
        double pw[MAXN] = {0}, me[MAXN] = {0};
        int cn[MAXN] = {0};
        for (int u = 0; u < pr.n; ++u) {
          pw[s.best_rgs[u]] += pr.power[u];
          me[s.best_rgs[u]] += pr.memory[u];
          cn[s.best_rgs[u]] += 1;
        }
        double z = 0;
        for (int gi = 0; gi < s.best_G; ++gi) {
          const double rho = (double)(cn[gi] - 1) / (double)(pr.n_microbatches + cn[gi] - 1);
          const double gv = pw[gi] * (1.0 - rho);
          z = gi == 0 ? gv : (gv < z ? gv : z);
        }
        r.z[0] = z;
      }
      r.optimal = optimal ? 1 : 0;
      for (int u = 0; u < pr.n; ++u) r.rgs[u] = s.best_rgs[u];
    }
  }

  // ---------------- serial replica engine
  if (!serial_ix.empty()) {
    const int P = (int)serial_ix.size();
    int max_n = 0;
    size_t tot_units = 0;
    for (int i : serial_ix) {
      max_n = std::max(max_n, problems[i].n);
      tot_units += problems[i].n;
    }
    if (max_n > 255) return fail(6, "hetplan_b200: more than 255 TP units unsupported");
    std::vector<double> hpw, hme;
    std::vector<int> htk, hnk;
    std::vector<size_t> off(P);
    size_t rgs_total = 0, k_total = 0;
    std::vector<size_t> rgs_off(P), k_off(P);
    for (int k = 0; k < P; ++k) {
      const hpk_grouping_problem& pr = problems[serial_ix[k]];
      off[k] = hpw.size();
      hpw.insert(hpw.end(), pr.power, pr.power + pr.n);
      hme.insert(hme.end(), pr.memory, pr.memory + pr.n);
      htk.insert(htk.end(), pr.type_key, pr.type_key + pr.n);
      hnk.insert(hnk.end(), pr.node_key, pr.node_key + pr.n);
      rgs_off[k] = rgs_total;
      rgs_total += (size_t)std::max(1, pr.top_k) * pr.n;
      k_off[k] = k_total;  // top_k results + (top_k + 1) list slots per problem
      k_total += (size_t)std::max(1, pr.top_k);
    }
    double *d_obj, *d_z;
    double *d_pw, *d_me, *d_scr;
    int *d_tk, *d_nk, *d_iscr, *d_rgs;
    SerialProb* d_probs;
    SerialCand* d_cands;
    HPK_CUDA(cudaMalloc(&d_pw, sizeof(double) * tot_units));
    HPK_CUDA(cudaMalloc(&d_me, sizeof(double) * tot_units));
    HPK_CUDA(cudaMalloc(&d_tk, sizeof(int) * tot_units));
    HPK_CUDA(cudaMalloc(&d_nk, sizeof(int) * tot_units));
    HPK_CUDA(cudaMalloc(&d_scr, sizeof(double) * (size_t)P * 2 * (max_n + 1)));
    HPK_CUDA(cudaMalloc(&d_iscr, sizeof(int) * (size_t)P * 4 * (max_n + 1)));
    HPK_CUDA(cudaMalloc(&d_rgs, sizeof(int) * rgs_total));
    HPK_CUDA(cudaMalloc(&d_probs, sizeof(SerialProb) * P));
    HPK_CUDA(cudaMalloc(&d_cands, sizeof(SerialCand) * (k_total + (size_t)P)));
    HPK_CUDA(cudaMalloc(&d_obj, sizeof(double) * k_total));
    HPK_CUDA(cudaMalloc(&d_z, sizeof(double) * k_total));
    std::vector<SerialProb> sp(P);
    for (int k = 0; k < P; ++k) {
      const hpk_grouping_problem& pr = problems[serial_ix[k]];
      SerialProb& s = sp[k];
      std::memset(&s, 0, sizeof(s));
      s.n = pr.n;
      s.K = pr.n_microbatches;
      s.top_k = std::max(1, pr.top_k);
      s.budget = pr.n <= pr.exact_threshold ? -1 : pr.node_budget;
      s.min_mem = pr.min_mem;
      s.p = d_pw + off[k];
      s.m = d_me + off[k];
      s.tkey = d_tk + off[k];
      s.nkey = d_nk + off[k];
      s.rgs_out = d_rgs + rgs_off[k];
      s.obj_out = d_obj + k_off[k];
      s.z_out = d_z + k_off[k];
      s.cand = d_cands + k_off[k] + (size_t)k;
    }
    HPK_CUDA(cudaMemcpyAsync(d_pw, hpw.data(), sizeof(double) * tot_units,
                             cudaMemcpyHostToDevice, c.stream));
    HPK_CUDA(cudaMemcpyAsync(d_me, hme.data(), sizeof(double) * tot_units,
                             cudaMemcpyHostToDevice, c.stream));
    HPK_CUDA(cudaMemcpyAsync(d_tk, htk.data(), sizeof(int) * tot_units, cudaMemcpyHostToDevice,
                             c.stream));
    HPK_CUDA(cudaMemcpyAsync(d_nk, hnk.data(), sizeof(int) * tot_units, cudaMemcpyHostToDevice,
                             c.stream));
    HPK_CUDA(cudaMemcpyAsync(d_probs, sp.data(), sizeof(SerialProb) * P, cudaMemcpyHostToDevice,
                             c.stream));
    HPK_CUDA(cudaEventRecord(c.ev0, c.stream));
    hpk_serial_kernel<<<(P + 31) / 32, 32, 0, c.stream>>>(d_probs, P, d_cands, d_scr, d_iscr,
                                                          max_n);
    HPK_CUDA(cudaGetLastError());
    HPK_CUDA(cudaEventRecord(c.ev1, c.stream));
    t_timing.kernel_launches += 1;
    HPK_CUDA(cudaMemcpyAsync(sp.data(), d_probs, sizeof(SerialProb) * P, cudaMemcpyDeviceToHost,
                             c.stream));
    std::vector<int> hrgs(rgs_total);
    HPK_CUDA(cudaMemcpyAsync(hrgs.data(), d_rgs, sizeof(int) * rgs_total,
                             cudaMemcpyDeviceToHost, c.stream));
    std::vector<double> hobj(k_total), hz(k_total);
    HPK_CUDA(cudaMemcpyAsync(hobj.data(), d_obj, sizeof(double) * k_total,
                             cudaMemcpyDeviceToHost, c.stream));
    HPK_CUDA(cudaMemcpyAsync(hz.data(), d_z, sizeof(double) * k_total, cudaMemcpyDeviceToHost,
                             c.stream));
    HPK_CUDA(cudaStreamSynchronize(c.stream));
    float ms = 0;
    cudaEventElapsedTime(&ms, c.ev0, c.ev1);
    t_timing.serial_ms += ms;
    for (int k = 0; k < P; ++k) {
      const int i = serial_ix[k];
      const hpk_grouping_problem& pr = problems[i];
      hpk_grouping_result& r = results[i];
      const SerialProb& s = sp[k];
      r.engine = 1;
      r.status = s.status;
      r.count = s.count;
      r.optimal = s.optimal;
      r.visited = s.visited;
      for (int t = 0; t < s.count; ++t) {
        r.objective[t] = hobj[k_off[k] + t];
        r.z[t] = hz[k_off[k] + t];
        for (int u = 0; u < pr.n; ++u) r.rgs[(size_t)t * pr.n + u] = hrgs[rgs_off[k] + t * pr.n + u];
      }
    }
    cudaFree(d_pw);
    cudaFree(d_me);
    cudaFree(d_tk);
    cudaFree(d_nk);
    cudaFree(d_scr);
    cudaFree(d_iscr);
    cudaFree(d_rgs);
    cudaFree(d_probs);
    cudaFree(d_cands);
    cudaFree(d_obj);
    cudaFree(d_z);
  }
  return 0;
}

}  // namespace hpk
