// hpk_pipeline.cu — the 1F1B pipeline simulator (simulate_pipeline,
// P/src/pipeline_sim.cpp:46-149; P = /root/reference/proj) on the B200,
// batched over every DP group of every plan of a call (simulate_1f1b,
// P/src/cost.cpp:149-182, hp_simulate c_api.cpp:286-303, the planner's
// validate_with_sim planner.cpp:207-219).
//
// One CTA per pipeline, one thread per stage (strided when P > blockDim). A
// stage's 2K tasks follow the reference's static order — min(K, P-1-p) warmup
// forwards, then F/B pairs, then the backward drain (:53-66) — and each task
// starts at max(stage free, producer end): F(p,m) waits for F(p-1,m), B(p,m)
// for B(p+1,m), B(P-1,m) for F(P-1,m) (:68-108). Threads resolve their next
// tasks in rounds separated by __syncthreads (the reference's ready-queue pass,
// whose result is independent of the resolution order because every start time
// is a max over dependency ends). Every value is the reference's own
// expression — max, then one add — so starts, ends, busy sums (stage order)
// and the makespan are bit-identical. The per-stage live-microbatch peak
// (:128-145: +1 at a forward start, -1 at a backward end, frees first on
// ties) is a merge of the stage's two time-sorted sequences, one thread per
// stage. Task times come back in stage order; the host sorts the event list
// the reference's way (:113-119).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "hetplan_b200.h"
#include "hpk_common.cuh"

void hpkp_fail(const std::string& msg);  // thread-local error of the hpk_* layer
namespace hpk_timing_bridge {
void add_pipeline(double ms, long long h2d, long long d2h);
}

namespace hpkq {

constexpr int THREADS = 128;

struct Pipe {
  int P, K;
  int stage_off;  // into the per-stage arrays
  int task_off;   // into the per-task arrays (P * 2K per pipeline)
  double makespan;
  int ok;
};

// Task i of stage p in the reference's static order: (forward?, microbatch).
__device__ __forceinline__ void task_of(int p, int i, int P, int K, bool* fwd, int* mb) {
  const int warm = min(K, P - 1 - p);
  if (i < warm) {
    *fwd = true;
    *mb = i;
  } else if (i < 2 * K - warm) {
    const int t = i - warm;
    *fwd = (t & 1) == 0;
    *mb = *fwd ? warm + (t >> 1) : (t >> 1);
  } else {
    *fwd = false;
    *mb = i - K;
  }
}

__global__ void __launch_bounds__(THREADS) pipeline_sim_kernel(
    Pipe* pipes, const double* fwd_t, const double* bwd_t, const double* send_f,
    const double* send_b, double* f_end, double* b_end, double* t_start, double* t_end,
    double* busy, int* peak) {
  Pipe& pp = pipes[blockIdx.x];
  const int P = pp.P, K = pp.K;
  const int so = pp.stage_off;
  const size_t to = pp.task_off;
  double* fe = f_end + (size_t)pp.task_off / 2;  // [P][K] forward ends (P*K per pipeline)
  double* be = b_end + (size_t)pp.task_off / 2;
  __shared__ int s_progress, s_left;
  for (int x = threadIdx.x; x < P * K; x += blockDim.x) {
    fe[x] = -1.0;
    be[x] = -1.0;
  }
  // per-stage cursor and free time live in registers of the owning thread
  constexpr int MAXL = 8;  // stages per thread (P <= 1024)
  int cur[MAXL];
  double freet[MAXL], bsum[MAXL];
#pragma unroll
  for (int k = 0; k < MAXL; ++k) {
    cur[k] = 0;
    freet[k] = 0.0;
    bsum[k] = 0.0;
  }
  double mk = 0.0;
  __syncthreads();
  while (true) {
    if (threadIdx.x == 0) {
      s_progress = 0;
      s_left = 0;
    }
    __syncthreads();
    int progressed = 0, left = 0;
#pragma unroll
    for (int k = 0; k < MAXL; ++k) {
      const int p = threadIdx.x + k * blockDim.x;
      if (p >= P) break;
      const double fdur = fwd_t[so + p] + (p + 1 < P ? send_f[so + p] : 0.0);
      const double bdur = bwd_t[so + p] + (p > 0 ? send_b[so + p] : 0.0);
      while (cur[k] < 2 * K) {
        bool fwd;
        int m;
        task_of(p, cur[k], P, K, &fwd, &m);
        double dep = 0.0;
        if (fwd) {
          if (p > 0) {
            dep = *((volatile double*)&fe[(p - 1) * K + m]);
            if (dep < 0) break;
          }
        } else if (p + 1 < P) {
          dep = *((volatile double*)&be[(p + 1) * K + m]);
          if (dep < 0) break;
        } else {
          dep = fe[p * K + m];  // precedes it in this stage's order
        }
        const double dur = fwd ? fdur : bdur;
        const double st = freet[k] < dep ? dep : freet[k];  // std::max(stage_free, dep)
        const double en = st + dur;
        freet[k] = en;
        (fwd ? fe : be)[p * K + m] = en;
        t_start[to + (size_t)p * 2 * K + cur[k]] = st;
        t_end[to + (size_t)p * 2 * K + cur[k]] = en;
        bsum[k] += dur;
        mk = mk < en ? en : mk;
        ++cur[k];
        progressed = 1;
      }
      if (cur[k] < 2 * K) left = 1;
    }
    __threadfence_block();
    if (progressed) s_progress = 1;
    if (left) s_left = 1;
    __syncthreads();
    const int prog = s_progress, lft = s_left;
    __syncthreads();
    if (!lft) break;
    if (!prog) {  // "1F1B schedule is deadlock-free" (:104) — cannot happen
      if (threadIdx.x == 0) pp.ok = 0;
      return;
    }
  }
  // makespan: max over the threads' maxima (exact)
  __shared__ unsigned long long s_mk;
  if (threadIdx.x == 0) s_mk = 0;
  __syncthreads();
  atomicMax(&s_mk, (unsigned long long)__double_as_longlong(mk));  // non-negative doubles
  __syncthreads();
#pragma unroll
  for (int k = 0; k < MAXL; ++k) {
    const int p = threadIdx.x + k * blockDim.x;
    if (p >= P) break;
    busy[so + p] = bsum[k];
    // peak live microbatches: merge forward starts (+1) and backward ends (-1),
    // both ascending in the stage's order; at equal times frees come first
    const double* ts = t_start + to + (size_t)p * 2 * K;
    const double* te = t_end + to + (size_t)p * 2 * K;
    int i = 0, j = 0, live = 0, best = 0;
    // next forward start / backward end in stage order
    auto next_f = [&](int from) {
      for (int q = from; q < 2 * K; ++q) {
        bool f;
        int mm;
        task_of(p, q, P, K, &f, &mm);
        if (f) return q;
      }
      return 2 * K;
    };
    auto next_b = [&](int from) {
      for (int q = from; q < 2 * K; ++q) {
        bool f;
        int mm;
        task_of(p, q, P, K, &f, &mm);
        if (!f) return q;
      }
      return 2 * K;
    };
    i = next_f(0);
    j = next_b(0);
    while (i < 2 * K || j < 2 * K) {
      bool take_b;
      if (i >= 2 * K) {
        take_b = true;
      } else if (j >= 2 * K) {
        take_b = false;
      } else {
        take_b = !(ts[i] < te[j]);  // (time, -1) sorts before (time, +1)
      }
      if (take_b) {
        --live;
        j = next_b(j + 1);
      } else {
        ++live;
        best = live > best ? live : best;
        i = next_f(i + 1);
      }
    }
    peak[so + p] = best;
  }
  if (threadIdx.x == 0) {
    pp.makespan = __longlong_as_double((long long)s_mk);
    pp.ok = 1;
  }
}

struct Ctx {
  int device = -1;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  HpkArena arena;
  std::mutex mu;
};
Ctx g_ctx[16];

}  // namespace hpkq

#define HPKQ_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess) {                                                              \
      hpkp_fail(std::string("hetplan_b200 CUDA error: ") + cudaGetErrorString(_e) +       \
                " at " #call);                                                            \
      return 5;                                                                           \
    }                                                                                     \
  } while (0)

extern "C" int hpk_pipeline_sim(hpk_pipeline* pipes, int n, int device) {
  using namespace hpkq;
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
  HPKQ_CUDA(cudaSetDevice(device));
  if (cx.device != device) {
    HPKQ_CUDA(cudaStreamCreateWithFlags(&cx.stream, cudaStreamNonBlocking));
    HPKQ_CUDA(cudaEventCreate(&cx.ev0));
    HPKQ_CUDA(cudaEventCreate(&cx.ev1));
    cx.device = device;
  }
  std::vector<Pipe> hp(n);
  size_t S = 0, T = 0;
  for (int k = 0; k < n; ++k) {
    const hpk_pipeline& in = pipes[k];
    if (in.n_stages < 1 || in.n_microbatches < 1) {
      hpkp_fail("invariant violated: pipeline needs at least one stage and microbatch "
                "[P >= 1 && K >= 1]");
      return 5;
    }
    if (in.n_stages > 8 * THREADS) {
      hpkp_fail("hetplan_b200: more than 1024 pipeline stages unsupported");
      return 6;
    }
    hp[k].P = in.n_stages;
    hp[k].K = in.n_microbatches;
    hp[k].stage_off = (int)S;
    hp[k].task_off = (int)T;
    hp[k].makespan = 0;
    hp[k].ok = 0;
    S += (size_t)in.n_stages;
    T += (size_t)in.n_stages * 2 * in.n_microbatches;
  }
  HpkArena& ar = cx.arena;
  ar.reset();
  const size_t o_p = ar.take(sizeof(Pipe) * n);
  const size_t o_f = ar.take(sizeof(double) * S);
  const size_t o_b = ar.take(sizeof(double) * S);
  const size_t o_sf = ar.take(sizeof(double) * S);
  const size_t o_sb = ar.take(sizeof(double) * S);
  const size_t in_end = ar.used;
  const size_t o_busy = ar.take(sizeof(double) * S);
  const size_t o_peak = ar.take(sizeof(int) * S);
  const size_t o_ts = ar.take(sizeof(double) * T);
  const size_t o_te = ar.take(sizeof(double) * T);
  const size_t out_end = ar.used;
  const size_t o_fe = ar.take(sizeof(double) * (T / 2 + 1));
  const size_t o_be = ar.take(sizeof(double) * (T / 2 + 1));
  HPKQ_CUDA(ar.fit());
  std::memcpy(ar.h + o_p, hp.data(), sizeof(Pipe) * n);
  for (int k = 0; k < n; ++k) {
    const hpk_pipeline& in = pipes[k];
    const size_t b = sizeof(double) * in.n_stages, off = sizeof(double) * hp[k].stage_off;
    std::memcpy(ar.h + o_f + off, in.forward, b);
    std::memcpy(ar.h + o_b + off, in.backward, b);
    std::memcpy(ar.h + o_sf + off, in.send_forward, b);
    std::memcpy(ar.h + o_sb + off, in.send_backward, b);
  }
  HPKQ_CUDA(cudaMemcpyAsync(ar.d, ar.h, in_end, cudaMemcpyHostToDevice, cx.stream));
  HPKQ_CUDA(cudaEventRecord(cx.ev0, cx.stream));
  pipeline_sim_kernel<<<n, THREADS, 0, cx.stream>>>(
      ar.dp<Pipe>(o_p), ar.dp<double>(o_f), ar.dp<double>(o_b), ar.dp<double>(o_sf),
      ar.dp<double>(o_sb), ar.dp<double>(o_fe), ar.dp<double>(o_be), ar.dp<double>(o_ts),
      ar.dp<double>(o_te), ar.dp<double>(o_busy), ar.dp<int>(o_peak));
  HPKQ_CUDA(cudaGetLastError());
  HPKQ_CUDA(cudaEventRecord(cx.ev1, cx.stream));
  HPKQ_CUDA(cudaMemcpyAsync(ar.h + o_busy, ar.d + o_busy, out_end - o_busy,
                            cudaMemcpyDeviceToHost, cx.stream));
  HPKQ_CUDA(cudaMemcpyAsync(ar.h + o_p, ar.d + o_p, sizeof(Pipe) * n, cudaMemcpyDeviceToHost,
                            cx.stream));
  HPKQ_CUDA(cudaStreamSynchronize(cx.stream));
  float ms = 0;
  HPKQ_CUDA(cudaEventElapsedTime(&ms, cx.ev0, cx.ev1));
  hpk_timing_bridge::add_pipeline(ms, (long long)in_end,
                                  (long long)(out_end - o_busy + sizeof(Pipe) * n));
  std::memcpy(hp.data(), ar.h + o_p, sizeof(Pipe) * n);
  for (int k = 0; k < n; ++k) {
    hpk_pipeline& out = pipes[k];
    if (!hp[k].ok) {
      hpkp_fail("invariant violated: 1F1B schedule is deadlock-free [progressed]");
      return 5;
    }
    out.makespan = hp[k].makespan;
    const int P = hp[k].P, K = hp[k].K;
    std::memcpy(out.busy, ar.h + o_busy + sizeof(double) * hp[k].stage_off, sizeof(double) * P);
    std::memcpy(out.peak_in_flight, ar.h + o_peak + sizeof(int) * hp[k].stage_off,
                sizeof(int) * P);
    if (out.task_start)
      std::memcpy(out.task_start, ar.h + o_ts + sizeof(double) * hp[k].task_off,
                  sizeof(double) * P * 2 * K);
    if (out.task_end)
      std::memcpy(out.task_end, ar.h + o_te + sizeof(double) * hp[k].task_off,
                  sizeof(double) * P * 2 * K);
  }
  return 0;
}
