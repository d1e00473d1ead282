// Regression test for the decide() miscompile seen with nvcc 12.9 (sm_100a):
// evaluates old and new formulations on a grid of cases against host results.
#include <cstdio>
#include <cuda_runtime.h>
struct PView { const double* RM; double mb_abs, md_abs; };
enum : int { DEC_PASS = 0, DEC_PRUNE = 1, DEC_EXACT = 2 };
__host__ __device__ __forceinline__ int decide_old(const PView& P, double A, double D, int next, double cut) {
  int db = DEC_PASS;
  if (cut >= 0) {
    if (A + P.mb_abs < cut) db = DEC_PRUNE;
    else if (A - P.mb_abs >= cut) db = DEC_PASS;
    else db = DEC_EXACT;
  }
  const double rem = P.RM[next];
  int dd;
  if (D - P.md_abs > rem) dd = DEC_PRUNE;
  else if (D + P.md_abs <= rem) dd = DEC_PASS;
  else dd = DEC_EXACT;
  if (db == DEC_PRUNE || dd == DEC_PRUNE) return DEC_PRUNE;
  if (db == DEC_PASS && dd == DEC_PASS) return DEC_PASS;
  return DEC_EXACT;
}
__host__ __device__ __forceinline__ int decide_new(const PView& P, double A, double D, int next, double cut) {
  const double rem = P.RM[next];
  const bool has_cut = cut >= 0;
  const bool b_prune = has_cut && (A + P.mb_abs < cut);
  const bool d_prune = D - P.md_abs > rem;
  if (b_prune || d_prune) return DEC_PRUNE;
  const bool b_pass = !has_cut || (A - P.mb_abs >= cut);
  const bool d_pass = D + P.md_abs <= rem;
  return (b_pass && d_pass) ? DEC_PASS : DEC_EXACT;
}
__global__ void k(const double* rm, const double* in, int n, double mb, double md, int* out) {
  __shared__ double sRM[4];
  if (threadIdx.x < 4) sRM[threadIdx.x] = rm[threadIdx.x];
  __syncthreads();
  PView P; P.RM = sRM; P.mb_abs = mb; P.md_abs = md;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int a = 0, b = 0;
    if ((threadIdx.x & 31) == (i & 31)) {   // owner-lane style divergence
      a = decide_old(P, in[3 * i], in[3 * i + 1], 2, in[3 * i + 2]);
      b = decide_new(P, in[3 * i], in[3 * i + 1], 2, in[3 * i + 2]);
    }
    out[2 * i] = a; out[2 * i + 1] = b;
  }
}
int main() {
  const double rm[4] = {0, 0, 100.0, 0};
  const double As[] = {10, 50, 50 + 1e-12, 90}, Ds[] = {50, 100, 100 + 1e-12, 150}, cuts[] = {-1, 0, 50, 60};
  const double mbs[] = {0.0, 1e-9}, mds[] = {0.0, 1e-9};
  int bad_old = 0, bad_new = 0, total = 0;
  for (double mb : mbs) for (double md : mds) {
    double in[3 * 64]; int n = 0;
    for (double A : As) for (double D : Ds) for (double c : cuts) { in[3*n] = A; in[3*n+1] = D; in[3*n+2] = c; ++n; }
    double *din, *drm; int* dout; int out[2 * 64];
    cudaMalloc(&din, sizeof(in)); cudaMalloc(&drm, 32); cudaMalloc(&dout, sizeof(out));
    cudaMemcpy(din, in, sizeof(in), cudaMemcpyHostToDevice); cudaMemcpy(drm, rm, 32, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(drm, din, n, mb, md, dout);
    cudaMemcpy(out, dout, sizeof(out), cudaMemcpyDeviceToHost);
    PView hp; hp.RM = rm; hp.mb_abs = mb; hp.md_abs = md;
    for (int i = 0; i < n; ++i) {
      const int want = decide_old(hp, in[3*i], in[3*i+1], 2, in[3*i+2]);
      const int want2 = decide_new(hp, in[3*i], in[3*i+1], 2, in[3*i+2]);
      if (want != want2) printf("host mismatch case %d\n", i);
      bad_old += out[2*i] != want; bad_new += out[2*i+1] != want; ++total;
    }
  }
  printf("cases %d: old formulation wrong on %d, new formulation wrong on %d\n", total, bad_old, bad_new);
  return 0;
}
