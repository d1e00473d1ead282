#include <cstdio>
#include <cuda_runtime.h>
struct PView { const double* p; const double* m; const double* f; const double* R; const double* RM; int n, exact_mem; double min_mem, mb_abs, md_abs; };
enum : int { DEC_PASS = 0, DEC_PRUNE = 1, DEC_EXACT = 2 };
__device__ __forceinline__ int decide(const PView& P, double A, double D, int next, double cut) {
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
__global__ void k(const double* rm, double A, double D, double cut, double mb, int* out) {
  __shared__ double sRM[8];
  if (threadIdx.x < 8) sRM[threadIdx.x] = rm[threadIdx.x];
  __syncwarp();
  PView P; P.RM = sRM; P.mb_abs = mb; P.md_abs = 0.0; P.exact_mem = 1;
  int l = 0;
  if ((threadIdx.x & 31) == 3) l = decide(P, A, D, 2, cut);
  out[threadIdx.x] = l;
}
int main() {
  double h[8] = {0, 0, 5280000000000.0, 0, 0, 0, 0, 0};
  double* d; int* o; int ho[32];
  cudaMalloc(&d, 64); cudaMalloc(&o, 128);
  cudaMemcpy(d, h, 64, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(d, 95.969230769230762, 1304960000000.0, 52.96551724137931, 2.46e-11, o);
  cudaMemcpy(ho, o, 128, cudaMemcpyDeviceToHost);
  printf("decide on lane 3 -> %d (expect 0 PASS)\n", ho[3]);
  return 0;
}
