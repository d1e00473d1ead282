// Latency microbenchmarks on B200 (design calibration for the warp DFS).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, int n) {
  const int lane = threadIdx.x & 31;
  double x = a + lane;
  __shared__ double sm[64];
  sm[lane] = x; sm[lane + 32] = x;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + a;                // DADD chain
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * a;                // DMUL chain
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (i + lane) & 31);  // SHFL.64 chain
  long long t3 = clock64();
  int j = lane;
  for (int i = 0; i < n; ++i) { j = (int)sm[j & 63] & 63; }  // LDS chain
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) {                          // divergent owner block + broadcast
    double v = 0;
    if (lane == (i & 31)) v = x * a + 1.0;
    x = __shfl_sync(0xffffffffu, v, i & 31);
  }
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) { if (lane == 0) sm[i & 63] = x; __syncwarp(); x = sm[(i + 1) & 63]; }
  long long t6 = clock64();
  out[threadIdx.x] = x + j;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}
int main() {
  double* d; long long* c; long long h[6];
  cudaMalloc(&d, 1024); cudaMalloc(&c, 64);
  const int n = 1000;
  k<<<1, 32>>>(d, c, 1.0000001, n);
  k<<<1, 32>>>(d, c, 1.0000001, n);
  cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  const char* names[6] = {"DADD dep", "DMUL dep", "SHFL.64 dep", "LDS dep", "owner-block+shfl", "sts+syncwarp+lds"};
  for (int i = 0; i < 6; ++i) printf("%-20s %.1f cycles/op\n", names[i], (double)h[i] / n);
  return 0;
}
