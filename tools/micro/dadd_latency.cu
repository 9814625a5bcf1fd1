// Dependent-latency probe: one warp, a chain of N dependent DADDs (and
// DFMAs), timed with clock64 -> cycles per dependent op on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double *out, long long *cyc, double x, int n) {
  double s = x, m = 1.0000001;
  long long t0 = clock64();
  for (int q = 0; q < n; ++q) {
#pragma unroll
    for (int u = 0; u < 16; ++u) s = __dadd_rn(s, m);
  }
  long long t1 = clock64();
  double f = x;
  for (int q = 0; q < n; ++q) {
#pragma unroll
    for (int u = 0; u < 16; ++u) f = __fma_rn(f, m, 1e-9);
  }
  long long t2 = clock64();
  double p = x;
  for (int q = 0; q < n; ++q) {
#pragma unroll
    for (int u = 0; u < 16; ++u) p = __dmul_rn(p, m);
  }
  long long t3 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
    out[0] = s + f + p;
  }
}

int main() {
  double *o; long long *c, h[3];
  cudaMalloc(&o, 8); cudaMalloc(&c, 24);
  const int n = 4096;
  chain<<<1, 32>>>(o, c, 1.0, 16);
  chain<<<1, 32>>>(o, c, 1.0, n);
  cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("cycles per dependent DADD %.2f  DFMA %.2f  DMUL %.2f\n",
         (double)h[0] / (16.0 * n), (double)h[1] / (16.0 * n),
         (double)h[2] / (16.0 * n));
  return 0;
}
