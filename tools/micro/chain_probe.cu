// One warp: the matvec consumer's inner structure without memory traffic --
// a chain of dependent DADDs over 64 register products, interleaved with the
// LDS + DMUL of the next 64 products (smem data) -- cycles per chained add.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void probe(double *out, long long *cyc, int tiles) {
  __shared__ double t[64 * 32], xv[64];
  for (int q = threadIdx.x; q < 64 * 32; q += 32) t[q] = 1.0 + q * 1e-9;
  for (int q = threadIdx.x; q < 64; q += 32) xv[q] = 0.5 + q * 1e-9;
  __syncwarp();
  const int lane = threadIdx.x;
  double p[64];
#pragma unroll
  for (int jj = 0; jj < 64; ++jj) p[jj] = __dmul_rn(t[jj * 32 + lane], xv[jj]);
  double acc = 0.0;
  long long t0 = clock64();
  for (int q = 0; q < tiles; ++q) {
#pragma unroll
    for (int jj = 0; jj < 64; ++jj) {
      acc = __dadd_rn(acc, p[jj]);
      if (MODE == 1) p[jj] = __dmul_rn(t[jj * 32 + lane], xv[jj]);
    }
    if (MODE == 1) asm volatile("" ::: "memory");
  }
  long long t1 = clock64();
  if (lane == 0) cyc[0] = t1 - t0;
  out[lane] = acc;
}

int main() {
  double *o; long long *c, h;
  cudaMalloc(&o, 256); cudaMalloc(&c, 8);
  const int tiles = 64;
  probe<0><<<1, 32>>>(o, c, 4);
  probe<0><<<1, 32>>>(o, c, tiles);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("chain only:            %.2f cycles per add\n", (double)h / (64.0 * tiles));
  probe<1><<<1, 32>>>(o, c, 4);
  probe<1><<<1, 32>>>(o, c, tiles);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("chain + LDS/DMUL next: %.2f cycles per add\n", (double)h / (64.0 * tiles));
  return 0;
}
