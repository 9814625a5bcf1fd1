// Throughput probe: FP64 DMMA (mma.sync m8n8k4 f64) vs DFMA on sm_100a.
// tools only (not part of the library): nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_kernel(double *out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5 + blockIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = q * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, "
          "{%3}, {%0,%1};"
          : "+d"(c[q][0]), "+d"(c[q][1])
          : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  if (s == 1.2345) out[0] = s;
}

// the dgemm kernel's issue pattern: an 8 x 4 grid of accumulators fed by 8
// A and 4 B fragments (distinct registers, each reused 4 or 8 times)
__global__ void dmma_grid_kernel(double *out, int iters) {
  double fa[8], fb[4];
#pragma unroll
  for (int x = 0; x < 8; ++x) fa[x] = 1.0 + (threadIdx.x + x) * 1e-9;
#pragma unroll
  for (int x = 0; x < 4; ++x) fb[x] = 0.5 + (blockIdx.x + x) * 1e-9;
  double c[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j][0] = c[i][j][1] = (i + j) * 1e-3;
  for (int it = 0; it < iters / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, "
            "{%3}, {%0,%1};"
            : "+d"(c[i][j][0]), "+d"(c[i][j][1])
            : "d"(fa[i]), "d"(fb[j]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[i][j][0] + c[i][j][1];
  if (s == 1.2345) out[0] = s;
}

__global__ void dfma_kernel(double *out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5 + blockIdx.x * 1e-9;
  double c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q] = q * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = __fma_rn(a, c[q], b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q];
  if (s == 1.2345) out[0] = s;
}

int main() {
  double *o;
  cudaMalloc(&o, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps = 4; warps <= 32; warps *= 2) {
    float ms;
    dmma_kernel<<<sms, 32 * warps>>>(o, 16);
    cudaEventRecord(e0);
    dmma_kernel<<<sms, 32 * warps>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * warps * sms;
    printf("DMMA m8n8k4 warps/SM %2d: %.2f TFLOP/s\n", warps,
           flops / (ms * 1e-3) / 1e12);
    if (warps <= 8) {  // 64 accumulators: no more than 8 warps fit
      dmma_grid_kernel<<<sms, 32 * warps>>>(o, 16);
      cudaEventRecord(e0);
      dmma_grid_kernel<<<sms, 32 * warps>>>(o, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (cudaGetLastError() == cudaSuccess)
        printf("DMMA 8x4 grid (dgemm pattern) warps/SM %2d: %.2f TFLOP/s\n",
               warps, flops / (ms * 1e-3) / 1e12);
    }
    dfma_kernel<<<sms, 32 * warps>>>(o, 16);
    cudaEventRecord(e0);
    dfma_kernel<<<sms, 32 * warps>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8.0 * iters * 32 * warps * sms;
    printf("DFMA        warps/SM %2d: %.2f TFLOP/s\n", warps,
           flops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
