// Energy probe: products per joule of DMUL vs DMMA m8n8k4 used as an outer
// product (one non-zero k: D = a b exactly rounded) on sm_100a, to decide
// whether the bitwise SEM kernels -- power-capped when sustained
// (profiles/r02/sem_clock.jsonl) -- could move their separately rounded
// products to the tensor pipe.  tools only:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 energy_probe.cu
//   ./a.out <kernel 0..3> <seconds>   (run under nvidia-smi sampling)
// kernel 0: DMUL chains, 1: DADD chains, 2: DMMA k=1 (3 of 4 k zero),
// 3: DMMA all four k non-zero.  Prints launches, seconds and products/s
// (DMMA k=1: 64 useful products per instruction per warp).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void dmul_kernel(double *out, int iters) {
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = 1.0 + (threadIdx.x + q) * 1e-7;
  const double a = 1.0 + 1e-13 * blockIdx.x, b = 1.0 - 1e-13;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = __dmul_rn(x[q], (it & 1) ? a : b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += x[q];
  if (s == 1.2345) out[0] = s;
}

__global__ void dadd_kernel(double *out, int iters) {
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = 1.0 + (threadIdx.x + q) * 1e-7;
  const double a = 1e-9 * (1 + blockIdx.x % 7);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = __dadd_rn(x[q], (it & 1) ? a : -a);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += x[q];
  if (s == 1.2345) out[0] = s;
}

template <bool K1>
__global__ void dmma_kernel(double *out, int iters) {
  const int lane = threadIdx.x & 31;
  // A[r][k] at lane (r, k = lane % 4), B[k][c] at lane (k = lane % 4, c):
  // K1 keeps only k = 0 non-zero
  const bool on = !K1 || (lane % 4) == 0;
  const double a = on ? 1.0 + lane * 1e-7 : 0.0;
  const double b = on ? 1.0 - lane * 1e-7 : 0.0;
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

int main(int argc, char **argv) {
  const int kid = argc > 1 ? atoi(argv[1]) : 0;
  const double secs = argc > 2 ? atof(argv[2]) : 2.0;
  double *o;
  cudaMalloc(&o, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * 4, iters = 20000;
  auto launch = [&] {
    switch (kid) {
      case 0: dmul_kernel<<<blocks, threads>>>(o, iters); break;
      case 1: dadd_kernel<<<blocks, threads>>>(o, iters); break;
      case 2: dmma_kernel<true><<<blocks, threads>>>(o, iters); break;
      default: dmma_kernel<false><<<blocks, threads>>>(o, iters); break;
    }
  };
  launch();
  cudaDeviceSynchronize();
  const auto t0 = std::chrono::steady_clock::now();
  long launches = 0;
  double el = 0;
  while (el < secs) {
    for (int r = 0; r < 4; ++r) launch();
    launches += 4;
    cudaDeviceSynchronize();
    el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
             .count();
  }
  const double warps = (double)blocks * threads / 32;
  // useful products (or adds) per launch
  double per = 0;
  if (kid <= 1) per = warps * 32 * 8 * (double)iters;
  else if (kid == 2) per = warps * 64 * 8 * (double)iters;
  else per = warps * 256 * 8 * (double)iters;
  printf("{\"kernel\": %d, \"launches\": %ld, \"seconds\": %.3f, "
         "\"ops_per_s\": %.4e}\n",
         kid, launches, el, per * launches / el);
  return 0;
}
