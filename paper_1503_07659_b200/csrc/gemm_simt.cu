// sgemm, bit-exact path (BASELINE config 5, exact mode).
//
// Reference arithmetic (the paper's DGEMM kernel in real*4,
// /root/reference/pkg/tests/test_fortran.py:72-103; interp.py / emitted C):
//   c(i,j) = c(i,j) + alpha*b(k,j)*a(i,k)   for k ascending
// parsed left-associatively (expr.py:243-255): c + ((alpha*b)*a), every
// operation rounded to f32 separately.  Column major a(m,l) at a[i + m k],
// b(l,n) at b[k + l j], c(m,n) at c[i + m j].
//
// This kernel keeps that exact chain per output element on the FP32 CUDA
// cores (FMUL + FADD, never FFMA): 128x128 CTA tiles, 8x8 register
// micro-tiles, 16-deep k slabs double buffered through registers.  alpha*b is
// formed once per (k,j) while staging B -- the same rounded product every
// (i) uses.  The tensor-core path (gemm_sm100.cu) is the fast mode.
#include "lfb_common.cuh"

namespace lfb {

constexpr int GS_BM = 128, GS_BN = 128, GS_BK = 16, GS_THREADS = 256;

__global__ void __launch_bounds__(GS_THREADS)
    sgemm_exact_kernel(float alpha, const float *__restrict__ a,
                       const float *__restrict__ b, float *__restrict__ c,
                       int l, int m, int n) {
  __shared__ float As[2][GS_BK][GS_BM];
  __shared__ float Bs[2][GS_BK][GS_BN];  // alpha*b(k,j)

  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // 16 x 16 threads, 8x8 each
  const int i0 = blockIdx.x * GS_BM, j0 = blockIdx.y * GS_BN;

  float acc[8][8];
#pragma unroll
  for (int ii = 0; ii < 8; ++ii)
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int gi = i0 + ty * 8 + ii, gj = j0 + tx * 8 + jj;
      acc[ii][jj] = (gi < m && gj < n) ? c[gi + (int64_t)m * gj] : 0.f;
    }

  // loader mapping: A slab 128(i) x 16(k): thread -> (i = tid % 128, k pair)
  //                 B slab 16(k) x 128(j): thread -> (k = tid % 16, j group)
  float ra[8], rb[8];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int ii = tid % GS_BM, kk = (tid / GS_BM) * 8 + q;
      const int gi = i0 + ii, gk = k0 + kk;
      ra[q] = (gi < m && gk < l) ? __ldg(a + gi + (int64_t)m * gk) : 0.f;
      const int kb = tid % GS_BK, jb = (tid / GS_BK) * 8 + q;
      const int gkb = k0 + kb, gj = j0 + jb;
      rb[q] = (gkb < l && gj < n) ? __ldg(b + gkb + (int64_t)l * gj) : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      As[buf][(tid / GS_BM) * 8 + q][tid % GS_BM] = ra[q];
      Bs[buf][tid % GS_BK][(tid / GS_BK) * 8 + q] = fmul(alpha, rb[q]);
    }
  };

  const int nk = (l + GS_BK - 1) / GS_BK;
  load(0);
  store(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load((t + 1) * GS_BK);
    const int kmax = min(GS_BK, l - t * GS_BK);
    for (int kk = 0; kk < kmax; ++kk) {
      float av[8], bv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        av[q] = As[buf][kk][ty * 8 + q];
        bv[q] = Bs[buf][kk][tx * 8 + q];
      }
#pragma unroll
      for (int ii = 0; ii < 8; ++ii)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          acc[ii][jj] = fadd(acc[ii][jj], fmul(bv[jj], av[ii]));
    }
    if (t + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }

#pragma unroll
  for (int ii = 0; ii < 8; ++ii)
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int gi = i0 + ty * 8 + ii, gj = j0 + tx * 8 + jj;
      if (gi < m && gj < n) c[gi + (int64_t)m * gj] = acc[ii][jj];
    }
}

int sgemm_exact(float alpha, const float *a, const float *b, float *c, int l,
                int m, int n, cudaStream_t s) {
  dim3 grid((m + GS_BM - 1) / GS_BM, (n + GS_BN - 1) / GS_BN);
  if (grid.y > 65535)
    return fail(LFB_ERR_UNSUPPORTED, "sgemm: n=%d too large for the grid", n);
  sgemm_exact_kernel<<<grid, GS_THREADS, 0, s>>>(alpha, a, b, c, l, m, n);
  return check_launch("lfb_sgemm_f32(exact)");
}

}  // namespace lfb
