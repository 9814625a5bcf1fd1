// SEM direct-stiffness summation -- the gather-scatter Q Q^T that assembles
// element-local SEM vectors.  Not in the reference
// (its Appendix-A operator is element-local, interp.py:385-399 runs the
// elements as independent outer loops); this completes the matrix-free
// operator of an SEM solver: w <- Q Q^T (semlap(u)).
//
// Mesh: a structured box of Ex x Ey x Ez hexahedral elements, n points per
// direction (p = n - 1), element e = ex + Ex (ey + Ey ez), local node
// (i, j, k) at w[i + n j + n^2 k + n^3 e] (the semlap layout), global node
// (X, Y, Z) = (ex p + i, ey p + j, ez p + k).  A node on an element face /
// edge / corner has 2 / 4 / 8 local copies.  One thread per global node in
// the requested Z range (grid-stride, 64-bit): the copies are summed left to
// right in ascending element order -- a fixed order, so the result is
// deterministic and bitwise the oracle's (oracle/lf_oracle.c
// lfo_dssum_f64) -- and the sum is written back to every copy.  Interior
// nodes (one copy) are not touched.  Warps walk X fastest: consecutive lanes
// hit consecutive i of the same element, so every copy access is coalesced.
//
// Multi-GPU (paper_1503_07659_b200/assembly.py): ranks own slabs of element
// layers in z; an interface plane's sum must be the single-GPU sum, so the
// lower rank forms the partial over its copies (mode 1), the upper rank
// continues that chain with its own copies (mode 2) and returns the total,
// which the lower rank writes back (mode 3) -- NCCL point-to-point between
// neighbours, bitwise the single-GPU result.
#include "lfb_common.cuh"

namespace lfb {

__device__ __forceinline__ int cands(int64_t X, int p, int E, int *el,
                                     int *loc) {
  const int64_t q = X / p, r = X - q * p;
  if (r == 0 && q > 0 && q < E) {
    el[0] = (int)q - 1, loc[0] = p;
    el[1] = (int)q, loc[1] = 0;
    return 2;
  }
  el[0] = q < E ? (int)q : E - 1;
  loc[0] = (int)(X - (int64_t)el[0] * p);
  return 1;
}

template <int MODE>
__global__ void __launch_bounds__(256)
    dssum_kernel(double *__restrict__ w, int n, int Ex, int Ey, int Ez,
                 int zlo, int zhi, const double *__restrict__ plane_in,
                 double *__restrict__ plane_out) {
  const int p = n - 1;
  const int64_t GX = (int64_t)Ex * p + 1, GY = (int64_t)Ey * p + 1;
  const int64_t total = GX * GY * (int64_t)(zhi - zlo + 1);
  const int64_t n2 = (int64_t)n * n, n3 = n2 * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t X = t % GX;
    const int64_t r = t / GX;
    const int64_t Y = r % GY;
    const int64_t Z = zlo + r / GY;
    if (MODE == 0 && (X % p) && (Y % p) && (Z % p)) continue;  // unique
    int ex[2], ey[2], ez[2], li[2], lj[2], lk[2];
    const int nx = cands(X, p, Ex, ex, li);
    const int ny = cands(Y, p, Ey, ey, lj);
    const int nz = cands(Z, p, Ez, ez, lk);
    int64_t off[8];
    int c = 0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int f = 0; f < 2; ++f)
          if (a < nz && b < ny && f < nx)
            off[c++] = li[f] + n * lj[b] + n2 * lk[a] +
                       n3 * (ex[f] + (int64_t)Ex * (ey[b] +
                                                    (int64_t)Ey * ez[a]));
    const int64_t pl = X + GX * Y;
    double s;
    int q0 = 0;
    if (MODE == 2 || MODE == 3) {
      s = plane_in[pl];
    } else {
      s = w[off[0]];
      q0 = 1;
    }
    if (MODE != 3)
      for (int q = q0; q < c; ++q) s = dadd(s, w[off[q]]);
    if (MODE == 1 || MODE == 2) plane_out[pl] = s;
    if (MODE != 1)
      for (int q = 0; q < c; ++q) w[off[q]] = s;
  }
}

}  // namespace lfb

extern "C" int lfb_dssum_f64(double *w, int n, int ex, int ey, int ez,
                             int zlo, int zhi, int mode,
                             const double *plane_in, double *plane_out,
                             lfb_stream stream) {
  using namespace lfb;
  if (n < 2 || ex < 1 || ey < 1 || ez < 1)
    return fail(LFB_ERR_ARG, "lfb_dssum_f64: need n >= 2 and >= 1 element "
                             "per direction (n=%d, %d x %d x %d)",
                n, ex, ey, ez);
  if (zlo < 0 || zhi > ez * (n - 1) || zlo > zhi)
    return fail(LFB_ERR_ARG, "lfb_dssum_f64: Z range [%d, %d] outside "
                             "[0, %d]", zlo, zhi, ez * (n - 1));
  if (mode < 0 || mode > 3)
    return fail(LFB_ERR_ARG, "lfb_dssum_f64: mode %d (0 local, 1 partial, "
                             "2 continue, 3 write)", mode);
  if (mode != 0 && ((zlo % (n - 1)) || zlo != zhi))
    return fail(LFB_ERR_ARG, "lfb_dssum_f64: modes 1-3 take one element "
                             "plane (zlo == zhi, a multiple of n-1)");
  if (!w || ((mode == 2 || mode == 3) && !plane_in) ||
      ((mode == 1 || mode == 2) && !plane_out))
    return fail(LFB_ERR_ARG, "lfb_dssum_f64: null buffer");
  const int64_t total = ((int64_t)ex * (n - 1) + 1) *
                        ((int64_t)ey * (n - 1) + 1) * (zhi - zlo + 1);
  int sms = sm_count(nullptr);
  if (sms <= 0) sms = 148;
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  if (blocks < 1) blocks = 1;
  cudaStream_t s = (cudaStream_t)stream;
  switch (mode) {
    case 0: dssum_kernel<0><<<(int)blocks, 256, 0, s>>>(w, n, ex, ey, ez, zlo, zhi, plane_in, plane_out); break;
    case 1: dssum_kernel<1><<<(int)blocks, 256, 0, s>>>(w, n, ex, ey, ez, zlo, zhi, plane_in, plane_out); break;
    case 2: dssum_kernel<2><<<(int)blocks, 256, 0, s>>>(w, n, ex, ey, ez, zlo, zhi, plane_in, plane_out); break;
    default: dssum_kernel<3><<<(int)blocks, 256, 0, s>>>(w, n, ex, ey, ez, zlo, zhi, plane_in, plane_out); break;
  }
  return check_launch("lfb_dssum_f64");
}
