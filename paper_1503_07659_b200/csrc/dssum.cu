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
// edge / corner has 2 / 4 / 8 local copies.  One thread per shared global
// node of the requested Z range: the copies are summed left to right in
// ascending element order -- a fixed order, so the result is deterministic
// and bitwise the oracle's (oracle/lf_oracle.c lfo_dssum_f64) -- and the
// sum is written back to every copy.  Interior nodes (one copy) are not
// touched.  CTAs walk rows of global nodes (see dssum_kernel).
//
// Multi-GPU (paper_1503_07659_b200/assembly.py): ranks own slabs of element
// layers in z; an interface plane's sum must be the single-GPU sum, so the
// lower rank forms the partial over its copies (mode 1), the upper rank
// continues that chain with its own copies (mode 2) and returns the total,
// which the lower rank writes back (mode 3) -- NCCL point-to-point between
// neighbours, bitwise the single-GPU result.
#include "lfb_common.cuh"

namespace lfb {

// the elements along one direction holding global coordinate X, and the
// local index in each: two (lower first) on an interior element plane, else
// one (then slot 1 repeats slot 0)
__device__ __forceinline__ int cands(int64_t X, int p, int E, int &el0,
                                     int &loc0, int &el1, int &loc1) {
  const int64_t q = X / p, r = X - q * p;
  if (r == 0 && q > 0 && q < E) {
    el0 = (int)q - 1, loc0 = p, el1 = (int)q, loc1 = 0;
    return 2;
  }
  el0 = q < E ? (int)q : E - 1;
  loc0 = (int)(X - (int64_t)el0 * p);
  el1 = el0, loc1 = loc0;
  return 1;
}

// one CTA per row (Y, Z) of global nodes, threads over X (uniform per
// CTA, so no divergence between "full" and "sparse" rows and no 64-bit
// division per node).  A row with Y or Z on an element plane is full: every
// node may be shared, consecutive X are consecutive i of one element
// (coalesced).  Otherwise only the nodes on x-element planes are shared
// (X = ex p, two copies): a sparse row has Ex + 1 candidates.
template <int MODE>
__device__ __forceinline__ void dssum_node(double *__restrict__ w, int n,
                                           int p, int Ex, int Ey, int Ez,
                                           int64_t X, int64_t Y, int64_t Z,
                                           int64_t pl,
                                           const double *__restrict__ pin,
                                           double *__restrict__ pout) {
  const int64_t n2 = (int64_t)n * n, n3 = n2 * n;
  int ex[2], ey[2], ez[2], li[2], lj[2], lk[2];
  const int nx = cands(X, p, Ex, ex[0], li[0], ex[1], li[1]);
  const int ny = cands(Y, p, Ey, ey[0], lj[0], ey[1], lj[1]);
  const int nz = cands(Z, p, Ez, ez[0], lk[0], ez[1], lk[1]);
  if (MODE == 0 && nx * ny * nz == 1) return;  // one copy: nothing to do
  // copy (a, b, f) at fixed slot 4a + 2b + f: lexicographic = ascending
  // element index; fully unrolled and predicated (no local-memory array)
  int64_t off[8];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int f = 0; f < 2; ++f)
        off[4 * a + 2 * b + f] =
            li[f] + n * lj[b] + n2 * lk[a] +
            n3 * (ex[f] + (int64_t)Ex * (ey[b] + (int64_t)Ey * ez[a]));
  double s = 0.0;
  bool first = !(MODE == 2 || MODE == 3);
  if (!first) s = pin[pl];
  if (MODE != 3) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if ((q >> 2) < nz && ((q >> 1) & 1) < ny && (q & 1) < nx) {
        const double v = w[off[q]];
        s = first ? v : dadd(s, v);
        first = false;
      }
    }
  }
  if (MODE == 1 || MODE == 2) pout[pl] = s;
  if (MODE != 1) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if ((q >> 2) < nz && ((q >> 1) & 1) < ny && (q & 1) < nx) w[off[q]] = s;
  }
}

template <int MODE>
__global__ void __launch_bounds__(256)
    dssum_kernel(double *__restrict__ w, int n, int Ex, int Ey, int Ez,
                 int zlo, int zhi, const double *__restrict__ plane_in,
                 double *__restrict__ plane_out) {
  const int p = n - 1;
  const int64_t GX = (int64_t)Ex * p + 1, GY = (int64_t)Ey * p + 1;
  const int64_t rows = GY * (int64_t)(zhi - zlo + 1);
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t Y = row % GY;
    const int64_t Z = zlo + row / GY;
    const bool full = MODE != 0 || Y % p == 0 || Z % p == 0;
    if (full) {
      for (int64_t X = threadIdx.x; X < GX; X += blockDim.x)
        dssum_node<MODE>(w, n, p, Ex, Ey, Ez, X, Y, Z, X + GX * Y, plane_in,
                         plane_out);
    } else {
      for (int64_t q = threadIdx.x + 1; q < Ex; q += blockDim.x)
        dssum_node<MODE>(w, n, p, Ex, Ey, Ez, q * p, Y, Z, q * p + GX * Y,
                         plane_in, plane_out);
    }
  }
}

// {{{ mode 0, order as a template parameter (the default)
//
// The generic kernel above is instruction-bound, not memory-bound: ncu
// (profiles/r02_dssum_v0.md) shows DRAM traffic at the sector floor (every
// 64-byte row segment of every element holds a shared node, so all of w is
// read and written once) but 463 M instructions for a 64^3 box -- three
// 64-bit divisions by the run-time p and eight 64-bit offsets per node.
// Here p is a compile-time constant, the y / z candidates and their offsets
// are computed once per row (uniform over the warp), and one *warp* walks a
// row (lanes over X in a full row, over the x-element planes in a sparse
// one), so sparse rows no longer idle 3/4 of a CTA.  Same nodes, same
// copies, same left-to-right sum: bitwise the generic kernel.
template <int N>
__device__ __forceinline__ int cands_t(int X, int E, int &el0, int &loc0,
                                       int &el1, int &loc1) {
  constexpr int P = N - 1;
  const int q = X / P, r = X - q * P;
  if (r == 0 && q > 0 && q < E) {
    el0 = q - 1, loc0 = P, el1 = q, loc1 = 0;
    return 2;
  }
  el0 = q < E ? q : E - 1;
  loc0 = X - el0 * P;
  el1 = el0, loc1 = loc0;
  return 1;
}

template <int N>
__global__ void __launch_bounds__(256)
    dssum_rows_kernel(double *__restrict__ w, int Ex, int Ey, int Ez,
                      int zlo, int zhi) {
  constexpr int P = N - 1;
  constexpr int64_t N2 = (int64_t)N * N, N3 = N2 * N;
  const int GX = Ex * P + 1, GY = Ey * P + 1;
  const int64_t rows = (int64_t)GY * (zhi - zlo + 1);
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t EX3 = N3 * Ex;
  for (int64_t row = warp0; row < rows; row += nwarps) {
    const int Y = (int)(row % GY);
    const int Z = zlo + (int)(row / GY);
    int ey[2], lj[2], ez[2], lk[2];
    const int ny = cands_t<N>(Y, Ey, ey[0], lj[0], ey[1], lj[1]);
    const int nz = cands_t<N>(Z, Ez, ez[0], lk[0], ez[1], lk[1]);
    // the (y, z) copies without the x part: slot 2a + b
    double *wyz[4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
        wyz[2 * a + b] = w + (N * lj[b] + N2 * lk[a] +
                              EX3 * (ey[b] + (int64_t)Ey * ez[a]));
    if (ny * nz > 1 || Y % P == 0 || Z % P == 0) {
      // full row: every node may be shared; lanes over X (consecutive i)
      for (int X = lane; X < GX; X += 32) {
        int ex[2], li[2];
        const int nx = cands_t<N>(X, Ex, ex[0], li[0], ex[1], li[1]);
        if (nx * ny * nz == 1) continue;
        double *cp[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) cp[q] = wyz[q >> 1] + li[q & 1] + N3 * ex[q & 1];
        double s = 0.0;
        bool first = true;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if ((q >> 2) < nz && ((q >> 1) & 1) < ny && (q & 1) < nx) {
            const double v = *cp[q];
            s = first ? v : dadd(s, v);
            first = false;
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if ((q >> 2) < nz && ((q >> 1) & 1) < ny && (q & 1) < nx) *cp[q] = s;
      }
    } else {
      // sparse row: only the x-element planes X = q P, 1 <= q < Ex, two
      // copies (element q - 1 at i = P, element q at i = 0)
      for (int q = 1 + lane; q < Ex; q += 32) {
        double *c1 = wyz[0] + N3 * q;
        double *c0 = c1 - (N3 - P);
        const double s = dadd(*c0, *c1);
        *c0 = s;
        *c1 = s;
      }
    }
  }
}

template <int N>
static void dssum_rows_launch(double *w, int ex, int ey, int ez, int zlo,
                              int zhi, cudaStream_t s) {
  const int64_t rows = ((int64_t)ey * (N - 1) + 1) * (zhi - zlo + 1);
  int sms = sm_count(nullptr);
  if (sms <= 0) sms = 148;
  static int per_sm = [] {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, dssum_rows_kernel<N>,
                                                  256, 0);
    return b > 0 ? b : 1;
  }();
  int64_t blocks = (rows + 7) / 8;  // 8 warps per CTA, one row each
  if (blocks > (int64_t)sms * per_sm)  // one wave, every CTA resident
    blocks = (int64_t)sms * per_sm;
  if (blocks < 1) blocks = 1;
  dssum_rows_kernel<N><<<(int)blocks, 256, 0, s>>>(w, ex, ey, ez, zlo, zhi);
}

static bool dssum_rows(int n, double *w, int ex, int ey, int ez, int zlo,
                       int zhi, cudaStream_t s) {
  switch (n) {
#define C(NN) \
  case NN: dssum_rows_launch<NN>(w, ex, ey, ez, zlo, zhi, s); return true;
    C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9) C(10) C(11) C(12) C(13) C(14)
    C(15) C(16)
#undef C
    default: return false;
  }
}

// }}}

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
  const int variant = mode >> 4;  // bits 4+: kernel variant (tuning)
  mode &= 15;
  if (mode > 3 || variant < 0)
    return fail(LFB_ERR_ARG, "lfb_dssum_f64: mode %d (0 local, 1 partial, "
                             "2 continue, 3 write)", mode);
  if (mode != 0 && ((zlo % (n - 1)) || zlo != zhi))
    return fail(LFB_ERR_ARG, "lfb_dssum_f64: modes 1-3 take one element "
                             "plane (zlo == zhi, a multiple of n-1)");
  if (!w || ((mode == 2 || mode == 3) && !plane_in) ||
      ((mode == 1 || mode == 2) && !plane_out))
    return fail(LFB_ERR_ARG, "lfb_dssum_f64: null buffer");
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0 && variant == 0 &&
      (int64_t)ex * (n - 1) + 1 < (int64_t(1) << 31) &&
      dssum_rows(n, w, ex, ey, ez, zlo, zhi, s))
    return check_launch("lfb_dssum_f64");
  const int64_t rows = ((int64_t)ey * (n - 1) + 1) * (zhi - zlo + 1);
  int sms = sm_count(nullptr);
  if (sms <= 0) sms = 148;
  int64_t blocks = rows;
  if (blocks > (int64_t)sms * 32) blocks = (int64_t)sms * 32;
  if (blocks < 1) blocks = 1;
  switch (mode) {
    case 0: dssum_kernel<0><<<(int)blocks, 256, 0, s>>>(w, n, ex, ey, ez, zlo, zhi, plane_in, plane_out); break;
    case 1: dssum_kernel<1><<<(int)blocks, 256, 0, s>>>(w, n, ex, ey, ez, zlo, zhi, plane_in, plane_out); break;
    case 2: dssum_kernel<2><<<(int)blocks, 256, 0, s>>>(w, n, ex, ey, ez, zlo, zhi, plane_in, plane_out); break;
    default: dssum_kernel<3><<<(int)blocks, 256, 0, s>>>(w, n, ex, ey, ez, zlo, zhi, plane_in, plane_out); break;
  }
  return check_launch("lfb_dssum_f64");
}
