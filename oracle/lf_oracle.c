/*
 * lf_oracle.c -- CPU restatement of the reference's execution of the five
 * BASELINE workloads.  TEST INFRASTRUCTURE ONLY: imported by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg as the checker /
 * CPU baseline; the product (paper_1503_07659_b200) never links or calls it.
 *
 * Semantics followed (file:line under /root/reference/pkg/src/loopforge):
 *   - interp.py:323-400 `interpret`: statements in schedule order, parallel
 *     inames as outermost loops (385-399); every BinOp rounds at its own
 *     dtype (169-187, numpy scalar ops); stores convert to the target dtype
 *     (376-378); literals take the width of their arithmetic context
 *     (140-145), so `s = 0` stores +0.0.
 *   - expr.py:243-255: + and * are left associative, so
 *     `s + a*b + c*d` is ((s + a*b) + c*d).
 *   - fortran.py:560-563, 638-658: subscripts shifted to 0-based, arrays
 *     column major (strides 1, n0, n0*n1, ...).
 *   - codegen.py:767 emit(...,"c") renders the same arithmetic; the
 *     reference compiles it with `cc -std=c99 -O1` (tests/c_oracle.py:96),
 *     which never contracts a*b+c into an FMA; build this file the same way.
 * Differences from the emitted C: 64-bit indices (the emitted C's `int`
 * offsets overflow past 2^31 elements, SURVEY.md §7 hard part 2).
 *
 * Pinned against the reference itself: tests/test_oracle.py compares every
 * function here with interpret() goldens (tests/golden/, made by
 * tests/golden/make_golden.py) and, when oracle/_ref is built, with the
 * reference's own emitted C on larger inputs.
 */
#include <stddef.h>
#include <stdint.h>

/* fill: out(i) = a          (fixtures.py fill_source; test_fortran.py:13-27) */
void lfo_fill_f64(double *out, double a, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = a;
}
void lfo_fill_f32(float *out, float a, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = a;
}

/* axpy: y(i) = y(i) + alpha*x(i) */
void lfo_axpy_f64(double *y, const double *x, double alpha, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = y[i] + alpha * x[i];
}
void lfo_axpy_f32(float *y, const float *x, float alpha, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = y[i] + alpha * x[i];
}

/* matvec: s = 0; s = s + a(i,j)*x(j) for j ascending; y(i) = s
 * rows [i0, i1) only, so callers can sample                 (Appendix B) */
void lfo_matvec_f64(double *y, const double *a, const double *x, int64_t n,
                    int64_t i0, int64_t i1) {
  for (int64_t i = i0; i < i1; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) s = s + a[i + n * j] * x[j];
    y[i] = s;
  }
}

/* semlap, n points per direction, elements [e0, e1)        (Appendix A) */
void lfo_semlap_f64(double *w, const double *u, const double *d,
                    const double *g, int64_t n, int64_t e0, int64_t e1) {
  const int64_t np = n * n * n;
  double wr[16 * 16 * 16], ws[16 * 16 * 16], wt[16 * 16 * 16];
  if (n < 1 || n > 16) return;
  for (int64_t e = e0; e < e1; ++e) {
    const double *ue = u + np * e;
    const double *ge = g + 6 * np * e;
    double *we = w + np * e;
    for (int64_t k = 0; k < n; ++k)
      for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) {
          double ur = 0.0, us = 0.0, ut = 0.0;
          for (int64_t l = 0; l < n; ++l) {
            ur = ur + d[i + n * l] * ue[l + n * j + n * n * k];
            us = us + d[j + n * l] * ue[i + n * l + n * n * k];
            ut = ut + d[k + n * l] * ue[i + n * j + n * n * l];
          }
          const double *gp = ge + 6 * (i + n * j + n * n * k);
          const int64_t p = i + n * j + n * n * k;
          wr[p] = gp[0] * ur + gp[1] * us + gp[2] * ut;
          ws[p] = gp[1] * ur + gp[3] * us + gp[4] * ut;
          wt[p] = gp[2] * ur + gp[4] * us + gp[5] * ut;
        }
    for (int64_t k = 0; k < n; ++k)
      for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) {
          double s = 0.0;
          for (int64_t l = 0; l < n; ++l)
            s = s + d[l + n * i] * wr[l + n * j + n * n * k] +
                d[l + n * j] * ws[i + n * l + n * n * k] +
                d[l + n * k] * wt[i + n * j + n * n * l];
          we[i + n * j + n * n * k] = s;
        }
  }
}

/* gemm (the paper's DGEMM, test_fortran.py:72-103):
 *   c(i,j) = c(i,j) + alpha*b(k,j)*a(i,k), k ascending
 * columns [j0, j1) of c only, so callers can sample.                      */
void lfo_sgemm_f32(float alpha, const float *a, const float *b, float *c,
                   int64_t l, int64_t m, int64_t n, int64_t j0, int64_t j1) {
  (void)n;
  for (int64_t j = j0; j < j1; ++j)
    for (int64_t k = 0; k < l; ++k) {
      const float ab = alpha * b[k + l * j];
      for (int64_t i = 0; i < m; ++i) c[i + m * j] = c[i + m * j] + ab * a[i + m * k];
    }
}
void lfo_dgemm_f64(double alpha, const double *a, const double *b, double *c,
                   int64_t l, int64_t m, int64_t n, int64_t j0, int64_t j1) {
  (void)n;
  for (int64_t j = j0; j < j1; ++j)
    for (int64_t k = 0; k < l; ++k) {
      const double ab = alpha * b[k + l * j];
      for (int64_t i = 0; i < m; ++i) c[i + m * j] = c[i + m * j] + ab * a[i + m * k];
    }
}

/* sum of squares in ascending index order (the SEM verification norm) */
double lfo_sumsq_f64(const double *w, int64_t n) {
  double s = 0.0;
  for (int64_t q = 0; q < n; ++q) s = s + w[q] * w[q];
  return s;
}

/* SEM direct-stiffness summation (gather-scatter, Q Q^T) on a structured
 * box of Ex x Ey x Ez elements of n points per direction (SURVEY.md §8(f)
 * row 4 -- not in the reference, whose operator is element-local; this is
 * the oracle of paper_1503_07659_b200/csrc/dssum.cu, same order of
 * operations).  Element e = ex + Ex (ey + Ey ez), local node (i, j, k) at
 * w[i + n j + n^2 k + n^3 e] (the semlap layout); global node
 * (X, Y, Z) = (ex p + i, ey p + j, ez p + k), p = n - 1.  A node on an
 * element boundary has 2, 4 or 8 local copies; their sum is formed left
 * to right in ascending element order and written back to every copy.
 * Nodes with zlo <= Z <= zhi only; mode 0 sum + write back, 1 sum into
 * plane_out[X + (Ex p + 1) Y] (partial of a rank's top interface), 2 start
 * from plane_in, add the copies, write back and to plane_out (the upper
 * rank of an interface), 3 write plane_in to the copies. */
static int64_t lfo_cands(int64_t X, int64_t p, int64_t E, int64_t *el,
                         int64_t *loc) {
  const int64_t q = X / p, r = X % p;
  if (r == 0 && q > 0 && q < E) {
    el[0] = q - 1, loc[0] = p;
    el[1] = q, loc[1] = 0;
    return 2;
  }
  el[0] = q < E ? q : E - 1;
  loc[0] = X - el[0] * p;
  return 1;
}

void lfo_dssum_f64(double *w, int64_t n, int64_t Ex, int64_t Ey, int64_t Ez,
                   int64_t zlo, int64_t zhi, int64_t mode,
                   const double *plane_in, double *plane_out) {
  const int64_t p = n - 1, GX = Ex * p + 1, GY = Ey * p + 1;
  const int64_t n3 = n * n * n;
  for (int64_t Z = zlo; Z <= zhi; ++Z)
    for (int64_t Y = 0; Y < GY; ++Y)
      for (int64_t X = 0; X < GX; ++X) {
        if (mode == 0 && X % p && Y % p && Z % p) continue;  /* unique */
        int64_t ex[2], ey[2], ez[2], li[2], lj[2], lk[2];
        const int64_t nx = lfo_cands(X, p, Ex, ex, li);
        const int64_t ny = lfo_cands(Y, p, Ey, ey, lj);
        const int64_t nz = lfo_cands(Z, p, Ez, ez, lk);
        int64_t off[8];
        int64_t c = 0;
        for (int64_t a = 0; a < nz; ++a)      /* ascending element index */
          for (int64_t b = 0; b < ny; ++b)
            for (int64_t f = 0; f < nx; ++f)
              off[c++] = li[f] + n * lj[b] + n * n * lk[a] +
                         n3 * (ex[f] + Ex * (ey[b] + Ey * ez[a]));
        const int64_t pl = X + GX * Y;
        double s;
        int64_t q0 = 0;
        if (mode == 2 || mode == 3) {
          s = plane_in[pl];
        } else {
          s = w[off[0]];
          q0 = 1;
        }
        if (mode != 3)
          for (int64_t q = q0; q < c; ++q) s = s + w[off[q]];
        if (mode == 1 || mode == 2) plane_out[pl] = s;
        if (mode != 1)
          for (int64_t q = 0; q < c; ++q) w[off[q]] = s;
      }
}
