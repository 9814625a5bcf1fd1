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
