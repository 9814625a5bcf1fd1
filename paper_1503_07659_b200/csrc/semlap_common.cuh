// Pieces shared by the two SEM kernels: the fused verification-norm epilogue.
#pragma once

#include <cuda.h>

#include "lfb_common.cuh"

namespace lfb {

// {{{ arithmetic of the two SEM modes
//
// F = false (default): the reference's arithmetic -- every * and + rounded
// separately, left-associative (bitwise the reference's result).
// F = true ("fma" variant 50): each multiply-add fused into one DFMA, same
// association order -- within the north star's 1e-12 fp64 tolerance and
// half the FP64 instructions (the FP64 pipe is the second ceiling, and the
// binding one at high orders).

// acc + a*b
template <bool F>
__device__ __forceinline__ double mac(double acc, double a, double b) {
  if constexpr (F) return __fma_rn(a, b, acc);
  else return dadd(acc, dmul(a, b));
}

// 0 + a*b, the first step of every accumulation chain.  The reference adds
// the product to the literal 0; that addition only changes a -0 product
// into +0, so the bitwise mode does it with two integer instructions
// instead of a DADD (3.6 % of the operator's FP64 instructions at n = 8).
template <bool F>
__device__ __forceinline__ double mac0(double a, double b) {
  const double p = dmul(a, b);
  if constexpr (F) return p;
  const long long bits = __double_as_longlong(p);
  return __longlong_as_double(bits == (long long)0x8000000000000000ULL
                                  ? 0LL : bits);
}

// (x0*y0 + x1*y1) + x2*y2
template <bool F>
__device__ __forceinline__ double comb3(double x0, double y0, double x1,
                                        double y1, double x2, double y2) {
  if constexpr (F) return __fma_rn(x2, y2, __fma_rn(x1, y1, dmul(x0, y0)));
  else return dadd(dadd(dmul(x0, y0), dmul(x1, y1)), dmul(x2, y2));
}

// }}}

// fixed-order block reduction of a per-thread sum(w*w) -> partials[blockIdx]
// (deterministic: warp shuffles in a fixed pattern, warps in index order)
__device__ __forceinline__ void block_sumsq_partial(double acc,
                                                    double *partials) {
  __shared__ double red[32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
    acc = dadd(acc, __shfl_down_sync(0xffffffffu, acc, off));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int q = 0; q < (int)(blockDim.x / 32); ++q) sum = dadd(sum, red[q]);
    partials[blockIdx.x] = sum;
  }
}

// partials[0..n) -> *out in index order (one thread; n ~ #SMs)
int sem_sumsq_finish(const double *partials, int n, double *out,
                     cudaStream_t s);

// -1 when the general kernel has no entry for (n, variant)
int sem_gen_dispatch(int n, int variant, double *w, const double *u,
                     const double *d, const double *g, int64_t nelt,
                     const lfb_launch *geom, cudaStream_t s,
                     int64_t *grid_out);

// -1 when the two-columns-per-thread kernel has no entry for (n, variant)
int sem_gen2_dispatch(int n, int variant, double *w, const double *u,
                      const double *d, const double *g, int64_t nelt,
                      const lfb_launch *geom, cudaStream_t s,
                      int64_t *grid_out);

// -1 when the DMMA kernel has no entry for (n, variant)
int sem_tc_dispatch(int n, int variant, double *w, const double *u,
                    const double *d, const double *g, int64_t nelt,
                    const lfb_launch *geom, cudaStream_t s,
                    int64_t *grid_out);

// -1 when the constant-bank kernel has no entry for (n, variant)
int sem_kc_dispatch(int n, int variant, double *w, const double *u,
                    const double *d, const double *g, int64_t nelt,
                    const lfb_launch *geom, cudaStream_t s,
                    int64_t *grid_out);

// -1 when the line-owner kernel has no entry for (n, variant)
int sem_line_dispatch(int n, int variant, double *w, const double *u,
                      const double *d, const double *g, int64_t nelt,
                      const lfb_launch *geom, cudaStream_t s,
                      int64_t *grid_out);

// u of n = 16 elements as a (16 x 256 nelt) 2-D tensor map with the 128-B
// swizzle (semlap_tc.cu); false when it cannot be encoded
bool sem_u16_map(CUtensorMap *map, const double *u, int64_t nelt);

int sem_slab_dispatch(int n, int variant, double *w, const double *u, const double *d,
                      const double *g, int64_t nelt, const lfb_launch *geom,
                      cudaStream_t s, int64_t *grid_out);

}  // namespace lfb
