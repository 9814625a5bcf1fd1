// Element-wise workloads: fill and axpy (BASELINE config 1).
//
// Reference arithmetic (interp.py:365-383 + 169-187, emitted C identical):
//   fill:  out[i] = a                      (store of the scalar argument)
//   axpy:  y[i] = y[i] + alpha*x[i]        (multiply rounded, then add)
// over the logical index space i = i_inner + B*i_outer, 0 <= i < n, that the
// split_iname(i, B, g.0, l.0) script defines (guard "1 + i_inner + B*i_outer
// <= n" unless assume(n mod B = 0), codegen.py:590-612).
//
// B200 mapping: HBM-bound streams.  CTA size = the l.0 extent (B) when it is a
// legal block size, each thread moves 16-byte vectors (st.global.v2.f64 /
// ld.global.nc.v2.f64), CTAs cover several logical work-groups each in a
// grid-stride walk sized to the SM count, scalar head/tail for ragged n or
// misaligned pointers.
#include "lfb_common.cuh"

namespace lfb {

template <typename T>
struct Vec;
template <>
struct Vec<double> {
  using V = double2;
  static constexpr int W = 2;
};
template <>
struct Vec<float> {
  using V = float4;
  static constexpr int W = 4;
};

template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) {
  return dmul(a, b);
}
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) {
  return fmul(a, b);
}
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) {
  return dadd(a, b);
}
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) {
  return fadd(a, b);
}

template <typename T>
__global__ void fill_vec_kernel(T *__restrict__ out, T a, int64_t nvec) {
  using V = typename Vec<T>::V;
  V v;
  T *pv = reinterpret_cast<T *>(&v);
#pragma unroll
  for (int c = 0; c < Vec<T>::W; ++c) pv[c] = a;
  V *o = reinterpret_cast<V *>(out);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nvec;
       q += stride)
    __stcs(o + q, v);
}

// fill through the TMA engine: a CTA writes `a` into a CHUNK-byte smem tile
// once, then one thread streams that tile to its share of the output with
// bulk shared->global copies (cp.async.bulk ... bulk_group).  No per-element
// store instructions at all; the copies only read smem, so the tile is reused
// for every chunk and the CTA waits for the reads before it exits.
constexpr int FILL_CHUNK = 32768;

template <typename T>
__global__ void __launch_bounds__(256, 1)
    fill_bulk_kernel(T *__restrict__ out, T a, int64_t nbytes) {
  extern __shared__ __align__(128) unsigned char fsmem[];
  T *tile = reinterpret_cast<T *>(fsmem);
  for (int q = threadIdx.x; q < FILL_CHUNK / (int)sizeof(T); q += blockDim.x)
    tile[q] = a;
  fence_proxy_async_smem();  // generic-proxy writes -> async-proxy reads
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t nchunks = (nbytes + FILL_CHUNK - 1) / FILL_CHUNK;
    unsigned char *o = reinterpret_cast<unsigned char *>(out);
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      const int64_t off = c * FILL_CHUNK;
      const int64_t rem = nbytes - off;
      const uint32_t bytes = (uint32_t)(rem < FILL_CHUNK ? rem : FILL_CHUNK);
      asm volatile(
          "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
              o + off),
          "r"(smem_u32(tile)), "r"(bytes)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

template <typename T>
__global__ void fill_scalar_kernel(T *__restrict__ out, T a, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += stride)
    out[q] = a;
}

template <typename T, int U>
__global__ void axpy_vec_kernel(T *__restrict__ y, const T *__restrict__ x,
                                T alpha, int64_t nvec) {
  using V = typename Vec<T>::V;
  constexpr int W = Vec<T>::W;
  V *yv = reinterpret_cast<V *>(y);
  const V *xv = reinterpret_cast<const V *>(x);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x;
       base < nvec; base += stride) {
    V ya[U], xa[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t q = base + (int64_t)u * blockDim.x;
      if (q < nvec) {
        ya[u] = __ldcs(yv + q);
        xa[u] = __ldcs(xv + q);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t q = base + (int64_t)u * blockDim.x;
      if (q < nvec) {
        T *py = reinterpret_cast<T *>(&ya[u]);
        const T *px = reinterpret_cast<const T *>(&xa[u]);
#pragma unroll
        for (int c = 0; c < W; ++c) py[c] = add_rn<T>(py[c], mul_rn<T>(alpha, px[c]));
        __stcs(yv + q, ya[u]);
      }
    }
  }
}

template <typename T>
__global__ void axpy_scalar_kernel(T *__restrict__ y, const T *__restrict__ x,
                                   T alpha, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += stride)
    y[q] = add_rn<T>(y[q], mul_rn<T>(alpha, x[q]));
}

// CTA size: the l.0 extent when it is a legal block, else 256.
static int block_of(const lfb_launch *geom) {
  if (geom && geom->local_extent[0] >= 32 && geom->local_extent[0] <= 1024 &&
      geom->local_extent[0] % 32 == 0 && geom->local_extent[1] <= 1 &&
      geom->local_extent[2] <= 1)
    return geom->local_extent[0];
  return 256;
}

static int check_geom(const char *what, const lfb_launch *geom, int64_t n) {
  if (!geom) return LFB_OK;
  if (geom->abi_version != LFB_ABI_VERSION)
    return fail(LFB_ERR_ARG, "%s: lfb_launch.abi_version %d != %d", what,
                geom->abi_version, LFB_ABI_VERSION);
  // the logical index space must cover [0, n): g.0 * l.0 >= n
  if (geom->group_extent[0] == 0) return LFB_OK;  // untransformed kernel
  int64_t covered = geom->group_extent[0] * (int64_t)geom->local_extent[0];
  if (covered < n)
    return fail(LFB_ERR_ARG,
                "%s: launch geometry covers %lld of n=%lld points", what,
                (long long)covered, (long long)n);
  return LFB_OK;
}

static int grid_for(int64_t work, int block, const lfb_launch *geom,
                    int per_thread) {
  int sms = sm_count(geom);
  if (sms <= 0) sms = 148;
  int per_sm = (geom && geom->ctas_per_sm > 0) ? geom->ctas_per_sm
                                                : (2048 / block);
  int64_t want = (work + (int64_t)block * per_thread - 1) /
                 ((int64_t)block * per_thread);
  int64_t cap = (int64_t)sms * per_sm;
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

template <typename T>
static int fill_impl(const char *what, T *out, T a, int n,
                     const lfb_launch *geom, lfb_stream stream) {
  if (n < 0) return fail(LFB_ERR_ARG, "%s: n=%d < 0", what, n);
  if (n == 0) return LFB_OK;
  if (!out) return fail(LFB_ERR_ARG, "%s: null output", what);
  if (int rc = check_geom(what, geom, n)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int block = block_of(geom);
  constexpr int W = Vec<T>::W;
  if (aligned(out, 16)) {
    int64_t nvec = n / W;
    const bool bulk = !(geom && geom->variant == 1);
    if (nvec && bulk) {
      // whole 16-byte vectors by bulk copies, one CTA per SM
      int sms = sm_count(geom);
      if (sms <= 0) sms = 148;
      const int64_t nbytes = nvec * 16;
      const int64_t chunks = (nbytes + FILL_CHUNK - 1) / FILL_CHUNK;
      const int per_sm = (geom && geom->ctas_per_sm > 0) ? geom->ctas_per_sm
                                                          : 1;
      const int64_t cap = (int64_t)sms * per_sm;
      const int grid = (int)(chunks < cap ? chunks : cap);
      cudaFuncSetAttribute(fill_bulk_kernel<T>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           FILL_CHUNK);
      fill_bulk_kernel<T><<<grid, 256, FILL_CHUNK, s>>>(out, a, nbytes);
    } else if (nvec) {
      fill_vec_kernel<T><<<grid_for(nvec, block, geom, 4), block, 0, s>>>(
          out, a, nvec);
    }
    int64_t done = nvec * W;
    if (done < n)
      fill_scalar_kernel<T><<<1, 32, 0, s>>>(out + done, a, n - done);
  } else {
    fill_scalar_kernel<T><<<grid_for(n, block, geom, 4), block, 0, s>>>(
        out, a, n);
  }
  return check_launch(what);
}

template <typename T>
static int axpy_impl(const char *what, T *y, const T *x, T alpha, int n,
                     const lfb_launch *geom, lfb_stream stream) {
  if (n < 0) return fail(LFB_ERR_ARG, "%s: n=%d < 0", what, n);
  if (n == 0) return LFB_OK;
  if (!y || !x) return fail(LFB_ERR_ARG, "%s: null array", what);
  if (int rc = check_geom(what, geom, n)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int block = block_of(geom);
  constexpr int W = Vec<T>::W;
  constexpr int U = 4;
  if (aligned(y, 16) && aligned(x, 16)) {
    int64_t nvec = n / W;
    if (nvec)
      axpy_vec_kernel<T, U><<<grid_for(nvec, block, geom, U), block, 0, s>>>(
          y, x, alpha, nvec);
    int64_t done = nvec * W;
    if (done < n)
      axpy_scalar_kernel<T><<<1, 32, 0, s>>>(y + done, x + done, alpha,
                                             n - done);
  } else {
    axpy_scalar_kernel<T><<<grid_for(n, block, geom, 4), block, 0, s>>>(
        y, x, alpha, n);
  }
  return check_launch(what);
}

}  // namespace lfb

extern "C" {

int lfb_fill_f64(double *out, double a, int n, const lfb_launch *geom,
                 lfb_stream stream) {
  return lfb::fill_impl<double>("lfb_fill_f64", out, a, n, geom, stream);
}

int lfb_fill_f32(float *out, float a, int n, const lfb_launch *geom,
                 lfb_stream stream) {
  return lfb::fill_impl<float>("lfb_fill_f32", out, a, n, geom, stream);
}

int lfb_axpy_f64(double *y, const double *x, double alpha, int n,
                 const lfb_launch *geom, lfb_stream stream) {
  return lfb::axpy_impl<double>("lfb_axpy_f64", y, x, alpha, n, geom, stream);
}

int lfb_axpy_f32(float *y, const float *x, float alpha, int n,
                 const lfb_launch *geom, lfb_stream stream) {
  return lfb::axpy_impl<float>("lfb_axpy_f32", y, x, alpha, n, geom, stream);
}

}  // extern "C"
