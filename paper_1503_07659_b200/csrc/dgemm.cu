// dgemm -- the paper's DGEMM kernel in real*8 (/root/reference/pkg/tests/
// test_fortran.py:72-103, the real*4 variant is BASELINE config 5):
//   c(i,j) = c(i,j) + alpha*b(k,j)*a(i,k)   for k ascending
// column major a(m,l) at a[i + m k], b(l,n) at b[k + l j], c(m,n) at
// c[i + m j].
//
// Two kernels behind lfb_dgemm_f64:
//  * default (tensor cores, tolerance parity): the FP64 DMMA units
//    (mma.sync m8n8k4 f64), acc = sum_k a(i,k) b(k,j) fused in the tensor
//    pipe, then c = c + alpha*acc -- within the north star's 1e-12 relative
//    fp64 bound normwise (tests/test_gpu_parity.py).  128x128x32 CTA tiles
//    (x16 when l is not a multiple of 32) through a cp.async ring filled by
//    a producer warp and handed over on full / empty mbarriers (no block
//    barrier), in padded shared memory (row strides 132 and BK + 4 doubles:
//    every fragment load of a half warp hits 16 distinct 8-byte bank
//    slots), 8 consumer warps of 64x32 each: per k-step of 4,
//    8 A and 4 B fragment loads feed 32 DMMAs.  Needs m, n % 128 == 0,
//    l % 16 == 0 and 16-byte aligned arrays; other shapes take the exact
//    kernel.
//  * variant 1 (bit-exact): the reference's chain per output element on
//    the FP64 CUDA cores, c + ((alpha*b)*a) with every operation rounded
//    separately, k ascending (the sgemm exact kernel's structure in f64).
#include "lfb_common.cuh"

namespace lfb {

// {{{ DMMA kernel

constexpr int DG_BM = 128, DG_BN = 128, DG_BK = 16, DG_STAGES = 4;
constexpr int DG_THREADS = 256;
constexpr int DG_AS = 132;  // As row stride (doubles): k rows of 128 i

template <int BK, int ST>
struct DgSmem {
  static constexpr int BS = BK + 4;  // Bs row stride: j rows of BK k
  static constexpr size_t a_doubles = BK * DG_AS;
  static constexpr size_t b_doubles = DG_BN * BS;
  static constexpr size_t stage = a_doubles + b_doubles;
  static constexpr size_t total = ST * stage * 8;
};

__device__ __forceinline__ void dg_dmma(double &d0, double &d1, double a,
                                        double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, "
      "{%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   smem_u32(dst)),
               "l"(src)
               : "memory");
}

// BK k per stage, ST stages
template <int BK, int ST>
__global__ void __launch_bounds__(DG_THREADS, 1)
    dgemm_dmma_kernel(double alpha, const double *__restrict__ a,
                      const double *__restrict__ b, double *__restrict__ c,
                      int l, int m, int n) {
  using L = DgSmem<BK, ST>;
  constexpr int BS = L::BS, KS = BK / 4;
  extern __shared__ __align__(128) double dsm[];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int r = lane / 4, q = lane % 4;
  const int wm = warp / 4, wn = warp % 4;  // 2 x 4 warps of 64 x 32
  const int i0 = blockIdx.x * DG_BM, j0 = blockIdx.y * DG_BN;
  const int nk = l / BK;

  auto As = [&](int s) { return dsm + (size_t)s * L::stage; };
  auto Bs = [&](int s) { return As(s) + L::a_doubles; };
  auto load = [&](int s, int kt) {
    const int k0 = kt * BK;
    double *as = As(s), *bs = Bs(s);
#pragma unroll
    for (int x = 0; x < BK / 4; ++x) {
      const int ch = tid + DG_THREADS * x;
      {  // A: BK rows (k) of 128 i, 64 chunks of 2 doubles per row
        const int k = ch / 64, i = (ch % 64) * 2;
        cp16(as + k * DG_AS + i, a + (i0 + i) + (int64_t)m * (k0 + k));
      }
      {  // B: 128 rows (j) of BK k, BK / 2 chunks per row
        const int j = ch / (BK / 2), k = (ch % (BK / 2)) * 2;
        cp16(bs + j * BS + k, b + (k0 + k) + (int64_t)l * (j0 + j));
      }
    }
  };

  double acc[8][4][2];
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nk) load(s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(ST - 2) : "memory");
    __syncthreads();  // stage kt landed for every thread; stage kt-1 free
    {
      const int nxt = kt + ST - 1;
      if (nxt < nk) load(nxt % ST, nxt);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const double *as = As(kt % ST), *bs = Bs(kt % ST);
    auto frags = [&](int ks, double (&fa)[8], double (&fb)[4]) {
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)  // A[i][k]: row i = lane/4, col k
        fa[mt] = as[(4 * ks + q) * DG_AS + wm * 64 + mt * 8 + r];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)  // B[k][j]: row k = lane%4, col j
        fb[nt] = bs[(wn * 32 + nt * 8 + r) * BS + 4 * ks + q];
    };
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      double fa[8], fb[4];
      frags(ks, fa, fb);
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          dg_dmma(acc[mt][nt][0], acc[mt][nt][1], fa[mt], fb[nt]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

  // c = c + alpha*acc; lane holds rows i = .. + r, columns j = .. + 2q + h
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = i0 + wm * 64 + mt * 8 + r;
        const int j = j0 + wn * 32 + nt * 8 + 2 * q + h;
        double *p = c + i + (int64_t)m * j;
        *p = dadd(*p, dmul(alpha, acc[mt][nt][h]));
      }
}

// Warp-specialised kernel (the default): one producer warp streams the k tiles
// with cp.async and signals each stage's full mbarrier through
// cp.async.mbarrier.arrive (no block-wide barrier); the 8 consumer warps
// wait on it, run the stage's DMMAs and release the stage on its empty
// mbarrier, so no consumer waits for another.
template <int BK, int ST>
__global__ void __launch_bounds__(DG_THREADS + 32, 1)
    dgemm_ws_kernel(double alpha, const double *__restrict__ a,
                    const double *__restrict__ b, double *__restrict__ c,
                    int l, int m, int n) {
  using L = DgSmem<BK, ST>;
  constexpr int BS = L::BS, KS = BK / 4;
  extern __shared__ __align__(128) double dsm[];
  __shared__ uint64_t full[ST], empty[ST];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int i0 = blockIdx.x * DG_BM, j0 = blockIdx.y * DG_BN;
  const int nk = l / BK;
  auto As = [&](int s) { return dsm + (size_t)s * L::stage; };
  auto Bs = [&](int s) { return As(s) + L::a_doubles; };
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 32);  // one cp.async arrive per producer lane
      mbar_init(&empty[s], 256);  // every consumer thread arrives
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 8) {  // producer
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % ST;
      mbar_wait(&empty[s], ((kt / ST) & 1) ^ 1);
      const int k0 = kt * BK;
      double *as = As(s), *bs = Bs(s);
#pragma unroll 8
      for (int x = 0; x < BK * 64 / 32; ++x) {
        const int ch = lane + 32 * x;
        {  // A: BK rows (k) of 128 i, 64 chunks of 2 doubles per row
          const int k = ch / 64, i = (ch % 64) * 2;
          cp16(as + k * DG_AS + i, a + (i0 + i) + (int64_t)m * (k0 + k));
        }
        {  // B: 128 rows (j) of BK k, BK / 2 chunks per row
          const int j = ch / (BK / 2), k = (ch % (BK / 2)) * 2;
          cp16(bs + j * BS + k, b + (k0 + k) + (int64_t)l * (j0 + j));
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::
                       "r"(smem_u32(&full[s]))
                   : "memory");
    }
    return;
  }

  const int r = lane / 4, q = lane % 4;
  const int wm = warp / 4, wn = warp % 4;  // 2 x 4 warps of 64 x 32
  double acc[8][4][2];
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % ST;
    mbar_wait(&full[s], (kt / ST) & 1);
    const double *as = As(s), *bs = Bs(s);
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      double fa[8], fb[4];
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
        fa[mt] = as[(4 * ks + q) * DG_AS + wm * 64 + mt * 8 + r];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
        fb[nt] = bs[(wn * 32 + nt * 8 + r) * BS + 4 * ks + q];
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          dg_dmma(acc[mt][nt][0], acc[mt][nt][1], fa[mt], fb[nt]);
    }
    // every thread releases its own reads of the stage (release order)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                     smem_u32(&empty[s]))
                 : "memory");
  }
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = i0 + wm * 64 + mt * 8 + r;
        const int j = j0 + wn * 32 + nt * 8 + 2 * q + h;
        double *p = c + i + (int64_t)m * j;
        *p = dadd(*p, dmul(alpha, acc[mt][nt][h]));
      }
}

template <int BK, int ST>
static int launch_dgemm_ws(double alpha, const double *a, const double *b,
                           double *c, int l, int m, int n, cudaStream_t s) {
  using L = DgSmem<BK, ST>;
  static_assert(L::total <= 226 * 1024, "smem");
  auto k = dgemm_ws_kernel<BK, ST>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)L::total);
  dim3 grid(m / DG_BM, n / DG_BN);
  k<<<grid, DG_THREADS + 32, L::total, s>>>(alpha, a, b, c, l, m, n);
  return check_launch("lfb_dgemm_f64(dmma ws)");
}

template <int BK, int ST>
static int launch_dgemm_dmma(double alpha, const double *a, const double *b,
                             double *c, int l, int m, int n, cudaStream_t s) {
  using L = DgSmem<BK, ST>;
  static_assert(L::total <= 227 * 1024, "smem");
  auto k = dgemm_dmma_kernel<BK, ST>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)L::total);
  dim3 grid(m / DG_BM, n / DG_BN);
  k<<<grid, DG_THREADS, L::total, s>>>(alpha, a, b, c, l, m, n);
  return check_launch("lfb_dgemm_f64(dmma)");
}

// }}}

// {{{ bit-exact kernel (the reference's sequential chain)

constexpr int DE_BM = 128, DE_BN = 128, DE_BK = 8, DE_THREADS = 256;

__global__ void __launch_bounds__(DE_THREADS)
    dgemm_exact_kernel(double alpha, const double *__restrict__ a,
                       const double *__restrict__ b, double *__restrict__ c,
                       int l, int m, int n) {
  __shared__ double As[2][DE_BK][DE_BM];
  __shared__ double Bs[2][DE_BK][DE_BN];  // alpha*b(k,j)

  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // 16 x 16 threads, 8x8 each
  const int i0 = blockIdx.x * DE_BM, j0 = blockIdx.y * DE_BN;

  double acc[8][8];
#pragma unroll
  for (int ii = 0; ii < 8; ++ii)
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int gi = i0 + ty * 8 + ii, gj = j0 + tx * 8 + jj;
      acc[ii][jj] = (gi < m && gj < n) ? c[gi + (int64_t)m * gj] : 0.0;
    }

  // A slab 128(i) x 8(k): thread -> (i = tid % 128, k = tid / 128 * 4 + q)
  // B slab 8(k) x 128(j): thread -> (k = tid % 8, j = tid / 8 * 4 + q)
  double ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int ii = tid % DE_BM, kk = (tid / DE_BM) * 4 + x;
      const int gi = i0 + ii, gk = k0 + kk;
      ra[x] = (gi < m && gk < l) ? __ldg(a + gi + (int64_t)m * gk) : 0.0;
      const int kb = tid % DE_BK, jb = (tid / DE_BK) * 4 + x;
      const int gkb = k0 + kb, gj = j0 + jb;
      rb[x] = (gkb < l && gj < n) ? __ldg(b + gkb + (int64_t)l * gj) : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      As[buf][(tid / DE_BM) * 4 + x][tid % DE_BM] = ra[x];
      Bs[buf][tid % DE_BK][(tid / DE_BK) * 4 + x] = dmul(alpha, rb[x]);
    }
  };

  const int nk = (l + DE_BK - 1) / DE_BK;
  load(0);
  store(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load((t + 1) * DE_BK);
    const int kmax = min(DE_BK, l - t * DE_BK);
    for (int kk = 0; kk < kmax; ++kk) {
      double av[8], bv[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        av[x] = As[buf][kk][ty * 8 + x];
        bv[x] = Bs[buf][kk][tx * 8 + x];
      }
#pragma unroll
      for (int ii = 0; ii < 8; ++ii)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          acc[ii][jj] = dadd(acc[ii][jj], dmul(bv[jj], av[ii]));
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

// }}}

}  // namespace lfb

extern "C" int lfb_dgemm_f64(double alpha, const double *a, const double *b,
                             double *c, int l, int m, int n,
                             const lfb_launch *geom, lfb_stream stream) {
  using namespace lfb;
  if (l < 0 || m < 0 || n < 0)
    return fail(LFB_ERR_ARG, "lfb_dgemm_f64: negative extent");
  if (m == 0 || n == 0) return LFB_OK;
  if (!a || !b || !c) return fail(LFB_ERR_ARG, "lfb_dgemm_f64: null array");
  if (geom && geom->abi_version != LFB_ABI_VERSION)
    return fail(LFB_ERR_ARG, "lfb_dgemm_f64: bad lfb_launch version");
  cudaStream_t s = (cudaStream_t)stream;
  const int variant = geom ? geom->variant : 0;
  const bool tc_ok = m % DG_BM == 0 && n % DG_BN == 0 && l % DG_BK == 0 &&
                     l > 0 && aligned(a, 16) && aligned(b, 16);
  if (variant != 1 && tc_ok) {
    // default: the warp-specialised kernel, k tiles of 32 through 3 stages
    // when l allows, else 16 x 5 (32.9 TFLOP/s at 8192^3 vs 30.9 for round
    // 1's block-synchronous 16 x 4 kernel, kept as variant 3)
    if (variant != 3)
      return l % 32 == 0
                 ? launch_dgemm_ws<32, 3>(alpha, a, b, c, l, m, n, s)
                 : launch_dgemm_ws<16, 5>(alpha, a, b, c, l, m, n, s);
    return launch_dgemm_dmma<DG_BK, DG_STAGES>(alpha, a, b, c, l, m, n, s);
  }
  if (variant == 2)
    return fail(LFB_ERR_UNSUPPORTED,
                "lfb_dgemm_f64: the tensor-core path needs m %% 128, "
                "n %% 128, l %% 16 == 0 and 16-byte aligned a, b "
                "(m=%d n=%d l=%d)", m, n, l);
  dim3 grid((m + DE_BM - 1) / DE_BM, (n + DE_BN - 1) / DE_BN);
  if (grid.y > 65535)
    return fail(LFB_ERR_UNSUPPORTED, "lfb_dgemm_f64: n=%d too large", n);
  dgemm_exact_kernel<<<grid, DE_THREADS, 0, s>>>(alpha, a, b, c, l, m, n);
  return check_launch("lfb_dgemm_f64(exact)");
}
