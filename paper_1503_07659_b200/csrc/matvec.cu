// Dense matrix-vector product (BASELINE config 2).
//
// Reference arithmetic (SURVEY.md Appendix B fixture, fixtures.py
// matvec_source; interp.py:323-400, emitted C identical):
//   for every row i:  s = 0
//                     for j ascending: s = s + a(i,j)*x(j)
//                     y(i) = s
// a is column major, a(i,j) at a[i + n j] (fortran.py:638-658).  The
// reference script's extract_subst + precompute stage x in a private 32-wide
// tile (transforms.py:541-684) -- a copy, so values are unchanged.
//
// Variants (lfb_launch.variant): 0 = split-j (below; within the north
// star's 1e-12 fp64 tolerance, HBM bound) when n >= 256, 1 = direct-load
// bitwise, 2 = split-j only, 3 = the bitwise TMA kernel.
//
// Bitwise kernels: every row is one sequential chain of 2n separately
// rounded operations; the device keeps that chain and parallelises over
// rows only.
// The kernel is HBM bound (8 n^2 bytes of a), so the design is about bytes in
// flight, not FLOPs:
//  * one CTA per 32-row panel: warp 0 computes (lane r owns row i0 + r),
//    warp 1 lane 0 is the TMA producer;
//  * the producer streams 32 x JT tiles of a with cp.async.bulk.tensor.2d
//    (a tensor map over the column-major matrix; out-of-range rows/columns
//    are zero filled and never summed) plus the matching x slice with a 1-D
//    bulk copy, through an S-stage full/empty mbarrier ring (S*16 KB in
//    flight per SM);
//  * the consumer reads its row from smem (conflict free: lanes hit
//    consecutive doubles) and x[j] as a broadcast.
// n odd (TMA needs 16-byte strides) or tiny n falls back to a direct-load
// kernel with the same arithmetic.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "lfb_common.cuh"

namespace lfb {

constexpr int MV_ROWS = 32;
constexpr int MV_JT = 64;
constexpr int MV_STAGES = 8;

struct MvSmem {
  static constexpr size_t bars = 256;
  static constexpr size_t tile_bytes = MV_ROWS * MV_JT * 8;  // 16 KB
  static constexpr size_t x_bytes = MV_JT * 8;
  static constexpr size_t tiles_off = 1024;
  static constexpr size_t xs_off = tiles_off + MV_STAGES * tile_bytes;
  static constexpr size_t total = xs_off + MV_STAGES * x_bytes;
};

// The consumer is software pipelined: a dependent DADD costs 8.1 cycles on
// B200 (tools/micro/dadd_latency.cu), so the row chain alone needs
// n x 8.1 cycles; the products of tile q + 1 (LDS + DMUL, independent) are
// interleaved with the 64 chained DADDs of tile q in program order, so the
// warp's in-order issue never waits on anything but the chain itself.  A
// stage is released as soon as its products are in registers.  Measured:
// the consumer's loop alone runs at 8.07 cycles per column
// (tools/micro/chain_probe.cu) and the stream alone at 6.1 TB/s (22 us at
// n = 4096), but together 35 us: the in-order consumer waits for tile q + 1
// before it can chain tile q, so memory latency and the chain only partly
// overlap (a variant that hands the products to a separate chain warp
// through a shared-memory ring measured the same, 36 us).  The split-j
// kernel below is the default.
template <int ROWS>
__global__ void __launch_bounds__(64, 1)
    matvec_tma_kernel(const __grid_constant__ CUtensorMap tmap_a,
                      double *__restrict__ y, const double *__restrict__ x,
                      int n) {
  constexpr int JT = MV_JT, ST = MV_STAGES;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem);
  uint64_t *empty = full + ST;
  double *tiles = reinterpret_cast<double *>(smem + MvSmem::tiles_off);
  double *xs = reinterpret_cast<double *>(smem + MvSmem::xs_off);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int i0 = blockIdx.x * ROWS;
  const int ntiles = (n + JT - 1) / JT;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 32);  // every lane of the consumer warp
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 1) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_a) : "memory");
      const uint64_t pol = policy_evict_first();
      for (int q = 0; q < ntiles; ++q) {
        const int s = q % ST;
        mbar_wait(&empty[s], ((q / ST) & 1) ^ 1);
        fence_proxy_async_smem();  // the consumer's reads, then TMA writes
        const int j0 = q * JT;
        const int jn = min(JT, n - j0);
        const uint32_t xb = (uint32_t)jn * 8;  // n even => multiple of 16
        mbar_arrive_expect_tx(&full[s], (uint32_t)(ROWS * JT * 8) + xb);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::"
            "complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
                smem_u32(tiles + (size_t)s * MV_ROWS * JT)),
            "l"(&tmap_a), "r"(i0), "r"(j0), "r"(smem_u32(&full[s])),
            "l"(pol)
            : "memory");
        bulk_g2s(xs + s * JT, x + j0, xb, &full[s]);
      }
    }
    return;
  }

  // consumer warp: lane owns row i0 + lane (lanes >= ROWS idle)
  auto release = [&](int s) {  // every lane releases its own reads
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                     smem_u32(&empty[s]))
                 : "memory");
  };
  const int r = lane < ROWS ? lane : 0;
  double acc = 0.0;  // "s = 0" (an i32 literal stored into the f64 scalar)
  const int nfull = n / JT;
  double p[JT];
  if (nfull > 0) {
    mbar_wait(&full[0], 0);
    const double *t0 = tiles, *x0 = xs;
#pragma unroll
    for (int jj = 0; jj < JT; ++jj) p[jj] = dmul(t0[jj * ROWS + r], x0[jj]);
    release(0);
  }
  constexpr int LD = 4;  // load distance: LDS latency / DADD latency
  for (int q = 0; q < nfull; ++q) {
    const bool nxt = q + 1 < nfull;
    const int sn = (q + 1) % ST;
    if (nxt) mbar_wait(&full[sn], ((q + 1) / ST) & 1);
    const double *tn = tiles + (size_t)sn * MV_ROWS * JT;
    const double *xn = xs + sn * JT;
    double la[LD], lx[LD];
#pragma unroll
    for (int d = 0; d < LD; ++d) {
      la[d] = nxt ? tn[d * ROWS + r] : 0.0;
      lx[d] = nxt ? xn[d] : 0.0;
    }
#pragma unroll
    for (int jj = 0; jj < JT; ++jj) {
      acc = dadd(acc, p[jj]);  // the reference's chain, column order
      const double a_ = la[jj % LD], x_ = lx[jj % LD];
      if (nxt && jj + LD < JT) {  // the load LD columns ahead
        la[jj % LD] = tn[(jj + LD) * ROWS + r];
        lx[jj % LD] = xn[jj + LD];
      }
      p[jj] = dmul(a_, x_);       // product of tile q + 1 (unused if none)
    }
    if (nxt) release(sn);
  }
  if (nfull < ntiles) {  // ragged last tile: exactly jn more terms
    const int q = nfull, s = q % ST;
    mbar_wait(&full[s], (q / ST) & 1);
    const double *t = tiles + (size_t)s * MV_ROWS * JT, *xt = xs + s * JT;
    const int jn = n - q * JT;
    for (int jj = 0; jj < jn; ++jj)
      acc = dadd(acc, dmul(t[jj * ROWS + r], xt[jj]));
    release(s);
  }
  if (lane < ROWS && i0 + lane < n) y[i0 + lane] = acc;
}

// {{{ split-j kernel (default; variant 2 forces it): tolerance parity, HBM
// bound
//
// The reference's row chain s = (((0 + a(i,0)x(0)) + a(i,1)x(1)) + ...) is
// n dependent DADDs; on B200 a dependent DADD costs ~18 cycles, so the bitwise
// kernel above is bound by that chain (4096 x 18 cycles = 37 us at n = 4096,
// profiles/r01_matvec.md), not by HBM.  This variant re-associates once:
// W consumer warps per 32-row panel each run the reference chain over one
// contiguous quarter of the columns (part 0 is bitwise the reference's
// prefix), and y(i) = ((p0 + p1) + p2) + p3.  Within the north star's 1e-12
// relative fp64 tolerance (tests: normwise), and the chains are W x shorter.
constexpr int MVS_W = 4;       // consumer warps = column parts
constexpr int MVS_STAGES = 3;  // ring depth per consumer warp

struct MvsSmem {
  static constexpr size_t tile_bytes = MV_ROWS * MV_JT * 8;  // 16 KB
  static constexpr size_t x_bytes = MV_JT * 8;
  static constexpr size_t nslot = (size_t)MVS_W * MVS_STAGES;
  static constexpr size_t tiles_off = 1024;
  static constexpr size_t xs_off = tiles_off + nslot * tile_bytes;
  static constexpr size_t red_off = xs_off + nslot * x_bytes;
  static constexpr size_t total = red_off + MVS_W * MV_ROWS * 8;
};

__global__ void __launch_bounds__(32 * (MVS_W + 1), 1)
    matvec_split_kernel(const __grid_constant__ CUtensorMap tmap_a,
                        double *__restrict__ y, const double *__restrict__ x,
                        int n) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem);
  uint64_t *empty = full + MvsSmem::nslot;
  double *tiles = reinterpret_cast<double *>(smem + MvsSmem::tiles_off);
  double *xs = reinterpret_cast<double *>(smem + MvsSmem::xs_off);
  double *red = reinterpret_cast<double *>(smem + MvsSmem::red_off);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int i0 = blockIdx.x * MV_ROWS;
  const int ntiles = (n + MV_JT - 1) / MV_JT;
  // part w owns tiles [t0(w), t0(w + 1))
  auto t0 = [&](int w) { return (int)(((int64_t)ntiles * w) / MVS_W); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < (int)MvsSmem::nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 32);  // every lane of the consumer warp
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == MVS_W) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_a) : "memory");
      const uint64_t pol = policy_evict_first();
      const int most = t0(MVS_W) - t0(MVS_W - 1);  // parts differ by <= 1
      for (int q = 0; q < most + 1; ++q) {
        for (int w = 0; w < MVS_W; ++w) {
          const int tq = t0(w) + q;
          if (tq >= t0(w + 1)) continue;
          const int slot = w * MVS_STAGES + q % MVS_STAGES;
          mbar_wait(&empty[slot], ((q / MVS_STAGES) & 1) ^ 1);
          fence_proxy_async_smem();  // the consumers' reads, then TMA writes
          const int j0 = tq * MV_JT;
          const int jn = min(MV_JT, n - j0);
          const uint32_t xb = (uint32_t)jn * 8;
          mbar_arrive_expect_tx(&full[slot], (uint32_t)MvsSmem::tile_bytes + xb);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::"
              "complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], "
              "%5;" ::"r"(smem_u32(tiles + (size_t)slot * MV_ROWS * MV_JT)),
              "l"(&tmap_a), "r"(i0), "r"(j0), "r"(smem_u32(&full[slot])),
              "l"(pol)
              : "memory");
          bulk_g2s(xs + slot * MV_JT, x + j0, xb, &full[slot]);
        }
      }
    }
    return;
  }

  // consumer warp `warp`: the reference chain over its column part
  double acc = 0.0;
  const int nt = t0(warp + 1) - t0(warp);
  for (int q = 0; q < nt; ++q) {
    const int slot = warp * MVS_STAGES + q % MVS_STAGES;
    mbar_wait(&full[slot], (q / MVS_STAGES) & 1);
    const double *tile = tiles + (size_t)slot * MV_ROWS * MV_JT;
    const double *xt = xs + slot * MV_JT;
    const int jn = min(MV_JT, n - (t0(warp) + q) * MV_JT);
    if (jn == MV_JT) {
#pragma unroll 16
      for (int jj = 0; jj < MV_JT; ++jj)
        acc = dadd(acc, dmul(tile[jj * MV_ROWS + lane], xt[jj]));
    } else {
      for (int jj = 0; jj < jn; ++jj)
        acc = dadd(acc, dmul(tile[jj * MV_ROWS + lane], xt[jj]));
    }
    // every lane releases its own reads of the slot (compute-sanitizer's
    // racecheck does not credit one lane's arrive after __syncwarp); the
    // producer fences the proxy after its wait
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                     smem_u32(&empty[slot]))
                 : "memory");
  }
  red[warp * MV_ROWS + lane] = acc;
  named_bar_sync(1, 32 * MVS_W);
  if (warp == 0) {
    double s = red[lane];
#pragma unroll
    for (int w = 1; w < MVS_W; ++w) s = dadd(s, red[w * MV_ROWS + lane]);
    if (i0 + lane < n) y[i0 + lane] = s;
  }
}

// }}}

// direct-load fallback: a warp per 32 rows, loads of a coalesced across lanes
__global__ void matvec_direct_kernel(double *__restrict__ y,
                                     const double *__restrict__ a,
                                     const double *__restrict__ x, int n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  const double *col = a + i;
  int j = 0;
  for (; j + 8 <= n; j += 8) {
    double av[8], xv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      av[q] = __ldg(col + (int64_t)(j + q) * n);
      xv[q] = __ldg(x + j + q);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = dadd(acc, dmul(av[q], xv[q]));
  }
  for (; j < n; ++j) acc = dadd(acc, dmul(__ldg(col + (int64_t)j * n), x[j]));
  y[i] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p,
                                cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static int matvec_impl(double *y, const double *a, const double *x, int n,
                       const lfb_launch *geom, cudaStream_t s) {
  const bool tma_ok = (n % 2 == 0) && n >= MV_JT && aligned(a, 16) &&
                      aligned(x, 16) && !(geom && geom->variant == 1);
  if (tma_ok) {
    auto encode = encode_fn();
    if (!encode)
      return fail(LFB_ERR_LAUNCH, "matvec: cuTensorMapEncodeTiled missing");
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)n * 8};
    cuuint32_t box[2] = {MV_ROWS, MV_JT};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                        const_cast<double *>(a), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(LFB_ERR_LAUNCH, "matvec: tensor map encode failed (%d)",
                  (int)r);
    const int grid = (n + MV_ROWS - 1) / MV_ROWS;
    const int var = geom ? geom->variant : 0;
    if ((var == 0 || var == 2) && n >= MVS_W * MV_JT) {
      cudaFuncSetAttribute(matvec_split_kernel,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)MvsSmem::total);
      matvec_split_kernel<<<grid, 32 * (MVS_W + 1), MvsSmem::total, s>>>(
          tm, y, x, n);
      return check_launch("lfb_matvec_f64");
    }
    // bitwise TMA kernel: 32-row panels (variant 3 / default for n < 256);
    // variant 4: 28-row panels (147 CTAs at n = 4096, measured 3 % slower)
    const bool r32 = !(geom && geom->variant == 4);
    if (!r32) {
      CUtensorMap tm28;
      cuuint32_t box28[2] = {28, MV_JT};
      if (encode(&tm28, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                 const_cast<double *>(a), dims, strides, box28, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(LFB_ERR_LAUNCH, "matvec: tensor map encode failed");
      cudaFuncSetAttribute(matvec_tma_kernel<28>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)MvSmem::total);
      matvec_tma_kernel<28><<<(n + 27) / 28, 64, MvSmem::total, s>>>(
          tm28, y, x, n);
      return check_launch("lfb_matvec_f64");
    }
    cudaFuncSetAttribute(matvec_tma_kernel<32>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)MvSmem::total);
    matvec_tma_kernel<32><<<grid, 64, MvSmem::total, s>>>(tm, y, x, n);
  } else {
    matvec_direct_kernel<<<(n + 127) / 128, 128, 0, s>>>(y, a, x, n);
  }
  return check_launch("lfb_matvec_f64");
}

}  // namespace lfb

extern "C" int lfb_matvec_f64(double *y, const double *a, const double *x,
                              int n, const lfb_launch *geom,
                              lfb_stream stream) {
  if (n < 0) return lfb::fail(LFB_ERR_ARG, "lfb_matvec_f64: n < 0");
  if (n == 0) return LFB_OK;
  if (!y || !a || !x)
    return lfb::fail(LFB_ERR_ARG, "lfb_matvec_f64: null array");
  if (geom && geom->abi_version != LFB_ABI_VERSION)
    return lfb::fail(LFB_ERR_ARG, "lfb_matvec_f64: bad lfb_launch version");
  if (geom && geom->group_extent[0] > 0 &&
      geom->group_extent[0] * (int64_t)geom->local_extent[0] < n)
    return lfb::fail(LFB_ERR_ARG,
                     "lfb_matvec_f64: launch geometry covers fewer than n "
                     "rows");
  return lfb::matvec_impl(y, a, x, n, geom, (cudaStream_t)stream);
}
