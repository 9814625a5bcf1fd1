// Tensor-product spectral-element Laplacian (BASELINE configs 3/4/5).
//
// Reference arithmetic: the Fortran fixture of SURVEY.md Appendix A
// (paper_1503_07659_b200/fixtures.py: semlap_source) lowered by
// fortran.py:667 and executed by interp.py:323-400 / emitted by
// codegen.py:767.  Per element e, with n points per direction and
// column-major layouts u,w[i + n j + n^2 k + n^3 e], d[a + n b] = d(a,b),
// g[c + 6(i + n j + n^2 k) + 6 n^3 e]:
//
//   phase 1, every point (i,j,k):
//     ur = 0; us = 0; ut = 0
//     for l ascending: ur = ur + d(i,l)*u(l,j,k)
//                      us = us + d(j,l)*u(i,l,k)
//                      ut = ut + d(k,l)*u(i,j,l)
//     wr = (g0*ur + g1*us) + g2*ut
//     ws = (g1*ur + g3*us) + g4*ut
//     wt = (g2*ur + g4*us) + g5*ut
//   phase 2, every point (i,j,k):
//     s = 0
//     for l ascending: s = ((s + d(l,i)*wr(l,j,k)) + d(l,j)*ws(i,l,k))
//                          + d(l,k)*wt(i,j,l)
//     w(i,j,k) = s
//
// every * and + rounded separately (no FMA), so the device result is bitwise
// the reference's.  Elements are independent.
//
// B200 design:
//  * persistent CTAs, one per SM, each owning a contiguous element range;
//  * G "element groups" of n^2 threads (rounded up to whole warps) per CTA,
//    thread (i,j) of a group owns the k-column of points (i,j,*);
//  * each group has a private ring of SG smem stages; a stage holds one
//    element's u (n^3 doubles) and g (6 n^3 doubles), filled by two 1-D bulk
//    copies on the TMA engine (cp.async.bulk + mbarrier complete_tx) issued
//    SG elements ahead, so HBM streams while the FP64 pipe works;
//  * the thread's own u column and wt column live in registers, d lives in
//    registers (n <= 8) or smem, wr/ws go through a padded per-group smem
//    scratch (row stride n+2 keeps 16-byte pairs aligned and the 4 j-rows of
//    a warp on distinct banks) between the two phases;
//  * w is stored straight from registers (each warp writes 256 contiguous
//    bytes per k plane);
//  * optional fused epilogue: per-CTA sum(w*w) partials (fixed order, so the
//    norm is deterministic) for the multi-GPU verification allreduce.
#include "lfb_common.cuh"

namespace lfb {

template <int N>
struct SemCfg {
  static constexpr int NP = N * N * N;
  static constexpr int T = ((N * N + 31) / 32) * 32;
  static constexpr int R = (N % 2 == 0) ? N + 2 : N + 1;
  static constexpr int SCR = R * N * N;
  static constexpr bool DREG = N <= 8;
  static constexpr int STAGE = 7 * NP;  // doubles: u then g
};

template <int N, int G, int SG>
struct SemSmem {
  using C = SemCfg<N>;
  static constexpr size_t bars = 128;  // up to 16 mbarriers
  static constexpr size_t d_off = bars;
  static constexpr size_t scr_off = d_off + 2 * N * N * 8;
  static constexpr size_t stage_off =
      ((scr_off + (size_t)G * 2 * C::SCR * 8) + 127) / 128 * 128;
  static constexpr size_t total = stage_off + (size_t)G * SG * C::STAGE * 8;
};

template <int N, int G, int SG, bool SUMSQ>
__global__ void __launch_bounds__(G *SemCfg<N>::T, 1)
    semlap_kernel(double *__restrict__ w, const double *__restrict__ u,
                  const double *__restrict__ d, const double *__restrict__ g,
                  int64_t nelt, double *__restrict__ partials) {
  using C = SemCfg<N>;
  using L = SemSmem<N, G, SG>;
  constexpr int NP = C::NP;
  constexpr int T = C::T;
  constexpr int R = C::R;
  static_assert(G * SG <= 16, "too many stages");
  static_assert((NP * 8) % 16 == 0, "bulk copies need 16-byte sizes");

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem);
  double *dn = reinterpret_cast<double *>(smem + L::d_off);  // d(a,b) at a+N b
  double *dt = dn + N * N;                                   // d(b,a) at a+N b
  double *scr = reinterpret_cast<double *>(smem + L::scr_off);
  double *stages = reinterpret_cast<double *>(smem + L::stage_off);

  const int tid = threadIdx.x;
  const int grp = tid / T;
  const int lt = tid % T;
  const int i = lt % N;
  const int j = lt / N;
  const bool active = lt < N * N;

  const int64_t begin = (nelt * blockIdx.x) / gridDim.x;
  const int64_t end = (nelt * (blockIdx.x + 1)) / gridDim.x;
  const int64_t count = end - begin;

  if (tid == 0) {
    for (int s = 0; s < G * SG; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const uint64_t pol = policy_evict_first();
  auto issue = [&](int st, int64_t e) {
    double *dst = stages + (size_t)st * C::STAGE;
    mbar_arrive_expect_tx(&bars[st], (uint32_t)(C::STAGE * 8));
    bulk_g2s_stream(dst, u + e * NP, NP * 8, &bars[st], pol);
    bulk_g2s_stream(dst + NP, g + e * 6 * NP, 6 * NP * 8, &bars[st], pol);
  };

  // prologue: each group leader fills its ring
  if (lt == 0) {
    for (int m = 0; m < SG; ++m) {
      int64_t t = grp + (int64_t)G * m;
      if (t < count) issue(grp * SG + m, begin + t);
    }
  }

  // d: natural and transposed copies (plain loads; 8 n^2 bytes per CTA)
  for (int q = tid; q < N * N; q += G * T) {
    double v = d[q];
    dn[q] = v;
    dt[(q / N) + N * (q % N)] = v;
  }
  __syncthreads();

  // per-thread d rows/columns (phase 1: d(i,l), d(j,l); phase 2: d(l,i), d(l,j))
  double d_il[C::DREG ? N : 1], d_jl[C::DREG ? N : 1];
  double d_li[C::DREG ? N : 1], d_lj[C::DREG ? N : 1];
  if constexpr (C::DREG) {
#pragma unroll
    for (int l = 0; l < N; ++l) {
      d_il[l] = dn[i + N * l];
      d_jl[l] = dn[j + N * l];
      d_li[l] = dn[l + N * i];
      d_lj[l] = dn[l + N * j];
    }
  }
  auto D_il = [&](int l) { if constexpr (C::DREG) return d_il[l]; else return dn[i + N * l]; };
  auto D_jl = [&](int l) { if constexpr (C::DREG) return d_jl[l]; else return dn[j + N * l]; };
  auto D_li = [&](int l) { if constexpr (C::DREG) return d_li[l]; else return dn[l + N * i]; };
  auto D_lj = [&](int l) { if constexpr (C::DREG) return d_lj[l]; else return dn[l + N * j]; };

  double *scr_r = scr + (size_t)grp * 2 * C::SCR;
  double *scr_s = scr_r + C::SCR;
  double acc = 0.0;

  for (int m = 0;; ++m) {
    const int64_t t = grp + (int64_t)G * m;
    if (t >= count) break;
    const int st = grp * SG + (m % SG);
    mbar_wait(&bars[st], (uint32_t)((m / SG) & 1));
    const double *su = stages + (size_t)st * C::STAGE;
    const double *sg = su + NP;

    double wt[N];
    if (active) {
      double ucol[N];
#pragma unroll
      for (int l = 0; l < N; ++l) ucol[l] = su[i + N * j + N * N * l];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double ur = 0.0, us = 0.0, ut = 0.0;
        const double *row = su + N * j + N * N * k;      // u(.,j,k)
        const double *col = su + i + N * N * k;          // u(i,.,k), stride N
        const double *dk = dt + N * k;                   // d(k,.)
#pragma unroll
        for (int l = 0; l < N; l += 2) {
          const double2 r2 = *reinterpret_cast<const double2 *>(row + l);
          const double2 k2 = *reinterpret_cast<const double2 *>(dk + l);
          ur = dadd(ur, dmul(D_il(l), r2.x));
          us = dadd(us, dmul(D_jl(l), col[N * l]));
          ut = dadd(ut, dmul(k2.x, ucol[l]));
          ur = dadd(ur, dmul(D_il(l + 1), r2.y));
          us = dadd(us, dmul(D_jl(l + 1), col[N * (l + 1)]));
          ut = dadd(ut, dmul(k2.y, ucol[l + 1]));
        }
        const double2 *gp =
            reinterpret_cast<const double2 *>(sg + 6 * (i + N * j + N * N * k));
        const double2 g01 = gp[0], g23 = gp[1], g45 = gp[2];
        const double wr = dadd(dadd(dmul(g01.x, ur), dmul(g01.y, us)), dmul(g23.x, ut));
        const double ws = dadd(dadd(dmul(g01.y, ur), dmul(g23.y, us)), dmul(g45.x, ut));
        wt[k] = dadd(dadd(dmul(g23.x, ur), dmul(g45.x, us)), dmul(g45.y, ut));
        scr_r[i + R * j + R * N * k] = wr;
        scr_s[i + R * j + R * N * k] = ws;
      }
    }
    named_bar_sync(1 + grp, T);  // stage consumed, scratch complete

    if (lt == 0) {
      const int64_t tn = t + (int64_t)G * SG;
      if (tn < count) {
        fence_proxy_async_smem();
        issue(st, begin + tn);
      }
    }

    if (active) {
      double *we = w + (begin + t) * NP + i + N * j;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
        const double *rr = scr_r + R * j + R * N * k;    // wr(.,j,k)
        const double *rs = scr_s + i + R * N * k;        // ws(i,.,k), stride R
        const double *dk = dn + N * k;                   // d(.,k)
#pragma unroll
        for (int l = 0; l < N; l += 2) {
          const double2 r2 = *reinterpret_cast<const double2 *>(rr + l);
          const double2 k2 = *reinterpret_cast<const double2 *>(dk + l);
          s = dadd(dadd(dadd(s, dmul(D_li(l), r2.x)), dmul(D_lj(l), rs[R * l])),
                   dmul(k2.x, wt[l]));
          s = dadd(dadd(dadd(s, dmul(D_li(l + 1), r2.y)),
                        dmul(D_lj(l + 1), rs[R * (l + 1)])),
                   dmul(k2.y, wt[l + 1]));
        }
        we[N * N * k] = s;
        if constexpr (SUMSQ) acc = dadd(acc, dmul(s, s));
      }
    }
    named_bar_sync(1 + grp, T);  // scratch reads done before the next phase 1
  }

  if constexpr (SUMSQ) {
    // fixed-order block reduction -> partials[blockIdx.x]
    __shared__ double red[32];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
      acc = dadd(acc, __shfl_down_sync(0xffffffffu, acc, off));
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double sum = 0.0;
      for (int q = 0; q < (G * T) / 32; ++q) sum = dadd(sum, red[q]);
      partials[blockIdx.x] = sum;
    }
  }
}

__global__ void sum_partials_kernel(const double *__restrict__ partials, int n,
                                    double *__restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < n; ++q) s = dadd(s, partials[q]);
    *out = s;
  }
}

struct SemLaunch {
  int grid, block;
  size_t smem;
};

template <int N, int G, int SG>
static int launch_sem(double *w, const double *u, const double *d,
                      const double *g, int64_t nelt, const lfb_launch *geom,
                      cudaStream_t s) {
  using L = SemSmem<N, G, SG>;
  const int block = G * SemCfg<N>::T;
  const size_t smem = L::total;
  int sms = sm_count(geom);
  if (sms <= 0) return fail(LFB_ERR_LAUNCH, "semlap: cannot query SM count");
  int per_sm = (geom && geom->ctas_per_sm > 0) ? geom->ctas_per_sm : 1;
  int64_t grid64 = (int64_t)sms * per_sm;
  int64_t min_per_cta = G;  // keep every group busy
  if (grid64 * min_per_cta > nelt)
    grid64 = (nelt + min_per_cta - 1) / min_per_cta;
  if (grid64 < 1) grid64 = 1;
  const int grid = (int)grid64;
  const bool sumsq = geom && geom->sumsq;
  if (sumsq && (!geom->workspace || geom->workspace_len < grid))
    return fail(LFB_ERR_ARG,
                "semlap: sumsq requested with workspace of %lld < %d doubles",
                (long long)(geom->workspace ? geom->workspace_len : 0), grid);
  if (sumsq) {
    auto k = semlap_kernel<N, G, SG, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    k<<<grid, block, smem, s>>>(w, u, d, g, nelt, geom->workspace);
    if (int rc = check_launch("lfb_semlap_f64")) return rc;
    sum_partials_kernel<<<1, 32, 0, s>>>(geom->workspace, grid, geom->sumsq);
  } else {
    auto k = semlap_kernel<N, G, SG, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    k<<<grid, block, smem, s>>>(w, u, d, g, nelt, nullptr);
  }
  return check_launch("lfb_semlap_f64");
}

template <int N, int G, int SG>
static int64_t sem_grid(int64_t nelt, const lfb_launch *geom) {
  int sms = sm_count(geom);
  if (sms <= 0) sms = 148;
  int per_sm = (geom && geom->ctas_per_sm > 0) ? geom->ctas_per_sm : 1;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid * G > nelt) grid = (nelt + G - 1) / G;
  return grid < 1 ? 1 : grid;
}

// {{{ dispatch on the order (n = points per direction) and tuning variant

#define LFB_SEM_CASES(X)        \
  X(2, 4, 3, 0) X(4, 4, 3, 0)   \
  X(6, 4, 3, 0) X(8, 3, 2, 0)   \
  X(8, 2, 3, 1) X(8, 4, 1, 2)   \
  X(8, 5, 1, 3) X(10, 2, 1, 0)

static int sem_dispatch(double *w, const double *u, const double *d,
                        const double *g, int64_t nelt, const lfb_launch *geom,
                        cudaStream_t s, int64_t *grid_out) {
  const int n = geom->npts;
  const int var = geom->variant;
#define X(NN, GG, SS, VV)                                                   \
  if (n == NN && var == VV) {                                               \
    if (grid_out) {                                                         \
      *grid_out = sem_grid<NN, GG, SS>(nelt, geom);                         \
      return LFB_OK;                                                        \
    }                                                                       \
    return launch_sem<NN, GG, SS>(w, u, d, g, nelt, geom, s);               \
  }
  LFB_SEM_CASES(X)
#undef X
  return fail(LFB_ERR_UNSUPPORTED,
              "semlap: no sm_100a kernel for n=%d points per direction "
              "(variant %d); built orders: n = 2, 4, 6, 8, 10",
              n, var);
}

// }}}

}  // namespace lfb

extern "C" {

int lfb_semlap_f64(double *w, const double *u, const double *d,
                   const double *g, int nelt, const lfb_launch *geom,
                   lfb_stream stream) {
  if (!geom || geom->abi_version != LFB_ABI_VERSION)
    return lfb::fail(LFB_ERR_ARG,
                     "lfb_semlap_f64: an lfb_launch with npts is required");
  if (nelt < 0) return lfb::fail(LFB_ERR_ARG, "lfb_semlap_f64: nelt < 0");
  if (geom->group_extent[0] > 0 &&
      geom->group_extent[0] * (int64_t)geom->local_extent[0] < nelt)
    return lfb::fail(LFB_ERR_ARG,
                     "lfb_semlap_f64: launch geometry covers %lld of %d "
                     "elements",
                     (long long)(geom->group_extent[0] *
                                 (int64_t)geom->local_extent[0]),
                     nelt);
  if (nelt == 0) {
    if (geom->sumsq)
      cudaMemsetAsync(geom->sumsq, 0, sizeof(double), (cudaStream_t)stream);
    return lfb::check_launch("lfb_semlap_f64");
  }
  if (!w || !u || !d || !g)
    return lfb::fail(LFB_ERR_ARG, "lfb_semlap_f64: null array");
  if (!lfb::aligned(u, 16) || !lfb::aligned(g, 16) || !lfb::aligned(w, 16))
    return lfb::fail(LFB_ERR_UNSUPPORTED,
                     "lfb_semlap_f64: u, g and w must be 16-byte aligned");
  return lfb::sem_dispatch(w, u, d, g, nelt, geom, (cudaStream_t)stream,
                           nullptr);
}

int64_t lfb_semlap_workspace(int npts, int nelt, const lfb_launch *geom) {
  lfb_launch tmp{};
  if (geom) tmp = *geom;
  tmp.abi_version = LFB_ABI_VERSION;
  tmp.npts = npts;
  int64_t grid = 0;
  if (lfb::sem_dispatch(nullptr, nullptr, nullptr, nullptr, nelt, &tmp,
                        nullptr, &grid))
    return -1;
  return grid;
}

}  // extern "C"
