// SEM Laplacian, any order: g streamed in k-slabs (BASELINE config 5 sweep).
//
// Same reference arithmetic as semlap.cu (every * and +
// rounded separately, l ascending), for the orders the staged kernel cannot
// hold: odd n (an element's u is not 16-byte aligned for odd e, and bulk
// copies need 16-byte granules) and n >= 12 (u + g of one element exceed a
// sensible smem stage: 189 KB at n = 15, 229 KB at n = 16).
//
// Per element group (n^2 threads rounded up to warps, thread (i,j) owns the
// k-column as in semlap.cu):
//  * u: double-buffered whole-element stage, one bulk copy per element,
//    issued one element ahead.  For odd n the copy starts at the 16-byte
//    boundary below the element and lands 8 bytes early in smem (the element
//    is read at offset uoff); only a final element whose rounded end would
//    run past the array is copied by the threads themselves.
//  * g: the phase-1 combine at slab k needs only g(:, :, :, k) = 6 n^2
//    doubles (48 n^2 bytes, always 16-byte aligned), streamed through an
//    SGS-deep slab ring, one bulk copy per slab, issued SGS slabs ahead.
//  * wr/ws: padded smem scratch (row stride n+1), wt and the u column in
//    registers, d from smem.
#include "lfb_common.cuh"
#include "semlap_common.cuh"

namespace lfb {

template <int N>
struct SlabCfg {
  static constexpr int N2 = N * N;
  static constexpr int NP = N * N * N;
  static constexpr int T = ((N2 + 31) / 32) * 32;
  static constexpr int R = N + 1;
  static constexpr int SCR = R * N * N;
  static constexpr int UST = (NP + 2 + 1) / 2 * 2;  // + 8-byte lead, even
  static constexpr int SLAB = 6 * N2;
};

template <int N, int G, int SGS>
struct SlabSmem {
  using C = SlabCfg<N>;
  static constexpr size_t bars = 256;  // G * (2 + SGS) <= 32 mbarriers
  static constexpr size_t d_off = bars;
  static constexpr size_t grp_off = (d_off + 2 * N * N * 8 + 127) / 128 * 128;
  static constexpr size_t grp_bytes =
      ((2 * (size_t)C::UST + (size_t)SGS * C::SLAB + 2 * (size_t)C::SCR) * 8 +
       127) / 128 * 128;
  static constexpr size_t total = grp_off + G * grp_bytes;
};

template <int N, int G, int SGS, bool SUMSQ>
__global__ void __launch_bounds__(G *SlabCfg<N>::T, 1)
    semlap_slab_kernel(double *__restrict__ w, const double *__restrict__ u,
                       const double *__restrict__ d,
                       const double *__restrict__ g, int64_t nelt,
                       double *__restrict__ partials) {
  using C = SlabCfg<N>;
  using L = SlabSmem<N, G, SGS>;
  constexpr int NP = C::NP, N2 = C::N2, T = C::T, R = C::R;
  static_assert(G * (2 + SGS) <= 32, "too many mbarriers");

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem);
  double *dn = reinterpret_cast<double *>(smem + L::d_off);
  double *dt = dn + N2;

  const int tid = threadIdx.x;
  const int grp = tid / T;
  const int lt = tid % T;
  const int i = lt % N;
  const int j = lt / N;
  const bool active = lt < N2;

  unsigned char *gbase = smem + L::grp_off + (size_t)grp * L::grp_bytes;
  double *ustage = reinterpret_cast<double *>(gbase);      // 2 x UST
  double *slabs = ustage + 2 * C::UST;                     // SGS x SLAB
  double *scr_r = slabs + SGS * C::SLAB;                   // SCR
  double *scr_s = scr_r + C::SCR;                          // SCR
  uint64_t *ubar = bars + grp * (2 + SGS);
  uint64_t *gbar = ubar + 2;

  const int64_t begin = (nelt * blockIdx.x) / gridDim.x;
  const int64_t end = (nelt * (blockIdx.x + 1)) / gridDim.x;
  const int64_t count = end - begin;
  // group grp handles CTA-local elements grp, grp + G, ...
  const int64_t mine = count > grp ? (count - grp + G - 1) / G : 0;

  if (tid == 0) {
    for (int q = 0; q < G * (2 + SGS); ++q) mbar_init(&bars[q], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const uint64_t pol = policy_evict_first();
  const int64_t u_bytes_total = nelt * NP * 8;

  // u of element e: 16-byte aligned superset, or a thread copy at the tail
  auto u_lead = [&](int64_t e) -> int { return (int)((e * NP) & 1); };
  auto u_span = [&](int64_t e) -> int64_t {
    return ((int64_t)(u_lead(e) + NP) * 8 + 15) / 16 * 16;
  };
  auto u_bulk_ok = [&](int64_t e) -> bool {
    return (e * NP - u_lead(e)) * 8 + u_span(e) <= u_bytes_total;
  };
  auto issue_u = [&](int64_t m) {
    const int64_t e = begin + grp + m * G;
    const int st = (int)(m & 1);
    if (u_bulk_ok(e)) {
      mbar_arrive_expect_tx(&ubar[st], (uint32_t)u_span(e));
      bulk_g2s_stream(ustage + st * C::UST, u + e * NP - u_lead(e),
                      (uint32_t)u_span(e), &ubar[st], pol);
    } else {
      mbar_arrive_expect_tx(&ubar[st], 0);  // threads copy it themselves
    }
  };
  auto issue_slab = [&](int64_t q) {  // q = m * N + k
    const int64_t m = q / N;
    const int k = (int)(q % N);
    const int64_t e = begin + grp + m * G;
    const int slot = (int)(q % SGS);
    mbar_arrive_expect_tx(&gbar[slot], (uint32_t)(C::SLAB * 8));
    bulk_g2s_stream(slabs + (size_t)slot * C::SLAB,
                    g + e * 6 * NP + (int64_t)k * 6 * N2, C::SLAB * 8,
                    &gbar[slot], pol);
  };

  if (lt == 0) {
    for (int64_t m = 0; m < 2 && m < mine; ++m) issue_u(m);
    for (int64_t q = 0; q < SGS && q < mine * N; ++q) issue_slab(q);
  }
  for (int q = tid; q < N2; q += G * T) {
    const double v = d[q];
    dn[q] = v;
    dt[(q / N) + N * (q % N)] = v;
  }
  __syncthreads();

  double acc = 0.0;
  for (int64_t m = 0; m < mine; ++m) {
    const int64_t e = begin + grp + m * G;
    const int st = (int)(m & 1);
    mbar_wait(&ubar[st], (uint32_t)((m >> 1) & 1));
    const double *su = ustage + st * C::UST + u_lead(e);
    if (!u_bulk_ok(e)) {
      double *dst = ustage + st * C::UST + u_lead(e);
      for (int q = lt; q < NP; q += T) dst[q] = u[e * NP + q];
      named_bar_sync(1 + grp, T);
    }

    double wt[N];
    double ucol[N];
    if (active) {
#pragma unroll
      for (int l = 0; l < N; ++l) ucol[l] = su[i + N * j + N2 * l];
    }
#pragma unroll 1
    for (int k = 0; k < N; ++k) {
      const int64_t q = m * N + k;
      const int slot = (int)(q % SGS);
      mbar_wait(&gbar[slot], (uint32_t)((q / SGS) & 1));
      if (active) {
        double ur = 0.0, us = 0.0, ut = 0.0;
        const double *row = su + N * j + N2 * k;
        const double *col = su + i + N2 * k;
        const double *dk = dt + N * k;
#pragma unroll
        for (int l = 0; l < N; ++l) {
          ur = dadd(ur, dmul(dn[i + N * l], row[l]));
          us = dadd(us, dmul(dn[j + N * l], col[N * l]));
          ut = dadd(ut, dmul(dk[l], ucol[l]));
        }
        const double *gp = slabs + (size_t)slot * C::SLAB + 6 * (i + N * j);
        const double g0 = gp[0], g1 = gp[1], g2 = gp[2], g3 = gp[3],
                     g4 = gp[4], g5 = gp[5];
        scr_r[i + R * j + R * N * k] =
            dadd(dadd(dmul(g0, ur), dmul(g1, us)), dmul(g2, ut));
        scr_s[i + R * j + R * N * k] =
            dadd(dadd(dmul(g1, ur), dmul(g3, us)), dmul(g4, ut));
        const double wtk = dadd(dadd(dmul(g2, ur), dmul(g4, us)), dmul(g5, ut));
#pragma unroll
        for (int kk = 0; kk < N; ++kk)
          if (kk == k) wt[kk] = wtk;
      }
      named_bar_sync(1 + grp, T);  // slab consumed (and, at k = N-1, u)
      if (lt == 0) {
        if (q + SGS < mine * N) {
          fence_proxy_async_smem();
          issue_slab(q + SGS);
        }
        if (k == N - 1 && m + 2 < mine) {
          fence_proxy_async_smem();
          issue_u(m + 2);
        }
      }
    }

    if (active) {
      double *we = w + e * NP + i + N * j;
#pragma unroll 1
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
        const double *rr = scr_r + R * j + R * N * k;
        const double *rs = scr_s + i + R * N * k;
        const double *dk = dn + N * k;
#pragma unroll
        for (int l = 0; l < N; ++l) {
          double wtl = 0.0;
#pragma unroll
          for (int kk = 0; kk < N; ++kk)
            if (kk == l) wtl = wt[kk];
          s = dadd(dadd(dadd(s, dmul(dn[l + N * i], rr[l])),
                        dmul(dn[l + N * j], rs[R * l])),
                   dmul(dk[l], wtl));
        }
        we[N2 * k] = s;
        if constexpr (SUMSQ) acc = dadd(acc, dmul(s, s));
      }
    }
    named_bar_sync(1 + grp, T);  // scratch reads done
  }

  if constexpr (SUMSQ) block_sumsq_partial(acc, partials);
}

template <int N, int G, int SGS>
int launch_sem_slab(double *w, const double *u, const double *d,
                    const double *g, int64_t nelt, const lfb_launch *geom,
                    cudaStream_t s, int64_t *grid_out) {
  using L = SlabSmem<N, G, SGS>;
  static_assert(L::total <= 227 * 1024, "smem");
  const int block = G * SlabCfg<N>::T;
  int sms = sm_count(geom);
  if (sms <= 0) sms = 148;
  int per_sm = (geom && geom->ctas_per_sm > 0) ? geom->ctas_per_sm : 1;
  int64_t grid64 = (int64_t)sms * per_sm;
  if (grid64 * G > nelt) grid64 = (nelt + G - 1) / G;
  if (grid64 < 1) grid64 = 1;
  const int grid = (int)grid64;
  if (grid_out) {
    *grid_out = grid;
    return LFB_OK;
  }
  const bool sumsq = geom && geom->sumsq;
  if (sumsq && (!geom->workspace || geom->workspace_len < grid))
    return fail(LFB_ERR_ARG, "semlap: sumsq workspace too small");
  if (sumsq) {
    auto k = semlap_slab_kernel<N, G, SGS, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)L::total);
    k<<<grid, block, L::total, s>>>(w, u, d, g, nelt, geom->workspace);
    if (int rc = check_launch("lfb_semlap_f64")) return rc;
    return sem_sumsq_finish(geom->workspace, grid, geom->sumsq, s);
  }
  auto k = semlap_slab_kernel<N, G, SGS, false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)L::total);
  k<<<grid, block, L::total, s>>>(w, u, d, g, nelt, nullptr);
  return check_launch("lfb_semlap_f64");
}

// n -> (groups per CTA, slab ring depth) that fit 227 KB
int sem_slab_dispatch(int n, double *w, const double *u, const double *d,
                      const double *g, int64_t nelt, const lfb_launch *geom,
                      cudaStream_t s, int64_t *grid_out) {
  switch (n) {
#define LFB_SLAB(NN, GG, SS)                                              \
  case NN:                                                                \
    return launch_sem_slab<NN, GG, SS>(w, u, d, g, nelt, geom, s, grid_out);
    LFB_SLAB(2, 4, 4)
    LFB_SLAB(3, 4, 4)
    LFB_SLAB(4, 4, 4)
    LFB_SLAB(5, 4, 4)
    LFB_SLAB(6, 4, 4)
    LFB_SLAB(7, 3, 4)
    LFB_SLAB(8, 3, 4)
    LFB_SLAB(9, 4, 4)
    LFB_SLAB(10, 4, 4)
    LFB_SLAB(11, 3, 4)
    LFB_SLAB(12, 2, 4)
    LFB_SLAB(13, 2, 4)
    LFB_SLAB(14, 1, 4)
    LFB_SLAB(15, 1, 4)
    LFB_SLAB(16, 1, 3)
#undef LFB_SLAB
    default:
      return fail(LFB_ERR_UNSUPPORTED,
                  "semlap: n=%d points per direction outside 2..16", n);
  }
}

}  // namespace lfb
