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
//  * wr/ws: padded smem scratch (row stride n+2 for even n so wr rows load
//    as 16-byte pairs, n+1 for odd n), wt and the u column in registers;
//    the broadcast d(k,l) / d(l,k) are constant-bank operands (dconst.cuh),
//    the per-thread d rows come from smem or registers (DREG).
#include "dconst.cuh"
#include "lfb_common.cuh"
#include "semlap_common.cuh"

namespace lfb {

// d(a,b) at c_dslab[N][a + N b] for the order being launched (dconst.cuh)
__constant__ double c_dslab[17][256];

template <int N>
__device__ __forceinline__ void slab_pair(const double *p, double &a,
                                          double &b) {
  if constexpr (N % 2 == 0) {
    const double2 v = *reinterpret_cast<const double2 *>(p);
    a = v.x, b = v.y;
  } else {
    a = p[0], b = p[1];
  }
}

template <int N>
struct SlabCfg {
  static constexpr int N2 = N * N;
  static constexpr int NP = N * N * N;
  static constexpr int T = ((N2 + 31) / 32) * 32;
  static constexpr int R = (N % 2 == 0) ? N + 2 : N + 1;  // even: pairs
  static constexpr int SCR = R * N * N;
  static constexpr int UST = (NP + 2 + 1) / 2 * 2;  // + 8-byte lead, even
  static constexpr int SLAB = 6 * N2;
};

template <int N, int G, int SGS, int KS>
struct SlabSmem {
  using C = SlabCfg<N>;
  static constexpr size_t bars = 256;  // G * (2 + SGS) <= 32 mbarriers
  static constexpr size_t d_off = bars;
  static constexpr size_t grp_off = (d_off + 2 * N * N * 8 + 127) / 128 * 128;
  static constexpr size_t grp_bytes =
      ((2 * (size_t)C::UST + (size_t)SGS * KS * C::SLAB + 2 * (size_t)C::SCR) *
           8 +
       127) / 128 * 128;
  static constexpr size_t total = grp_off + G * grp_bytes;
};

// KS consecutive k-slices of g per bulk copy (one ring slot), N / KS copies
// per element (the last one shorter when KS does not divide N).  Both phases
// are fully unrolled over k and l, so the n independent accumulation chains
// of a thread's column overlap in the FP64 pipe.
template <int N, int G, int SGS, int KS, bool DREG, bool SUMSQ, bool F>
__global__ void __launch_bounds__(G *SlabCfg<N>::T, 1)
    semlap_slab_kernel(double *__restrict__ w, const double *__restrict__ u,
                       const double *__restrict__ d,
                       const double *__restrict__ g, int64_t nelt,
                       double *__restrict__ partials) {
  using C = SlabCfg<N>;
  using L = SlabSmem<N, G, SGS, KS>;
  constexpr int NP = C::NP, N2 = C::N2, T = C::T, R = C::R;
  constexpr int STEPS = (N + KS - 1) / KS;  // slab copies per element
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
  double *slabs = ustage + 2 * C::UST;                     // SGS x KS x SLAB
  double *scr_r = slabs + SGS * KS * C::SLAB;              // SCR
  double *scr_s = scr_r + C::SCR;                          // SCR
  uint64_t *ubar = bars + grp * (2 + SGS);
  uint64_t *gbar = ubar + 2;

  // interleaved: group q0 = blockIdx.x * G + grp takes elements q0, q0 + Q..
  const int64_t q0 = (int64_t)blockIdx.x * G + grp;
  const int64_t Q = (int64_t)gridDim.x * G;
  const int64_t mine = nelt > q0 ? (nelt - q0 + Q - 1) / Q : 0;
  auto elem = [&](int64_t m) -> int64_t { return q0 + m * Q; };

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
    const int64_t e = elem(m);
    const int st = (int)(m & 1);
    if (u_bulk_ok(e)) {
      mbar_arrive_expect_tx(&ubar[st], (uint32_t)u_span(e));
      bulk_g2s_stream(ustage + st * C::UST, u + e * NP - u_lead(e),
                      (uint32_t)u_span(e), &ubar[st], pol);
    } else {
      mbar_arrive_expect_tx(&ubar[st], 0);  // threads copy it themselves
    }
  };
  auto issue_slab = [&](int64_t q) {  // q = m * STEPS + step
    const int64_t m = q / STEPS;
    const int step = (int)(q % STEPS);
    const int k0 = step * KS;
    const int nk = (N - k0) < KS ? (N - k0) : KS;
    const int64_t e = elem(m);
    const int slot = (int)(q % SGS);
    mbar_arrive_expect_tx(&gbar[slot], (uint32_t)(nk * C::SLAB * 8));
    bulk_g2s_stream(slabs + (size_t)slot * KS * C::SLAB,
                    g + e * 6 * NP + (int64_t)k0 * 6 * N2, nk * C::SLAB * 8,
                    &gbar[slot], pol);
  };

  const int64_t nsteps = mine * STEPS;
  if (lt == 0) {
    for (int64_t m = 0; m < 2 && m < mine; ++m) issue_u(m);
    for (int64_t q = 0; q < SGS && q < nsteps; ++q) issue_slab(q);
  }
  for (int q = tid; q < N2; q += G * T) {
    const double v = d[q];
    dn[q] = v;
    dt[(q / N) + N * (q % N)] = v;
  }
  __syncthreads();

  double acc = 0.0;
  for (int64_t m = 0; m < mine; ++m) {
    const int64_t e = elem(m);
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
    double da[N], db[N];  // d(i,.), d(j,.) (DREG)
    if (active) {
#pragma unroll
      for (int l = 0; l < N; ++l) ucol[l] = su[i + N * j + N2 * l];
      if constexpr (DREG) {
#pragma unroll
        for (int l = 0; l < N; ++l) da[l] = dn[i + N * l], db[l] = dn[j + N * l];
      }
    }
#pragma unroll
    for (int step = 0; step < STEPS; ++step) {
      const int64_t q = m * STEPS + step;
      const int slot = (int)(q % SGS);
      mbar_wait(&gbar[slot], (uint32_t)((q / SGS) & 1));
      if (active) {
        const double *gs = slabs + (size_t)slot * KS * C::SLAB;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = step * KS + kk;
          if (k < N) {
            double ur = 0.0, us = 0.0, ut = 0.0;
            const double *row = su + N * j + N2 * k;
            const double *col = su + i + N2 * k;
#pragma unroll
            for (int l = 0; l < N; l += 2) {
              double r0, r1 = 0.0;
              if (l + 1 < N) slab_pair<N>(row + l, r0, r1);
              else r0 = row[l];
#pragma unroll
              for (int h = 0; h < 2 && l + h < N; ++h) {
                const int ll = l + h;
                const double a = DREG ? da[ll] : dn[i + N * ll];
                const double b = DREG ? db[ll] : dn[j + N * ll];
                ur = mac<F>(ur, a, h ? r1 : r0);
                us = mac<F>(us, b, col[N * ll]);
                // d(k,l): from the constant bank (uniform load)
                ut = mac<F>(ut, c_dslab[N][k + N * ll], ucol[ll]);
              }
            }
            const double *gp = gs + kk * C::SLAB + 6 * (i + N * j);
            const double2 g01 = *reinterpret_cast<const double2 *>(gp);
            const double2 g23 = *reinterpret_cast<const double2 *>(gp + 2);
            const double2 g45 = *reinterpret_cast<const double2 *>(gp + 4);
            scr_r[i + R * j + R * N * k] =
                comb3<F>(g01.x, ur, g01.y, us, g23.x, ut);
            scr_s[i + R * j + R * N * k] =
                comb3<F>(g01.y, ur, g23.y, us, g45.x, ut);
            wt[k] = comb3<F>(g23.x, ur, g45.x, us, g45.y, ut);
          }
        }
      }
      named_bar_sync(1 + grp, T);  // slot consumed (and, last step, u)
      if (lt == 0) {
        if (q + SGS < nsteps) {
          fence_proxy_async_smem();
          issue_slab(q + SGS);
        }
        if (step == STEPS - 1 && m + 2 < mine) {
          fence_proxy_async_smem();
          issue_u(m + 2);
        }
      }
    }

    if (active) {
      if constexpr (DREG) {
#pragma unroll
        for (int l = 0; l < N; ++l) da[l] = dt[i + N * l], db[l] = dt[j + N * l];
      }
      double *we = w + e * NP + i + N * j;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
        const double *rr = scr_r + R * j + R * N * k;  // wr(., j, k)
        const double *rs = scr_s + i + R * N * k;      // ws(i, ., k)
#pragma unroll
        for (int l = 0; l < N; l += 2) {
          double r0, r1 = 0.0;
          if (l + 1 < N) slab_pair<N>(rr + l, r0, r1);
          else r0 = rr[l];
#pragma unroll
          for (int h = 0; h < 2 && l + h < N; ++h) {
            const int ll = l + h;
            const double a = DREG ? da[ll] : dt[i + N * ll];
            const double b = DREG ? db[ll] : dt[j + N * ll];
            s = mac<F>(mac<F>(mac<F>(s, a, h ? r1 : r0), b, rs[R * ll]),
                       c_dslab[N][ll + N * k], wt[ll]);  // d(l,k)
          }
        }
        we[N2 * k] = s;
        if constexpr (SUMSQ) acc = dadd(acc, dmul(s, s));
      }
    }
    named_bar_sync(1 + grp, T);  // scratch reads done
  }

  if constexpr (SUMSQ) block_sumsq_partial(acc, partials);
}

template <int N, int G, int SGS, int KS, bool DREG, bool F>
int launch_sem_slab(double *w, const double *u, const double *d,
                    const double *g, int64_t nelt, const lfb_launch *geom,
                    cudaStream_t s, int64_t *grid_out) {
  using L = SlabSmem<N, G, SGS, KS>;
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
  auto k = sumsq ? semlap_slab_kernel<N, G, SGS, KS, DREG, true, F>
                 : semlap_slab_kernel<N, G, SGS, KS, DREG, false, F>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)L::total);
  {
    std::unique_lock<std::mutex> lk;
    bool capturing = false;
    int slot = N;  // one constant slot per order
    if (int rc = dconst_acquire(c_dslab, 256 * 8, 2, &slot, d, N, s, &lk,
                                &capturing))
      return rc;
    k<<<grid, block, L::total, s>>>(w, u, d, g, nelt,
                                    sumsq ? geom->workspace : nullptr);
    dconst_release(2, slot, s, capturing);
  }
  if (int rc = check_launch("lfb_semlap_f64")) return rc;
  return sumsq ? sem_sumsq_finish(geom->workspace, grid, geom->sumsq, s)
               : LFB_OK;
}

// (n, variant) -> (groups per CTA, ring depth, slices per copy, d in regs)
// variant 0 / 9: default; 30..: tuning alternatives (n >= 12)
#define LFB_SLAB_TABLE(X)       \
  X(2, 0, 4, 4, 1, false)       \
  X(3, 0, 4, 4, 1, false)       \
  X(4, 0, 4, 4, 1, false)       \
  X(5, 0, 4, 4, 1, false)       \
  X(6, 0, 4, 4, 1, false)       \
  X(7, 0, 3, 4, 1, false)       \
  X(8, 0, 3, 4, 1, false)       \
  X(9, 0, 4, 4, 1, false)       \
  X(10, 0, 4, 4, 1, false)      \
  X(11, 0, 3, 4, 1, false)      \
  X(12, 0, 2, 3, 2, true)       \
  X(12, 30, 2, 4, 1, false)     \
  X(12, 31, 3, 2, 1, false)     \
  X(13, 0, 2, 4, 1, true)       \
  X(13, 31, 2, 4, 1, false)      \
  X(14, 0, 1, 4, 2, true)       \
  X(14, 30, 1, 4, 1, false)     \
  X(14, 31, 1, 3, 2, false)     \
  X(15, 0, 1, 3, 2, false)      \
  X(15, 30, 1, 4, 1, false)     \
  X(16, 0, 1, 2, 3, false)      \
  X(16, 30, 1, 3, 1, false)     \
  X(16, 31, 1, 3, 2, false)

int sem_slab_dispatch(int n, int variant, double *w, const double *u,
                      const double *d, const double *g, int64_t nelt,
                      const lfb_launch *geom, cudaStream_t s,
                      int64_t *grid_out) {
  const int v = variant == 9 ? 0 : variant;
#define X(NN, VV, GG, SS, KK, DR)                                         \
  if (n == NN && v == VV)                                                 \
    return launch_sem_slab<NN, GG, SS, KK, DR, false>(w, u, d, g, nelt,   \
                                                      geom, s, grid_out); \
  if (VV == 0 && n == NN && v == 50 && n >= 12) /* FMA mode */           \
    return launch_sem_slab<NN, GG, SS, KK, DR, VV == 0 && NN >= 12>(      \
        w, u, d, g, nelt, geom, s, grid_out);
  LFB_SLAB_TABLE(X)
#undef X
  return fail(LFB_ERR_UNSUPPORTED,
              "semlap: no sm_100a kernel variant %d for n=%d points per "
              "direction (supported n = 2..16)",
              variant, n);
}

}  // namespace lfb
