// SEM Laplacian, n = 7..12: two k-columns per thread (variants 60, 61).
//
// Same arithmetic as semlap_gen.cu (variant 60 bitwise, 61 DFMA mode;
// semlap_common.cuh mac/mac0/comb3).  ncu on the one-column kernel at
// n = 9..10 (profiles/r01_sem_fma_n9.md): L1 LSU data pipe 85-94 %, stalls
// mio_throttle / short_scoreboard.  Thread (i, jj) here owns the columns
// (i, jj, *) and (i, jj + H, *), H = ceil(n/2): the u(i, ., k) column of the
// us contraction and the ws(i, ., k) column of the phase-2 sum are loaded
// once for both points (the per-lane-distinct loads that cost the most
// wavefronts), the rows u(., j, k) / wr(., j, k) once per point as before.
// About a quarter fewer shared-memory wavefronts per point.
//
// Staging as in semlap_gen.cu: E elements per chunk, u and g of a chunk by
// bulk copies into an S-deep per-group ring.
#include "dconst.cuh"
#include "lfb_common.cuh"
#include "semlap_common.cuh"

namespace lfb {

__constant__ double c_dg2[13][144];  // d(a,b) at [N][a + N b]

template <int N, int E>
struct Gen2Cfg {
  static constexpr int N2 = N * N;
  static constexpr int NP = N * N * N;
  static constexpr int H = (N + 1) / 2;      // second column: j + H
  static constexpr int PE = N * H;           // threads per element
  static constexpr int LANES = E * PE;
  static constexpr int T = ((LANES + 31) / 32) * 32;
  static constexpr int R = (N % 2 == 0) ? N + 2 : N + 1;
  static constexpr int SCR = R * N * N;
  static constexpr int GPART = 6 * E * NP;
  static constexpr int UPART = ((E * NP + 1) + 1) / 2 * 2;
  static constexpr int STAGE = GPART + UPART;
};

template <int N, int E, int G, int S>
struct Gen2Smem {
  using C = Gen2Cfg<N, E>;
  static constexpr size_t bars = ((size_t)8 * G * S + 127) / 128 * 128;
  static constexpr size_t d_off = bars;
  static constexpr size_t scr_off =
      (d_off + 2 * (size_t)C::N2 * 8 + 127) / 128 * 128;
  static constexpr size_t stage_off =
      (scr_off + (size_t)G * E * 2 * C::SCR * 8 + 127) / 128 * 128;
  static constexpr size_t total = stage_off + (size_t)G * S * C::STAGE * 8;
};

template <int N>
__device__ __forceinline__ void pair2(const double *p, double &a, double &b) {
  if constexpr (N % 2 == 0) {
    const double2 v = *reinterpret_cast<const double2 *>(p);
    a = v.x, b = v.y;
  } else {
    a = p[0], b = p[1];
  }
}

template <int N, int E, int G, int S, bool SUMSQ, bool F>
__global__ void __launch_bounds__(G *Gen2Cfg<N, E>::T, 1)
    semlap_gen2_kernel(double *__restrict__ w, const double *__restrict__ u,
                       const double *__restrict__ d,
                       const double *__restrict__ g, int64_t nelt,
                       double *__restrict__ partials) {
  using C = Gen2Cfg<N, E>;
  using L = Gen2Smem<N, E, G, S>;
  constexpr int N2 = C::N2, NP = C::NP, T = C::T, R = C::R, H = C::H;
  static_assert(G <= 15, "named barrier ids 1..15");

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem);
  double *dn = reinterpret_cast<double *>(smem + L::d_off);  // d(a,b) @ a+N b
  double *dt = dn + N2;                                      // d(b,a) @ a+N b
  double *scr = reinterpret_cast<double *>(smem + L::scr_off);
  double *stages = reinterpret_cast<double *>(smem + L::stage_off);

  const int tid = threadIdx.x;
  const int grp = tid / T;
  const int lt = tid % T;
  const int el = lt / C::PE;
  const int pt = lt % C::PE;
  const int i = pt % N;
  const int jj = pt / N;
  const int jc[2] = {jj, jj + H};
  const bool vc1 = jj + H < N;
  const int j1 = vc1 ? jj + H : jj;  // loads stay in range for odd n
  const bool lane_on = lt < C::LANES;

  const int64_t nchunks = (nelt + E - 1) / E;
  const int64_t q0 = (int64_t)blockIdx.x * G + grp;
  const int64_t Q = (int64_t)gridDim.x * G;
  const int64_t mine = nchunks > q0 ? (nchunks - q0 + Q - 1) / Q : 0;
  const int64_t u_total_bytes = nelt * NP * 8;

  auto chunk = [&](int64_t m) -> int64_t { return q0 + m * Q; };
  auto chunk_elems = [&](int64_t c) -> int {
    const int64_t r = nelt - c * E;
    return (int)(r < E ? r : E);
  };
  auto u_lead = [&](int64_t c) -> int { return (int)((c * E * NP) & 1); };
  auto u_span = [&](int64_t c) -> int64_t {
    return ((int64_t)(u_lead(c) + chunk_elems(c) * NP) * 8 + 15) / 16 * 16;
  };
  auto u_bulk_ok = [&](int64_t c) -> bool {
    return (c * E * NP - u_lead(c)) * 8 + u_span(c) <= u_total_bytes;
  };

  if (tid == 0) {
    for (int s = 0; s < G * S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const uint64_t pol = policy_evict_first();
  auto issue = [&](int st, int64_t c) {
    double *dst = stages + (size_t)st * C::STAGE;
    const int ne = chunk_elems(c);
    const uint32_t gbytes = (uint32_t)(48 * ne * NP);
    const uint32_t ubytes = u_bulk_ok(c) ? (uint32_t)u_span(c) : 0u;
    mbar_arrive_expect_tx(&bars[st], gbytes + ubytes);
    bulk_g2s_stream(dst, g + c * E * 6 * NP, gbytes, &bars[st], pol);
    if (ubytes)
      bulk_g2s_stream(dst + C::GPART, u + c * E * NP - u_lead(c), ubytes,
                      &bars[st], pol);
  };
  if (lt == 0) {
    for (int m = 0; m < S && m < mine; ++m) issue(grp * S + m, chunk(m));
  }
  for (int q = tid; q < N2; q += blockDim.x) {
    const double v = d[q];
    dn[q] = v;
    dt[(q / N) + N * (q % N)] = v;
  }
  __syncthreads();

  double *scr_r = scr + (size_t)(grp * E + el) * 2 * C::SCR;
  double *scr_s = scr_r + C::SCR;
  double acc = 0.0;

  for (int64_t m = 0; m < mine; ++m) {
    const int64_t c = chunk(m);
    const int st = grp * S + (int)(m % S);
    mbar_wait(&bars[st], (uint32_t)((m / S) & 1));
    const double *sg = stages + (size_t)st * C::STAGE;
    double *su0 = stages + (size_t)st * C::STAGE + C::GPART + u_lead(c);
    const int ne = chunk_elems(c);
    if (!u_bulk_ok(c)) {
      for (int q = lt; q < ne * NP; q += T) su0[q] = u[c * E * NP + q];
      named_bar_sync(1 + grp, T);
    }
    const bool active = lane_on && el < ne;
    const double *su = su0 + el * NP;
    const double *sge = sg + el * 6 * NP;

    double wt0[N], wt1[N];
    if (active) {
      double da[N], db0[N], db1[N];  // d(i,.), d(j0,.), d(j1,.)
#pragma unroll
      for (int l = 0; l < N; ++l) {
        da[l] = dn[i + N * l];
        db0[l] = dn[jj + N * l];
        db1[l] = dn[j1 + N * l];
      }
      double uc0[N], uc1[N];
#pragma unroll
      for (int l = 0; l < N; ++l) {
        uc0[l] = su[i + N * jj + N2 * l];
        uc1[l] = su[i + N * j1 + N2 * l];
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double *row0 = su + N * jj + N2 * k;  // u(., j0, k)
        const double *row1 = su + N * j1 + N2 * k;  // u(., j1, k)
        const double *col = su + i + N2 * k;        // u(i, ., k), shared
        double ur0, ur1, us0, us1, ut0, ut1;
#pragma unroll
        for (int l = 0; l < N; l += 2) {
          double a0, a1 = 0.0, b0, b1 = 0.0;
          if (l + 1 < N) {
            pair2<N>(row0 + l, a0, a1);
            pair2<N>(row1 + l, b0, b1);
          } else {
            a0 = row0[l];
            b0 = row1[l];
          }
#pragma unroll
          for (int h = 0; h < 2 && l + h < N; ++h) {
            const int ll = l + h;
            const double cv = col[N * ll];
            const double dk = c_dg2[N][k + N * ll];  // d(k,l)
            const double r0 = h ? a1 : a0, r1 = h ? b1 : b0;
            if (ll == 0) {
              ur0 = mac0<F>(da[0], r0);
              ur1 = mac0<F>(da[0], r1);
              us0 = mac0<F>(db0[0], cv);
              us1 = mac0<F>(db1[0], cv);
              ut0 = mac0<F>(dk, uc0[0]);
              ut1 = mac0<F>(dk, uc1[0]);
            } else {
              ur0 = mac<F>(ur0, da[ll], r0);
              ur1 = mac<F>(ur1, da[ll], r1);
              us0 = mac<F>(us0, db0[ll], cv);
              us1 = mac<F>(us1, db1[ll], cv);
              ut0 = mac<F>(ut0, dk, uc0[ll]);
              ut1 = mac<F>(ut1, dk, uc1[ll]);
            }
          }
        }
        {
          const double *gp = sge + 6 * (i + N * jj + N2 * k);
          const double2 g01 = *reinterpret_cast<const double2 *>(gp);
          const double2 g23 = *reinterpret_cast<const double2 *>(gp + 2);
          const double2 g45 = *reinterpret_cast<const double2 *>(gp + 4);
          scr_r[i + R * jj + R * N * k] =
              comb3<F>(g01.x, ur0, g01.y, us0, g23.x, ut0);
          scr_s[i + R * jj + R * N * k] =
              comb3<F>(g01.y, ur0, g23.y, us0, g45.x, ut0);
          wt0[k] = comb3<F>(g23.x, ur0, g45.x, us0, g45.y, ut0);
        }
        if (vc1) {
          const double *gp = sge + 6 * (i + N * j1 + N2 * k);
          const double2 g01 = *reinterpret_cast<const double2 *>(gp);
          const double2 g23 = *reinterpret_cast<const double2 *>(gp + 2);
          const double2 g45 = *reinterpret_cast<const double2 *>(gp + 4);
          scr_r[i + R * j1 + R * N * k] =
              comb3<F>(g01.x, ur1, g01.y, us1, g23.x, ut1);
          scr_s[i + R * j1 + R * N * k] =
              comb3<F>(g01.y, ur1, g23.y, us1, g45.x, ut1);
          wt1[k] = comb3<F>(g23.x, ur1, g45.x, us1, g45.y, ut1);
        } else {
          wt1[k] = 0.0;
        }
      }
    }
    named_bar_sync(1 + grp, T);  // stage consumed, scratch complete

    if (lt == 0 && m + S < mine) {
      fence_proxy_async_smem();
      issue(st, chunk(m + S));
    }

    if (active) {
      double da[N], db0[N], db1[N];  // d(., i), d(., j0), d(., j1)
#pragma unroll
      for (int l = 0; l < N; ++l) {
        da[l] = dt[i + N * l];
        db0[l] = dt[jj + N * l];
        db1[l] = dt[j1 + N * l];
      }
      double *we = w + (c * E + el) * NP + i;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double *rr0 = scr_r + R * jj + R * N * k;  // wr(., j0, k)
        const double *rr1 = scr_r + R * j1 + R * N * k;  // wr(., j1, k)
        const double *rs = scr_s + i + R * N * k;        // ws(i, ., k)
        double s0, s1;
#pragma unroll
        for (int l = 0; l < N; l += 2) {
          double a0, a1 = 0.0, b0, b1 = 0.0;
          if (l + 1 < N) {
            pair2<N>(rr0 + l, a0, a1);
            pair2<N>(rr1 + l, b0, b1);
          } else {
            a0 = rr0[l];
            b0 = rr1[l];
          }
#pragma unroll
          for (int h = 0; h < 2 && l + h < N; ++h) {
            const int ll = l + h;
            const double sv = rs[R * ll];
            const double dk = c_dg2[N][ll + N * k];  // d(l,k)
            const double r0 = h ? a1 : a0, r1 = h ? b1 : b0;
            s0 = mac<F>(mac<F>(ll == 0 ? mac0<F>(da[0], r0)
                                       : mac<F>(s0, da[ll], r0),
                               db0[ll], sv),
                        dk, wt0[ll]);
            s1 = mac<F>(mac<F>(ll == 0 ? mac0<F>(da[0], r1)
                                       : mac<F>(s1, da[ll], r1),
                               db1[ll], sv),
                        dk, wt1[ll]);
          }
        }
        we[N * jj + N2 * k] = s0;
        if (vc1) we[N * j1 + N2 * k] = s1;
        if constexpr (SUMSQ) {
          acc = dadd(acc, dmul(s0, s0));
          if (vc1) acc = dadd(acc, dmul(s1, s1));
        }
      }
    }
    named_bar_sync(1 + grp, T);  // scratch reads done before the next chunk
  }

  if constexpr (SUMSQ) block_sumsq_partial(acc, partials);
}

template <int N, int E, int G, int S, bool F>
static int launch_gen2(double *w, const double *u, const double *d,
                       const double *g, int64_t nelt, const lfb_launch *geom,
                       cudaStream_t s, int64_t *grid_out) {
  using L = Gen2Smem<N, E, G, S>;
  static_assert(L::total <= 227 * 1024, "smem");
  constexpr int block = G * Gen2Cfg<N, E>::T;
  int sms = sm_count(geom);
  if (sms <= 0) sms = 148;
  const int per_sm = (geom && geom->ctas_per_sm > 0) ? geom->ctas_per_sm : 1;
  const int64_t nchunks = (nelt + E - 1) / E;
  int64_t grid64 = (int64_t)sms * per_sm;
  if (grid64 * G > nchunks) grid64 = (nchunks + G - 1) / G;
  if (grid64 < 1) grid64 = 1;
  const int grid = (int)grid64;
  if (grid_out) {
    *grid_out = grid;
    return LFB_OK;
  }
  const bool sumsq = geom && geom->sumsq;
  if (sumsq && (!geom->workspace || geom->workspace_len < grid))
    return fail(LFB_ERR_ARG, "semlap: sumsq workspace too small");
  auto k = sumsq ? semlap_gen2_kernel<N, E, G, S, true, F>
                 : semlap_gen2_kernel<N, E, G, S, false, F>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)L::total);
  {
    std::unique_lock<std::mutex> lk;
    bool capturing = false;
    int slot = N;
    if (int rc = dconst_acquire(c_dg2, 144 * 8, 4, &slot, d, N, s, &lk,
                                &capturing))
      return rc;
    k<<<grid, block, L::total, s>>>(w, u, d, g, nelt,
                                    sumsq ? geom->workspace : nullptr);
    dconst_release(4, slot, s, capturing);
  }
  if (int rc = check_launch("lfb_semlap_f64")) return rc;
  return sumsq ? sem_sumsq_finish(geom->workspace, grid, geom->sumsq, s)
               : LFB_OK;
}

// (n, E, G, S): variant 60 bitwise, 61 DFMA mode
#define LFB_GEN2_TABLE(X) \
  X(7, 1, 6, 1)           \
  X(9, 1, 4, 1)           \
  X(10, 1, 3, 1)          \
  X(11, 1, 2, 1)          \
  X(12, 1, 1, 1)

int sem_gen2_dispatch(int n, int variant, double *w, const double *u,
                      const double *d, const double *g, int64_t nelt,
                      const lfb_launch *geom, cudaStream_t s,
                      int64_t *grid_out) {
#define X(NN, EE, GG, SS)                                                  \
  if (n == NN && variant == 60)                                            \
    return launch_gen2<NN, EE, GG, SS, false>(w, u, d, g, nelt, geom, s,   \
                                              grid_out);                   \
  if (n == NN && variant == 61)                                            \
    return launch_gen2<NN, EE, GG, SS, true>(w, u, d, g, nelt, geom, s,    \
                                             grid_out);
  LFB_GEN2_TABLE(X)
#undef X
  return -1;
}

}  // namespace lfb
