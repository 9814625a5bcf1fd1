// SEM Laplacian, general order: E-element chunks staged whole (BASELINE
// config 5 sweep, orders 1..10 except the hand-tuned n = 8).
//
// Same reference arithmetic as semlap.cu (every * and +
// rounded separately, l ascending, left-associative sums), so the result is
// bitwise the reference's.
//
// Design:
//  * A *group* of T threads (whole warps) owns a chunk of E consecutive
//    elements at a time; thread lt maps to element el = lt / n^2 of the chunk
//    and point column (i, j) = (p % n, p / n), p = lt % n^2, and computes the
//    k-column (i, j, *) of that element.  E is chosen so E n^2 fills the
//    warps (n = 4: E = 2 -> 32 of 32 lanes; n = 6: E = 3 -> 108 of 128), so
//    small orders do not idle half the FP64 lanes.
//  * Per chunk, g (6 E n^3 doubles, always 16-byte aligned) and u (E n^3
//    doubles; for odd n the copy starts at the 16-byte boundary below and the
//    stage is read at an 8-byte lead) arrive by two bulk copies (TMA engine,
//    mbarrier complete_tx, L2 evict_first) into an S-deep stage ring per
//    group, re-armed as soon as phase 1 has consumed a stage.  A final chunk
//    whose rounded u span would read past the array is copied by the threads.
//  * Chunks are interleaved over all groups of the persistent grid, so the
//    concurrently streamed chunks are adjacent in HBM.
//  * Both phases fully unrolled over k and l: n independent accumulation
//    chains per thread give the FP64 pipe the ILP it needs at low occupancy.
//  * the broadcast d(k,l) / d(l,k) of the ut contractions come from the
//    constant bank (dconst.cuh: uniform loads, no LSU traffic); the
//    per-thread rows d(i,.), d(j,.) from smem (dn = d, dt = d^T), optionally
//    kept in registers (DREG).
#include "dconst.cuh"
#include "lfb_common.cuh"
#include "semlap_common.cuh"

namespace lfb {

// d(a,b) at c_dgen[N][a + N b] for the order being launched (dconst.cuh)
__constant__ double c_dgen[12][128];

template <int N, int E>
struct GenCfg {
  static constexpr int N2 = N * N;
  static constexpr int NP = N * N * N;
  static constexpr int LANES = E * N2;
  static constexpr int T = ((LANES + 31) / 32) * 32;
  static constexpr int R = (N % 2 == 0) ? N + 2 : N + 1;  // scratch row
  static constexpr int SCR = R * N * N;                    // per element
  static constexpr int GPART = 6 * E * NP;                 // doubles
  static constexpr int UPART = ((E * NP + 1) + 1) / 2 * 2; // + lead, even
  static constexpr int STAGE = GPART + UPART;
};

template <int N, int E, int G, int S>
struct GenSmem {
  using C = GenCfg<N, E>;
  static constexpr size_t bars = ((size_t)8 * G * S + 127) / 128 * 128;
  static constexpr size_t d_off = bars;
  static constexpr size_t scr_off =
      (d_off + 2 * (size_t)C::N2 * 8 + 127) / 128 * 128;
  static constexpr size_t stage_off =
      (scr_off + (size_t)G * E * 2 * C::SCR * 8 + 127) / 128 * 128;
  static constexpr size_t total = stage_off + (size_t)G * S * C::STAGE * 8;
};

template <int N>
__device__ __forceinline__ void ld_pair(const double *p, double &a,
                                        double &b) {
  if constexpr (N % 2 == 0) {
    const double2 v = *reinterpret_cast<const double2 *>(p);
    a = v.x, b = v.y;
  } else {
    a = p[0], b = p[1];
  }
}

template <int N, int E, int G, int S, bool DREG, bool SUMSQ, bool F>
__global__ void __launch_bounds__(G *GenCfg<N, E>::T, 1)
    semlap_gen_kernel(double *__restrict__ w, const double *__restrict__ u,
                      const double *__restrict__ d,
                      const double *__restrict__ g, int64_t nelt,
                      double *__restrict__ partials) {
  using C = GenCfg<N, E>;
  using L = GenSmem<N, E, G, S>;
  constexpr int N2 = C::N2, NP = C::NP, T = C::T, R = C::R;
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
  const int el = lt / N2;
  const int pt = lt % N2;
  const int i = pt % N;
  const int j = pt / N;
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
    if (!u_bulk_ok(c)) {  // last chunk of an odd-n array: copy u by hand
      for (int q = lt; q < ne * NP; q += T) su0[q] = u[c * E * NP + q];
      named_bar_sync(1 + grp, T);
    }
    const bool active = lane_on && el < ne;
    const double *su = su0 + el * NP;
    const double *sge = sg + el * 6 * NP;

    double wt[N];
    if (active) {
      double da[N], db[N];  // d(i,.) and d(j,.)
      if constexpr (DREG) {
#pragma unroll
        for (int l = 0; l < N; ++l) da[l] = dn[i + N * l], db[l] = dn[j + N * l];
      }
      double ucol[N];
#pragma unroll
      for (int l = 0; l < N; ++l) ucol[l] = su[i + N * j + N2 * l];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double *row = su + N * j + N2 * k;  // u(., j, k)
        const double *col = su + i + N2 * k;      // u(i, ., k)
        double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
        for (int l = 0; l + 1 < N; l += 2) {
          double r0, r1;
          ld_pair<N>(row + l, r0, r1);
          const double k0 = c_dgen[N][k + N * l];  // d(k,l): constant bank
          const double k1 = c_dgen[N][k + N * (l + 1)];
          const double a0 = DREG ? da[l] : dn[i + N * l];
          const double a1 = DREG ? da[l + 1] : dn[i + N * (l + 1)];
          const double b0 = DREG ? db[l] : dn[j + N * l];
          const double b1 = DREG ? db[l + 1] : dn[j + N * (l + 1)];
          ur = mac<F>(ur, a0, r0);
          us = mac<F>(us, b0, col[N * l]);
          ut = mac<F>(ut, k0, ucol[l]);
          ur = mac<F>(ur, a1, r1);
          us = mac<F>(us, b1, col[N * (l + 1)]);
          ut = mac<F>(ut, k1, ucol[l + 1]);
        }
        if constexpr (N % 2 == 1) {
          constexpr int l = N - 1;
          const double a0 = DREG ? da[l] : dn[i + N * l];
          const double b0 = DREG ? db[l] : dn[j + N * l];
          ur = mac<F>(ur, a0, row[l]);
          us = mac<F>(us, b0, col[N * l]);
          ut = mac<F>(ut, c_dgen[N][k + N * l], ucol[l]);
        }
        const double *gp = sge + 6 * (i + N * j + N2 * k);
        const double2 g01 = *reinterpret_cast<const double2 *>(gp);
        const double2 g23 = *reinterpret_cast<const double2 *>(gp + 2);
        const double2 g45 = *reinterpret_cast<const double2 *>(gp + 4);
        scr_r[i + R * j + R * N * k] =
            comb3<F>(g01.x, ur, g01.y, us, g23.x, ut);
        scr_s[i + R * j + R * N * k] = comb3<F>(g01.y, ur, g23.y, us, g45.x, ut);
        wt[k] = comb3<F>(g23.x, ur, g45.x, us, g45.y, ut);
      }
    }
    named_bar_sync(1 + grp, T);  // stage consumed, scratch complete

    if (lt == 0 && m + S < mine) {
      fence_proxy_async_smem();
      issue(st, chunk(m + S));
    }

    if (active) {
      double da[N], db[N];  // d(., i) and d(., j)
      if constexpr (DREG) {
#pragma unroll
        for (int l = 0; l < N; ++l) da[l] = dt[i + N * l], db[l] = dt[j + N * l];
      }
      double *we = w + (c * E + el) * NP + i + N * j;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double *rr = scr_r + R * j + R * N * k;  // wr(., j, k)
        const double *rs = scr_s + i + R * N * k;      // ws(i, ., k)
        double s = 0.0;
#pragma unroll
        for (int l = 0; l + 1 < N; l += 2) {
          double r0, r1;
          ld_pair<N>(rr + l, r0, r1);
          const double k0 = c_dgen[N][l + N * k];  // d(l,k)
          const double k1 = c_dgen[N][l + 1 + N * k];
          const double a0 = DREG ? da[l] : dt[i + N * l];
          const double a1 = DREG ? da[l + 1] : dt[i + N * (l + 1)];
          const double b0 = DREG ? db[l] : dt[j + N * l];
          const double b1 = DREG ? db[l + 1] : dt[j + N * (l + 1)];
          s = mac<F>(mac<F>(mac<F>(s, a0, r0), b0, rs[R * l]), k0, wt[l]);
          s = mac<F>(mac<F>(mac<F>(s, a1, r1), b1, rs[R * (l + 1)]), k1,
                     wt[l + 1]);
        }
        if constexpr (N % 2 == 1) {
          constexpr int l = N - 1;
          const double a0 = DREG ? da[l] : dt[i + N * l];
          const double b0 = DREG ? db[l] : dt[j + N * l];
          s = mac<F>(mac<F>(mac<F>(s, a0, rr[l]), b0, rs[R * l]),
                     c_dgen[N][l + N * k], wt[l]);
        }
        we[N2 * k] = s;
        if constexpr (SUMSQ) acc = dadd(acc, dmul(s, s));
      }
    }
    named_bar_sync(1 + grp, T);  // scratch reads done before the next chunk
  }

  if constexpr (SUMSQ) block_sumsq_partial(acc, partials);
}

template <int N, int E, int G, int S, bool DREG, bool F>
static int launch_gen(double *w, const double *u, const double *d,
                      const double *g, int64_t nelt, const lfb_launch *geom,
                      cudaStream_t s, int64_t *grid_out) {
  using L = GenSmem<N, E, G, S>;
  static_assert(L::total <= 227 * 1024, "smem");
  constexpr int block = G * GenCfg<N, E>::T;
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
  auto k = sumsq ? semlap_gen_kernel<N, E, G, S, DREG, true, F>
                 : semlap_gen_kernel<N, E, G, S, DREG, false, F>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)L::total);
  {
    std::unique_lock<std::mutex> lk;
    bool capturing = false;
    int slot = N;  // one constant slot per order
    if (int rc = dconst_acquire(c_dgen, 128 * 8, 1, &slot, d, N, s, &lk,
                                &capturing))
      return rc;
    k<<<grid, block, L::total, s>>>(w, u, d, g, nelt,
                                    sumsq ? geom->workspace : nullptr);
    dconst_release(1, slot, s, capturing);
  }
  if (int rc = check_launch("lfb_semlap_f64")) return rc;
  return sumsq ? sem_sumsq_finish(geom->workspace, grid, geom->sumsq, s)
               : LFB_OK;
}

// (n, variant) -> (E, G, S, DREG); variant 0 = default for that n, from the
// round-1 B200 sweep (profiles/r01/sem_sweep.jsonl).  One stage per group
// (re-armed after phase 1, so the load overlaps phase 2 and the other
// groups) with as many groups as smem allows beat deeper rings everywhere.
#define LFB_GEN_TABLE(X)        \
  X(2, 0, 8, 8, 1, true)        \
  X(3, 0, 7, 8, 1, true)        \
  X(4, 0, 2, 14, 1, true)       \
  X(4, 20, 2, 8, 3, true)       \
  X(4, 21, 4, 6, 2, true)       \
  X(5, 0, 5, 4, 1, true)        \
  X(5, 20, 5, 3, 1, true)       \
  X(5, 21, 1, 14, 2, true)      \
  X(5, 22, 5, 2, 2, true)       \
  X(6, 0, 3, 4, 1, true)        \
  X(6, 20, 2, 6, 1, true)       \
  X(6, 21, 1, 8, 2, true)       \
  X(6, 22, 2, 4, 2, true)       \
  X(7, 0, 2, 4, 1, true)        \
  X(7, 20, 2, 3, 1, true)       \
  X(7, 21, 1, 8, 1, true)       \
  X(7, 22, 1, 5, 2, true)       \
  X(8, 20, 1, 3, 2, true)       \
  X(8, 21, 1, 4, 1, true)       \
  X(8, 22, 1, 4, 1, false)      \
  X(9, 0, 1, 4, 1, false)       \
  X(9, 20, 1, 2, 2, true)       \
  X(9, 21, 1, 3, 1, true)       \
  X(10, 0, 1, 3, 1, false)      \
  X(10, 20, 1, 2, 1, true)      \
  X(10, 21, 1, 3, 1, true)      \
  X(11, 0, 1, 2, 1, false)       \
  X(11, 20, 1, 2, 1, true)

int sem_gen_dispatch(int n, int variant, double *w, const double *u,
                     const double *d, const double *g, int64_t nelt,
                     const lfb_launch *geom, cudaStream_t s,
                     int64_t *grid_out) {
#define X(NN, VV, EE, GG, SS, DR)                                          \
  if (n == NN && variant == VV)                                            \
    return launch_gen<NN, EE, GG, SS, DR, false>(w, u, d, g, nelt, geom,   \
                                                 s, grid_out);             \
  if (VV == 0 && n == NN && variant == 50) /* default config, FMA mode */  \
    return launch_gen<NN, EE, GG, SS, DR, VV == 0>(w, u, d, g, nelt, geom, \
                                                   s, grid_out);
  LFB_GEN_TABLE(X)
#undef X
  return -1;  // no generic-kernel entry for (n, variant)
}

}  // namespace lfb
