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
// B200 design: persistent CTAs (one per SM); G "element
// groups" of n^2 threads (whole warps) per CTA; thread (i,j) of a group owns
// the k-column of points (i,j,*) -- its u column and its wt column stay in
// registers, wr/ws cross the threads through a padded smem scratch (row
// stride n+2: 16-byte pairs stay aligned and the 4 j-rows of a warp land on
// distinct banks).  Two ways to feed a group from HBM:
//
//  * staged  (semlap_kernel): one 1-D bulk copy (TMA engine, mbarrier
//    complete_tx) each for u (n^3 doubles) and g (6 n^3) of a whole element
//    into an SG-deep per-group stage ring, issued as soon as phase 1 frees a
//    stage;
//  * streamed (semlap_cpa_kernel): u by bulk copy into a per-group double
//    buffer, and g -- 6/7 of the bytes, needed only at the phase-1 combine --
//    streamed per k-slice by each thread for its OWN point with 16-byte
//    cp.async into a small per-thread ring (no cross-thread sync at all),
//    P slices ahead.  Half the smem per group, so up to 7-8 groups (14-16
//    warps) per SM hide the FP64 and smem latencies.
//
// Optional fused epilogue: per-CTA sum(w*w) partials in a fixed order (a
// deterministic verification norm for the multi-GPU all-reduce).
#include "lfb_common.cuh"
#include "semlap_common.cuh"

namespace lfb {

template <int N>
struct SemCfg {
  static constexpr int N2 = N * N;
  static constexpr int NP = N * N * N;
  static constexpr int T = ((N2 + 31) / 32) * 32;
  static constexpr int R = (N % 2 == 0) ? N + 2 : N + 1;
  static constexpr int SCR = R * N * N;
  static constexpr int STAGE = 7 * NP;  // doubles: u then g
};

// element order of a persistent CTA: contiguous range or interleaved
struct ElemMap {
  int64_t base, stride, count;
  __device__ ElemMap(int64_t nelt, bool interleave) {
    if (interleave) {
      base = blockIdx.x;
      stride = gridDim.x;
      count = nelt > base ? (nelt - base + stride - 1) / stride : 0;
    } else {
      base = (nelt * blockIdx.x) / gridDim.x;
      stride = 1;
      count = (nelt * (blockIdx.x + 1)) / gridDim.x - base;
    }
  }
  __device__ int64_t operator()(int64_t t) const { return base + t * stride; }
};

// {{{ per-thread d rows: registers for the whole kernel, or per phase

template <int N>
struct DRows {
  double a[N], b[N];
  // phase 1: a = d(i,.), b = d(j,.)   (rows of d = columns of dt)
  __device__ __forceinline__ void load_phase1(const double *dt, int i, int j) {
#pragma unroll
    for (int l = 0; l < N; l += 2) {
      const double2 x = *reinterpret_cast<const double2 *>(dt + l + N * i);
      const double2 y = *reinterpret_cast<const double2 *>(dt + l + N * j);
      a[l] = x.x, a[l + 1] = x.y, b[l] = y.x, b[l + 1] = y.y;
    }
  }
  // phase 2: a = d(.,i), b = d(.,j)
  __device__ __forceinline__ void load_phase2(const double *dn, int i, int j) {
#pragma unroll
    for (int l = 0; l < N; l += 2) {
      const double2 x = *reinterpret_cast<const double2 *>(dn + l + N * i);
      const double2 y = *reinterpret_cast<const double2 *>(dn + l + N * j);
      a[l] = x.x, a[l + 1] = x.y, b[l] = y.x, b[l + 1] = y.y;
    }
  }
};

// }}}

// {{{ the two phases for one thread's column (even N: paired smem loads)

// phase 1 at slice k: returns wr, ws, wt of point (i,j,k)
// uT (optional): transposed copy, u(i,l,k) at uT[l + R i + R N k], so the
// us column becomes 16-byte pairs like the ur row
template <int N, bool UT>
__device__ __forceinline__ void phase1_point(const double *su,
                                             const double *uT,
                                             const double *dt,
                                             const double *ucol,
                                             const DRows<N> &dr,
                                             const double *gp, int i, int j,
                                             int k, double &wr, double &ws,
                                             double &wt) {
  constexpr int R = SemCfg<N>::R;
  double ur = 0.0, us = 0.0, ut = 0.0;
  const double *row = su + N * j + N * N * k;  // u(.,j,k)
  const double *col = su + i + N * N * k;      // u(i,.,k), stride N
  const double *colT = uT + R * i + R * N * k; // u(i,.,k), contiguous
  const double *dk = dt + N * k;               // d(k,.)
#pragma unroll
  for (int l = 0; l < N; l += 2) {
    const double2 r2 = *reinterpret_cast<const double2 *>(row + l);
    const double2 k2 = *reinterpret_cast<const double2 *>(dk + l);
    double c0, c1;
    if constexpr (UT) {
      const double2 c2 = *reinterpret_cast<const double2 *>(colT + l);
      c0 = c2.x, c1 = c2.y;
    } else {
      c0 = col[N * l], c1 = col[N * (l + 1)];
    }
    ur = dadd(ur, dmul(dr.a[l], r2.x));
    us = dadd(us, dmul(dr.b[l], c0));
    ut = dadd(ut, dmul(k2.x, ucol[l]));
    ur = dadd(ur, dmul(dr.a[l + 1], r2.y));
    us = dadd(us, dmul(dr.b[l + 1], c1));
    ut = dadd(ut, dmul(k2.y, ucol[l + 1]));
  }
  const double2 *g2 = reinterpret_cast<const double2 *>(gp);
  const double2 g01 = g2[0], g23 = g2[1], g45 = g2[2];
  wr = dadd(dadd(dmul(g01.x, ur), dmul(g01.y, us)), dmul(g23.x, ut));
  ws = dadd(dadd(dmul(g01.y, ur), dmul(g23.y, us)), dmul(g45.x, ut));
  wt = dadd(dadd(dmul(g23.x, ur), dmul(g45.x, us)), dmul(g45.y, ut));
}

// phase 2 at slice k
// TS: ws is stored transposed, ws(i,l,k) at scr_s[l + R i + R N k]
template <int N, bool TS>
__device__ __forceinline__ double phase2_point(const double *scr_r,
                                               const double *scr_s,
                                               const double *dn,
                                               const double *wt,
                                               const DRows<N> &dr, int i,
                                               int j, int k) {
  constexpr int R = SemCfg<N>::R;
  double s = 0.0;
  const double *rr = scr_r + R * j + R * N * k;  // wr(.,j,k)
  const double *rs = TS ? scr_s + R * i + R * N * k  // ws(i,.,k) contiguous
                        : scr_s + i + R * N * k;     // ws(i,.,k) stride R
  const double *dk = dn + N * k;                 // d(.,k)
#pragma unroll
  for (int l = 0; l < N; l += 2) {
    const double2 r2 = *reinterpret_cast<const double2 *>(rr + l);
    const double2 k2 = *reinterpret_cast<const double2 *>(dk + l);
    double s0, s1;
    if constexpr (TS) {
      const double2 s2 = *reinterpret_cast<const double2 *>(rs + l);
      s0 = s2.x, s1 = s2.y;
    } else {
      s0 = rs[R * l], s1 = rs[R * (l + 1)];
    }
    s = dadd(dadd(dadd(s, dmul(dr.a[l], r2.x)), dmul(dr.b[l], s0)),
             dmul(k2.x, wt[l]));
    s = dadd(dadd(dadd(s, dmul(dr.a[l + 1], r2.y)), dmul(dr.b[l + 1], s1)),
             dmul(k2.y, wt[l + 1]));
  }
  return s;
}

template <bool TS, int N>
__device__ __forceinline__ int ws_index(int i, int j, int k) {
  constexpr int R = SemCfg<N>::R;
  return TS ? j + R * i + R * N * k : i + R * j + R * N * k;
}

// }}}

__device__ __forceinline__ void stage_d(const double *__restrict__ d,
                                        double *dn, double *dt, int n) {
  for (int q = threadIdx.x; q < n * n; q += blockDim.x) {
    const double v = d[q];
    dn[q] = v;
    dt[(q / n) + n * (q % n)] = v;
  }
}

// {{{ staged kernel

template <int N, int G, int SG, bool TR>
struct SemSmem {
  using C = SemCfg<N>;
  static constexpr int NSCR = TR ? 3 : 2;  // wr, ws (+ uT)
  static constexpr size_t bars = 128;  // up to 16 mbarriers
  static constexpr size_t d_off = bars;
  static constexpr size_t scr_off = d_off + 2 * N * N * 8;
  static constexpr size_t stage_off =
      ((scr_off + (size_t)G * NSCR * C::SCR * 8) + 127) / 128 * 128;
  static constexpr size_t total = stage_off + (size_t)G * SG * C::STAGE * 8;
};

template <int N, int G, int SG, bool DPH, bool IL, bool TR, bool SUMSQ>
__global__ void __launch_bounds__(G *SemCfg<N>::T, 1)
    semlap_kernel(double *__restrict__ w, const double *__restrict__ u,
                  const double *__restrict__ d, const double *__restrict__ g,
                  int64_t nelt, double *__restrict__ partials) {
  using C = SemCfg<N>;
  using L = SemSmem<N, G, SG, TR>;
  constexpr int NP = C::NP, T = C::T, R = C::R;
  static_assert(G * SG <= 16, "too many stages");
  static_assert(N % 2 == 0, "paired loads need even n");

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
  const ElemMap emap(nelt, IL);
  const int64_t count = emap.count;

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
  if (lt == 0) {
    for (int m = 0; m < SG; ++m) {
      const int64_t t = grp + (int64_t)G * m;
      if (t < count) issue(grp * SG + m, emap(t));
    }
  }
  stage_d(d, dn, dt, N);
  __syncthreads();

  DRows<N> d1, d2;  // with DPH they are reloaded every phase
  if constexpr (!DPH) {
    d1.load_phase1(dt, i, j);
    d2.load_phase2(dn, i, j);
  }
  double *scr_r = scr + (size_t)grp * L::NSCR * C::SCR;
  double *scr_s = scr_r + C::SCR;
  double *uT = scr_s + C::SCR;  // TR only
  double acc = 0.0;

  for (int m = 0;; ++m) {
    const int64_t t = grp + (int64_t)G * m;
    if (t >= count) break;
    const int64_t e = emap(t);
    const int st = grp * SG + (m % SG);
    mbar_wait(&bars[st], (uint32_t)((m / SG) & 1));
    const double *su = stages + (size_t)st * C::STAGE;
    const double *sg = su + NP;

    double wt[N];
    double ucol[N];
    if (active) {
      if constexpr (DPH) d1.load_phase1(dt, i, j);
#pragma unroll
      for (int l = 0; l < N; ++l) ucol[l] = su[i + N * j + N * N * l];
      if constexpr (TR) {
        // u(i,j,k) -> uT[j + R i + R N k]: the us columns become rows
#pragma unroll
        for (int k = 0; k < N; ++k) uT[j + R * i + R * N * k] = ucol[k];
      }
    }
    if constexpr (TR) named_bar_sync(1 + grp, T);
    if (active) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double wr, ws;
        phase1_point<N, TR>(su, uT, dt, ucol, d1,
                            sg + 6 * (i + N * j + N * N * k), i, j, k, wr, ws,
                            wt[k]);
        scr_r[i + R * j + R * N * k] = wr;
        scr_s[ws_index<TR, N>(i, j, k)] = ws;
      }
    }
    named_bar_sync(1 + grp, T);  // stage consumed, scratch complete

    if (lt == 0) {
      const int64_t tn = t + (int64_t)G * SG;
      if (tn < count) {
        fence_proxy_async_smem();
        issue(st, emap(tn));
      }
    }

    if (active) {
      if constexpr (DPH) d2.load_phase2(dn, i, j);
      double *we = w + e * NP + i + N * j;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double s =
            phase2_point<N, TR>(scr_r, scr_s, dn, wt, d2, i, j, k);
        we[N * N * k] = s;
        if constexpr (SUMSQ) acc = dadd(acc, dmul(s, s));
      }
    }
    named_bar_sync(1 + grp, T);  // scratch reads done before the next phase 1
  }

  if constexpr (SUMSQ) block_sumsq_partial(acc, partials);
}

// }}}

// {{{ streamed kernel: u by bulk copy, g by per-thread cp.async ring

template <int N, int G, int P>
struct CpaSmem {
  using C = SemCfg<N>;
  static constexpr int D = P + 1;  // ring slots per thread
  static constexpr size_t bars = 128;
  static constexpr size_t d_off = bars;
  static constexpr size_t grp_off = (d_off + 2 * N * N * 8 + 127) / 128 * 128;
  static constexpr size_t u_bytes = 2 * (size_t)C::NP * 8;
  static constexpr size_t g_bytes = (size_t)D * C::T * 48;
  static constexpr size_t scr_bytes = 2 * (size_t)C::SCR * 8;
  static constexpr size_t grp_bytes =
      (u_bytes + g_bytes + scr_bytes + 127) / 128 * 128;
  static constexpr size_t total = grp_off + G * grp_bytes;
};

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   smem_u32(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int K>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory");
}

template <int N, int G, int P, bool IL, bool SUMSQ>
__global__ void __launch_bounds__(G *SemCfg<N>::T, 1)
    semlap_cpa_kernel(double *__restrict__ w, const double *__restrict__ u,
                      const double *__restrict__ d,
                      const double *__restrict__ g, int64_t nelt,
                      double *__restrict__ partials) {
  using C = SemCfg<N>;
  using L = CpaSmem<N, G, P>;
  constexpr int NP = C::NP, T = C::T, R = C::R, D = L::D;
  static_assert(N % 2 == 0 && N % D == 0, "slot index must be static");
  static_assert(P >= 1, "prefetch distance");

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem);
  double *dn = reinterpret_cast<double *>(smem + L::d_off);
  double *dt = dn + N * N;

  const int tid = threadIdx.x;
  const int grp = tid / T;
  const int lt = tid % T;
  const int i = lt % N;
  const int j = lt / N;
  const bool active = lt < N * N;
  const ElemMap emap(nelt, IL);
  // this group's elements: CTA-local t = grp + G m
  const int64_t mine =
      emap.count > grp ? (emap.count - grp + G - 1) / G : 0;

  unsigned char *gb = smem + L::grp_off + (size_t)grp * L::grp_bytes;
  double *ubuf = reinterpret_cast<double *>(gb);                      // 2 NP
  double *gring = reinterpret_cast<double *>(gb + L::u_bytes);        // D T 6
  double *scr_r = reinterpret_cast<double *>(gb + L::u_bytes + L::g_bytes);
  double *scr_s = scr_r + C::SCR;
  uint64_t *ubar = bars + 2 * grp;

  if (tid == 0) {
    for (int s = 0; s < 2 * G; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const uint64_t pol = policy_evict_first();
  auto issue_u = [&](int64_t m) {
    const int st = (int)(m & 1);
    mbar_arrive_expect_tx(&ubar[st], NP * 8);
    bulk_g2s_stream(ubuf + st * NP, u + emap(grp + G * m) * NP, NP * 8,
                    &ubar[st], pol);
  };
  // slice q = m*N + k of this thread's own point -> ring slot q % D
  const int64_t nslices = mine * N;
  auto issue_g = [&](int64_t q) {
    if (active && q < nslices) {
      const int64_t e = emap(grp + G * (q / N));
      const int k = (int)(q % N);
      const double *src = g + 6 * (e * NP + i + N * j + N * N * k);
      double *dst = gring + ((size_t)(q % D) * T + lt) * 6;
      cp_async16(dst, src);
      cp_async16(dst + 2, src + 2);
      cp_async16(dst + 4, src + 4);
    }
    cp_async_commit();  // empty groups keep the per-thread count uniform
  };

  if (lt == 0) {
    if (mine > 0) issue_u(0);
    if (mine > 1) issue_u(1);
  }
#pragma unroll
  for (int q = 0; q < P; ++q) issue_g(q);
  stage_d(d, dn, dt, N);
  __syncthreads();

  DRows<N> dr;
  double acc = 0.0;
  for (int64_t m = 0; m < mine; ++m) {
    const int64_t e = emap(grp + G * m);
    const int st = (int)(m & 1);
    mbar_wait(&ubar[st], (uint32_t)((m >> 1) & 1));
    const double *su = ubuf + st * NP;

    double wt[N];
    if (active) {
      dr.load_phase1(dt, i, j);
      double ucol[N];
#pragma unroll
      for (int l = 0; l < N; ++l) ucol[l] = su[i + N * j + N * N * l];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const int64_t q = m * N + k;
        cp_async_wait<P - 1>();  // own slice q has landed
        issue_g(q + P);          // into slot (q - 1) % D, consumed last step
        double wr, ws;
        phase1_point<N, false>(su, nullptr, dt, ucol, dr,
                        gring + ((size_t)(k % D) * T + lt) * 6, i, j, k, wr,
                        ws, wt[k]);
        scr_r[i + R * j + R * N * k] = wr;
        scr_s[i + R * j + R * N * k] = ws;
      }
    } else {
#pragma unroll
      for (int k = 0; k < N; ++k) issue_g(m * N + k + P);
    }
    named_bar_sync(1 + grp, T);  // u stage consumed, scratch complete
    if (lt == 0 && m + 2 < mine) {
      fence_proxy_async_smem();
      issue_u(m + 2);
    }

    if (active) {
      dr.load_phase2(dn, i, j);
      double *we = w + e * NP + i + N * j;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double s =
            phase2_point<N, false>(scr_r, scr_s, dn, wt, dr, i, j, k);
        we[N * N * k] = s;
        if constexpr (SUMSQ) acc = dadd(acc, dmul(s, s));
      }
    }
    named_bar_sync(1 + grp, T);  // scratch reads done
  }
  cp_async_wait<0>();

  if constexpr (SUMSQ) block_sumsq_partial(acc, partials);
}

// }}}

__global__ void sum_partials_kernel(const double *__restrict__ partials, int n,
                                    double *__restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < n; ++q) s = dadd(s, partials[q]);
    *out = s;
  }
}

int sem_sumsq_finish(const double *partials, int n, double *out,
                     cudaStream_t s) {
  sum_partials_kernel<<<1, 32, 0, s>>>(partials, n, out);
  return check_launch("lfb_semlap_f64(sumsq)");
}

// {{{ launch + dispatch

static int sem_grid(int64_t nelt, int groups, const lfb_launch *geom) {
  int sms = sm_count(geom);
  if (sms <= 0) sms = 148;
  int per_sm = (geom && geom->ctas_per_sm > 0) ? geom->ctas_per_sm : 1;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid * groups > nelt) grid = (nelt + groups - 1) / groups;
  return (int)(grid < 1 ? 1 : grid);
}

template <typename K>
static int launch_persistent(K kern_plain, K kern_sumsq, size_t smem,
                             int block, int groups, double *w, const double *u,
                             const double *d, const double *g, int64_t nelt,
                             const lfb_launch *geom, cudaStream_t s,
                             int64_t *grid_out) {
  const int grid = sem_grid(nelt, groups, geom);
  if (grid_out) {
    *grid_out = grid;
    return LFB_OK;
  }
  const bool sumsq = geom && geom->sumsq;
  if (sumsq && (!geom->workspace || geom->workspace_len < grid))
    return fail(LFB_ERR_ARG,
                "semlap: sumsq requested with workspace of %lld < %d doubles",
                (long long)(geom->workspace ? geom->workspace_len : 0), grid);
  K k = sumsq ? kern_sumsq : kern_plain;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  k<<<grid, block, smem, s>>>(w, u, d, g, nelt,
                              sumsq ? geom->workspace : nullptr);
  if (int rc = check_launch("lfb_semlap_f64")) return rc;
  return sumsq ? sem_sumsq_finish(geom->workspace, grid, geom->sumsq, s)
               : LFB_OK;
}

template <int N, int G, int SG, bool DPH, bool IL, bool TR>
static int launch_staged(double *w, const double *u, const double *d,
                         const double *g, int64_t nelt, const lfb_launch *geom,
                         cudaStream_t s, int64_t *grid_out) {
  using L = SemSmem<N, G, SG, TR>;
  static_assert(L::total <= 227 * 1024, "smem");
  return launch_persistent(semlap_kernel<N, G, SG, DPH, IL, TR, false>,
                           semlap_kernel<N, G, SG, DPH, IL, TR, true>,
                           L::total, G * SemCfg<N>::T, G, w, u, d, g, nelt,
                           geom, s, grid_out);
}

template <int N, int G, int P, bool IL>
static int launch_cpa(double *w, const double *u, const double *d,
                      const double *g, int64_t nelt, const lfb_launch *geom,
                      cudaStream_t s, int64_t *grid_out) {
  static_assert(CpaSmem<N, G, P>::total <= 227 * 1024, "smem");
  return launch_persistent(semlap_cpa_kernel<N, G, P, IL, false>,
                           semlap_cpa_kernel<N, G, P, IL, true>,
                           CpaSmem<N, G, P>::total, G * SemCfg<N>::T, G, w, u,
                           d, g, nelt, geom, s, grid_out);
}

// (n, variant) -> kernel.  variant 0 is the tuned default per order.
#define LFB_SEM_TABLE(S, A)                                                 \
  S(8, 39, 4, 1, false, true, false)                                        \
  S(8, 1, 2, 3, false, false, false)                                        \
  S(8, 2, 4, 1, false, false, false)                                        \
  S(8, 3, 5, 1, false, false, false)                                        \
  S(8, 4, 3, 2, false, false, false)                                        \
  S(8, 5, 4, 1, false, true, false)                                         \
  S(8, 6, 5, 1, true, false, false)                                         \
  S(8, 7, 5, 1, true, true, false)                                          \
  S(8, 16, 4, 1, false, true, true)                                         \
  S(8, 17, 4, 1, false, false, true)                                        \
  S(8, 18, 4, 1, true, true, true)                                          \
  S(8, 19, 3, 2, false, true, true)                                         \
  A(8, 10, 6, 3, false)                                                     \
  A(8, 11, 7, 3, false)                                                     \
  A(8, 12, 6, 3, true)                                                      \
  A(8, 13, 7, 3, true)                                                      \
  A(8, 14, 8, 1, true)                                                      \
  A(8, 15, 7, 1, true)

static int sem_dispatch(double *w, const double *u, const double *d,
                        const double *g, int64_t nelt, const lfb_launch *geom,
                        cudaStream_t s, int64_t *grid_out) {
  const int n = geom->npts;
  const int var0 = geom->variant;
#define S(NN, VV, GG, SS, DPH, IL, TR)                                      \
  if (n == NN && var == VV)                                                 \
    return launch_staged<NN, GG, SS, DPH, IL, TR>(w, u, d, g, nelt, geom,   \
                                                  s, grid_out);
#define A(NN, VV, GG, PP, IL)                                               \
  if (n == NN && var == VV)                                                 \
    return launch_cpa<NN, GG, PP, IL>(w, u, d, g, nelt, geom, s, grid_out);
  {
    // d in the constant bank (semlap_kc.cu): the default for n = 8
    const int rc = sem_kc_dispatch(n, var0, w, u, d, g, nelt, geom, s,
                                   grid_out);
    if (rc != -1) return rc;
  }
  if ((var0 >= 70 && var0 <= 73) ||
      (var0 == 0 && (n == 13 || n == 15 || n == 16))) {
    // line owners for phase 1 (semlap_line.cu), n = 9..16; the bitwise
    // default at n = 13, 15, 16 (+10..13 % over the k-slab kernel, which
    // stays the default at n = 12, 14: equal there)
    const int rc = sem_line_dispatch(n, var0 == 0 ? 70 : var0, w, u, d, g,
                                     nelt, geom, s, grid_out);
    if (rc != -1) return rc;
  }
  if (var0 == 60 || var0 == 61 ||
      (var0 == 50 && (n == 9 || n == 10))) {
    // two k-columns per thread (semlap_gen2.cu), n = 7, 9..12; the DFMA-mode
    // default at n = 9, 10 (+2..5 % over one column per thread)
    const int rc = sem_gen2_dispatch(n, var0 == 50 ? 61 : var0, w, u, d, g,
                                     nelt, geom, s, grid_out);
    if (rc != -1) return rc;
  }
  if ((var0 >= 51 && var0 <= 54) ||
      (var0 == 50 && (n == 7 || n == 8 || n >= 12))) {
    // FP64 tensor cores (semlap_tc.cu), n = 8..16; the interleaved-phase
    // kernel (52) is the DFMA-mode default for n >= 12, where it beats the
    // column kernels by 12-28 %, at n = 7 (+11 %), and at n = 8, where it
    // matches them in isolation and stays 8 % faster under the power cap
    const int rc = sem_tc_dispatch(n, var0 == 50 ? 52 : var0, w, u, d, g,
                                   nelt, geom, s, grid_out);
    if (rc != -1) return rc;
  }
  const int var = var0;
  LFB_SEM_TABLE(S, A)
#undef S
#undef A
  // other orders: whole-chunk staging (n <= 11), else / variant 9 the k-slab
  // streaming kernel
  if (var == 0 || var >= 20) {
    const int rc = sem_gen_dispatch(n, var, w, u, d, g, nelt, geom, s,
                                    grid_out);
    if (rc != -1) return rc;
  }
  return sem_slab_dispatch(n, var, w, u, d, g, nelt, geom, s, grid_out);
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
