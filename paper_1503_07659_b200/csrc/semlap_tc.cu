// SEM Laplacian on the FP64 tensor cores (DMMA m8n8k4), n = 9..16, DFMA
// tolerance mode (variant 51).
//
// Arithmetic: the reference's operator, with every
// multiply-add fused and the three contractions of phase 2 accumulated one
// after the other instead of interleaved per l -- fp64 within the north
// star's 1e-12 relative (checked per point against the magnitude of the
// summed terms, tests/test_gpu_parity.py), not bitwise.
//
// Why: at high order the per-thread column kernels (semlap_gen/slab) are
// bound by shared-memory instructions (ncu: L1 LSU pipe 72-84 %): every
// scalar multiply-add of ur/us and of the phase-2 sums needs one operand
// from smem, and a warp-wide LDS costs >= 2 wavefronts however few addresses
// it reads.  As 8x8x4 matrix products the same contractions need one
// conflict-free LDS.64 per 256 multiply-adds (the d operand stays in
// registers), and DMMA reaches the FP64 peak with 4 warps per SM
// (tools/micro/dmma_probe.cu: 35-37 TFLOP/s).
//
// Mapping (NT = 2 tiles of 8 per direction, 4 warps per element): warp
// (it, jt) owns the 8x8 tile of points i in [8it, 8it+8), j in [8jt, 8jt+8)
// for every k; the accumulator tiles are transposed (rows j, columns i), so
// lane l holds (j = 8jt + l/4, i = 8it + 2(l%4) + {0,1}): two k-columns per
// thread, adjacent in i.
//   ur^T(:, :, k) = u(:, :, k)^T . D^T    A = u slice, B = d (registers)
//   us^T(:, :, k) = D . u(:, :, k)^T      A = d (registers), B = u slice
//   ut(i, j, :) = D . u(i, j, :)          the thread's own columns: DFMA with
//                                         d(k,l) from the constant bank
//   phase 2: w = D^T . wr + ws . D (DMMA, wr/ws from smem) + D-contraction
//            of the thread's own wt columns (DFMA).
// Rows / columns >= n of a tile are padding: d is zero there and the padded
// smem is zero, so they contribute exact zeros and are never stored.
//
// Shared memory per element group: the u of one element and a ring of g
// k-slabs (TMA bulk copies), a padded copy of the current u slice (row
// stride P = 20 doubles: the fragment loads of a half warp hit 16 distinct
// 8-byte bank slots), and wr / ws for the whole element in the same padded
// layout.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <string.h>

#include "dconst.cuh"
#include "lfb_common.cuh"
#include "semlap_common.cuh"

namespace lfb {

// d(a,b) at c_dtc[ROW][a + N b]: ROW = N for the variant-51 kernel and slot
// 0 of the interleaved-phase kernel, N + 10 for its slot 1 -- two rotating
// slots per order (dconst.cuh), so same-order launches on two streams do
// not serialise on one slot
__constant__ double c_dtc[27][256];

template <int N>
struct TcCfg {
  static constexpr int NT = (N + 7) / 8;     // 8-wide tiles per direction
  static constexpr int W = NT * NT;          // warps per element
  static constexpr int T = 32 * W;
  static constexpr int KT = (N + 3) / 4;     // k-steps of 4
  static constexpr int P = 8 * NT + 4;       // padded row stride (20)
  static constexpr int B = 8 * NT;           // padded column extent (16)
  static constexpr int NP = N * N * N;
  static constexpr int UST = (NP + 2 + 1) / 2 * 2;  // + 8-byte lead, even
  static constexpr int SL = P * B;           // one padded slice
  static constexpr int SLAB = 6 * N * N;     // g of one k-slice
};

template <int N, int G, int SGS, int KS>
struct TcSmem {
  using C = TcCfg<N>;
  static constexpr size_t bars = 256;
  static constexpr size_t grp_doubles =
      (size_t)C::UST + (size_t)SGS * KS * C::SLAB + 3 * (size_t)C::SL * N;
  static constexpr size_t grp_bytes = (grp_doubles * 8 + 127) / 128 * 128;
  static constexpr size_t total = bars + G * grp_bytes;
};

// D = A(8x4, row) * B(4x8, col) + D; lane l holds a = A[l/4][l%4],
// b = B[l%4][l/4], d = D[l/4][2(l%4) + {0,1}]
__device__ __forceinline__ void dmma(double &d0, double &d1, double a,
                                     double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, "
      "{%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

template <int N, int ROW = N>
__device__ __forceinline__ double dtc(int a, int b) {  // d(a,b), 0 outside
  return (a < N && b < N) ? c_dtc[ROW][a + N * b] : 0.0;
}

template <int N, int G, int SGS, int KS, bool SUMSQ>
__global__ void __launch_bounds__(G *TcCfg<N>::T, 1)
    semlap_tc_kernel(double *__restrict__ w, const double *__restrict__ u,
                     const double *__restrict__ g, int64_t nelt,
                     double *__restrict__ partials) {
  using C = TcCfg<N>;
  using L = TcSmem<N, G, SGS, KS>;
  constexpr int NP = C::NP, T = C::T, KT = C::KT, P = C::P, SL = C::SL;
  constexpr int N2 = N * N;
  static_assert(N > 8 && N <= 16, "n = 9..16");
  static_assert(G * (1 + SGS) <= 32, "mbarriers");

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem);

  const int tid = threadIdx.x;
  const int grp = tid / T;
  const int lt = tid % T;
  const int warp = lt / 32, lane = lt % 32;
  const int it = warp / C::NT, jt = warp % C::NT;
  const int r = lane / 4, q = lane % 4;
  // accumulator rows = j, columns = i: the two points of a thread are
  // adjacent in i (one 16-byte store of w) and the g reads of a quarter
  // warp spread over the banks
  const int j = 8 * jt + r;
  const int i0 = 8 * it + 2 * q;       // accumulator columns i0, i0 + 1
  const bool vj = j < N;
  const bool v0 = vj && i0 < N, v1 = vj && i0 + 1 < N;

  double *gb = reinterpret_cast<double *>(smem + L::bars +
                                          (size_t)grp * L::grp_bytes);
  double *ust0 = gb;                         // u of the element (UST)
  double *slabs = ust0 + C::UST;             // SGS x KS x 6 N^2
  double *upd = slabs + SGS * KS * C::SLAB;  // u: N padded slices
  double *wrp = upd + (size_t)SL * N;        // wr: N padded slices
  double *wsp = wrp + (size_t)SL * N;        // ws: N padded slices
  uint64_t *ubar = bars + grp * (1 + SGS);
  uint64_t *gbar = ubar + 1;

  const int64_t q0 = (int64_t)blockIdx.x * G + grp;
  const int64_t Q = (int64_t)gridDim.x * G;
  const int64_t mine = nelt > q0 ? (nelt - q0 + Q - 1) / Q : 0;
  auto elem = [&](int64_t m) -> int64_t { return q0 + m * Q; };

  if (tid == 0) {
    for (int x = 0; x < G * (1 + SGS); ++x) mbar_init(&bars[x], 1);
    fence_mbar_init();
  }
  // zero the padded buffers once: padding stays zero for the whole kernel
  for (int x = lt; x < 3 * SL * N; x += T) upd[x] = 0.0;
  __syncthreads();

  const uint64_t pol = policy_evict_first();
  // u of element e: bulk copy of the 16-byte aligned superset (odd n: the
  // element starts 8 bytes into it for odd e); a final element whose
  // rounded end would run past the array is copied by the threads
  const int64_t u_bytes_total = nelt * NP * 8;
  auto u_lead = [&](int64_t e) -> int { return (int)((e * NP) & 1); };
  auto u_span = [&](int64_t e) -> int64_t {
    return ((int64_t)(u_lead(e) + NP) * 8 + 15) / 16 * 16;
  };
  auto u_bulk_ok = [&](int64_t e) -> bool {
    return (e * NP - u_lead(e)) * 8 + u_span(e) <= u_bytes_total;
  };
  auto issue_u = [&](int64_t m) {
    const int64_t e = elem(m);
    if (u_bulk_ok(e)) {
      mbar_arrive_expect_tx(ubar, (uint32_t)u_span(e));
      bulk_g2s_stream(ust0, u + e * NP - u_lead(e), (uint32_t)u_span(e),
                      ubar, pol);
    } else {
      mbar_arrive_expect_tx(ubar, 0);
    }
  };
  // slab q = KS consecutive k-slices of g (q = m * N / KS + k / KS)
  static_assert(N % KS == 0, "KS divides n");  // odd n: KS = 1
  auto issue_slab = [&](int64_t sq) {
    const int64_t e = elem(sq / (N / KS));
    const int k0 = (int)(sq % (N / KS)) * KS;
    const int slot = (int)(sq % SGS);
    mbar_arrive_expect_tx(&gbar[slot], (uint32_t)(KS * C::SLAB * 8));
    bulk_g2s_stream(slabs + (size_t)slot * KS * C::SLAB,
                    g + e * 6 * NP + (int64_t)k0 * 6 * N2, KS * C::SLAB * 8,
                    &gbar[slot], pol);
  };
  const int64_t nslabs = mine * (N / KS);
  if (lt == 0) {
    if (mine > 0) issue_u(0);
    for (int64_t s = 0; s < SGS && s < nslabs; ++s) issue_slab(s);
  }

  // d fragments (registers for the whole kernel):
  //   ur : A = d(i, l)       a = d(8it + r, 4ks + q)
  //   us : B = d(j, l)^T     b = d(8jt + r, 4ks + q)   [B[l][j] = d(j,l)]
  //   w1 : A = d(l, i)^T     a = d(4ks + q, 8it + r)
  //   w2 : B = d(l, j)       b = d(4ks + q, 8jt + r)
  double fa_r[KT], fb_s[KT], fa_t[KT], fb_t[KT];
#pragma unroll
  for (int ks = 0; ks < KT; ++ks) {
    fa_r[ks] = dtc<N>(8 * it + r, 4 * ks + q);
    fb_s[ks] = dtc<N>(8 * jt + r, 4 * ks + q);
    fa_t[ks] = dtc<N>(4 * ks + q, 8 * it + r);
    fb_t[ks] = dtc<N>(4 * ks + q, 8 * jt + r);
  }

  double acc_sq = 0.0;
  for (int64_t m = 0; m < mine; ++m) {
    const int64_t e = elem(m);
    mbar_wait(ubar, (uint32_t)(m & 1));
    const double *ust = ust0 + u_lead(e);
    if (!u_bulk_ok(e)) {
      for (int x = lt; x < NP; x += T) ust0[u_lead(e) + x] = u[e * NP + x];
      named_bar_sync(1 + grp, T);
    }

    // padded copy of the whole element: u(a, b, k) at a + P b + SL k
    for (int x = lt; x < NP; x += T) {
      const int a = x % N, b = (x / N) % N, k = x / N2;
      upd[a + P * b + SL * k] = ust[x];
    }
    // the thread's own two k-columns u(i, j0 + c, :) -> ut for every k:
    // 2N independent DFMA chains (d(k,l) are constant-bank operands)
    double t0[N], t1[N];
    {
      double uc0[N], uc1[N];
#pragma unroll
      for (int l = 0; l < N; ++l) {
        uc0[l] = v0 ? ust[i0 + N * j + N2 * l] : 0.0;
        uc1[l] = v1 ? ust[i0 + 1 + N * j + N2 * l] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < N; ++k) t0[k] = t1[k] = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double dk = c_dtc[N][k + N * l];
          t0[k] = __fma_rn(dk, uc0[l], t0[k]);
          t1[k] = __fma_rn(dk, uc1[l], t1[k]);
        }
      }
    }
    named_bar_sync(1 + grp, T);  // padded u complete, u stage consumed
    if (lt == 0 && m + 1 < mine) {
      fence_proxy_async_smem();
      issue_u(m + 1);  // overlaps both phases of this element
    }

    // ---- phase 1: ur / us on the tensor cores, combine with g
    double wt0[N], wt1[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int64_t s = m * N + k;
      const double *sl = upd + SL * k;
      double r0 = 0.0, r1 = 0.0, s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KT; ++ks) {
        // ur^T: A[j][l] = u(l, j, k) at l + P j, B[l][i] = d(i, l)
        dmma(r0, r1, sl[(4 * ks + q) + P * (8 * jt + r)], fa_r[ks]);
        // us^T: A[j][l] = d(j, l), B[l][i] = u(i, l, k) at i + P l
        dmma(s0, s1, fb_s[ks], sl[(8 * it + r) + P * (4 * ks + q)]);
      }
      if (k % KS == 0) mbar_wait(&gbar[(s / KS) % SGS],
                                 (uint32_t)((s / KS / SGS) & 1));
      // combine with g at (i, j0 + c, k)
      const double *gs = slabs + (size_t)((s / KS) % SGS) * KS * C::SLAB +
                         (size_t)(k % KS) * C::SLAB;
      double *wr_k = wrp + (size_t)SL * k;
      double *ws_k = wsp + (size_t)SL * k;
      if (v0) {
        const double2 *g2 =
            reinterpret_cast<const double2 *>(gs + 6 * (i0 + N * j));
        const double2 g01 = g2[0], g23 = g2[1], g45 = g2[2];
        wr_k[i0 + P * j] = comb3<true>(g01.x, r0, g01.y, s0, g23.x, t0[k]);
        ws_k[i0 + P * j] = comb3<true>(g01.y, r0, g23.y, s0, g45.x, t0[k]);
        wt0[k] = comb3<true>(g23.x, r0, g45.x, s0, g45.y, t0[k]);
      } else {
        wt0[k] = 0.0;
      }
      if (v1) {
        const double2 *g2 =
            reinterpret_cast<const double2 *>(gs + 6 * (i0 + 1 + N * j));
        const double2 g01 = g2[0], g23 = g2[1], g45 = g2[2];
        wr_k[i0 + 1 + P * j] =
            comb3<true>(g01.x, r1, g01.y, s1, g23.x, t1[k]);
        ws_k[i0 + 1 + P * j] =
            comb3<true>(g01.y, r1, g23.y, s1, g45.x, t1[k]);
        wt1[k] = comb3<true>(g23.x, r1, g45.x, s1, g45.y, t1[k]);
      } else {
        wt1[k] = 0.0;
      }
      if (k % KS == KS - 1 || k == N - 1) {
        named_bar_sync(1 + grp, T);  // slab consumed
        const int64_t slab = s / KS;
        if (lt == 0 && slab + SGS < nslabs) {
          fence_proxy_async_smem();
          issue_slab(slab + SGS);
        }
      }
    }
    // the own-column contraction of phase 2 for every k (2N chains),
    // the starting value of the tensor-core sums below
#pragma unroll
    for (int k = 0; k < N; ++k) t0[k] = t1[k] = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double dk = c_dtc[N][l + N * k];
        t0[k] = __fma_rn(dk, wt0[l], t0[k]);
        t1[k] = __fma_rn(dk, wt1[l], t1[k]);
      }
    }
    // (the last slab barrier above made wr / ws complete)

    // ---- phase 2
    double *we = w + e * NP;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const double *wr_k = wrp + (size_t)SL * k;
      const double *ws_k = wsp + (size_t)SL * k;
      double a0 = t0[k], a1 = t1[k];
#pragma unroll
      for (int ks = 0; ks < KT; ++ks) {
        // sum_l d(l,i) wr(l,j,k): A[j][l] = wr(l,j,k), B[l][i] = d(l,i)
        dmma(a0, a1, wr_k[(4 * ks + q) + P * (8 * jt + r)], fa_t[ks]);
        // sum_l ws(i,l,k) d(l,j): A[j][l] = d(l,j), B[l][i] = ws(i,l,k)
        dmma(a0, a1, fb_t[ks], ws_k[(8 * it + r) + P * (4 * ks + q)]);
      }
      if (N % 2 == 0 && v1) {  // even n: 16-byte aligned pair
        *reinterpret_cast<double2 *>(we + i0 + N * j + N2 * k) =
            make_double2(a0, a1);
      } else {
        if (v0) we[i0 + N * j + N2 * k] = a0;
        if (v1) we[i0 + 1 + N * j + N2 * k] = a1;
      }
      if constexpr (SUMSQ) {
        if (v0) acc_sq = dadd(acc_sq, dmul(a0, a0));
        if (v1) acc_sq = dadd(acc_sq, dmul(a1, a1));
      }
    }
    named_bar_sync(1 + grp, T);  // wr / ws / padded u reads done
  }

  if constexpr (SUMSQ) block_sumsq_partial(acc_sq, partials);
}

// {{{ interleaved-phase DMMA kernel (variant 52)
//
// The first DMMA kernel keeps wr / ws of a whole element (2 x 40 KB at
// n = 16) because phase 2 starts only when phase 1 is complete -- the
// D-contraction of wt over l needs every slice.  That leaves one 4-warp
// group per SM, latency bound.  Here the two DMMA sums of phase 2 for slice
// k (d^T.wr and ws.d) are formed right after phase 1 has produced wr / ws of
// slice k -- they only need that slice -- and kept per thread (2 values per
// k); the own-column sum over wt is added once phase 1 is complete.  wr / ws
// shrink to a 2-slice ring, the ur / us fragments are read straight from the
// staged u (zeroed smem makes every padded read finite), and 2-3 groups
// (8-12 warps) fit per SM.  Arithmetic as variant 51 (DFMA mode, within
// 1e-12; the phase-2 sums are added in a different order).
template <int N, int G, int SGS, int KS, bool SWZ = false>
struct Tc2Smem {
  using C = TcCfg<N>;
  // SWZ (n = 16): u staged by a 2-D TMA with the 128-B swizzle, no lead
  static constexpr int UST = SWZ ? C::NP : (C::NP + 2 + 1) / 2 * 2;
  static constexpr size_t grp_doubles =
      (size_t)UST + (size_t)SGS * KS * C::SLAB + 4 * (size_t)C::SL;
  static constexpr size_t galign = SWZ ? 1024 : 128;  // swizzle atoms
  static constexpr size_t grp_bytes =
      (grp_doubles * 8 + galign - 1) / galign * galign;
  static constexpr size_t bars = SWZ ? 1024 : 512;  // up to 64 mbarriers
  static constexpr size_t total = bars + G * grp_bytes + (SWZ ? 1024 : 0);
};

// index of u(c, R) in the staged element, R = j + N k the row: plain, or
// (n = 16) the TMA 128-B swizzle -- 16-byte chunk c/2 of row R XOR R mod 8 --
// which spreads the ur^T fragment (8 rows x 4 columns) over all banks
// instead of 4 (the row stride of 128 B maps every row to the same banks)
template <int N, bool SWZ>
__device__ __forceinline__ int uidx(int c, int R) {
  if constexpr (SWZ)
    return R * 16 + ((((c >> 1) ^ (R & 7)) << 1) | (c & 1));
  else
    return c + N * R;
}

template <int N, int G, int SGS, int KS, bool SUMSQ, bool SWZ = false,
          int ROW = N>
__global__ void __launch_bounds__(G *TcCfg<N>::T, 1)
    semlap_tc2_kernel(double *__restrict__ w, const double *__restrict__ u,
                      const double *__restrict__ g, int64_t nelt,
                      double *__restrict__ partials,
                      const __grid_constant__ CUtensorMap umap) {
  using C = TcCfg<N>;
  using L = Tc2Smem<N, G, SGS, KS, SWZ>;
  constexpr int NP = C::NP, T = C::T, KT = C::KT, P = C::P, SL = C::SL;
  constexpr int N2 = N * N;
  static_assert(N >= 7 && N <= 16, "n = 7..16");
  static_assert(N % KS == 0, "KS divides n");
  static_assert(G * (1 + SGS) <= 64 && G <= 15, "mbarriers, barrier ids");
  static_assert(!SWZ || N == 16, "swizzled staging: 128-B rows (n = 16)");

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = smem_raw;
  if constexpr (SWZ) {  // the swizzle pattern is of the absolute address
    const uint32_t a = smem_u32(smem_raw);
    smem += ((a + 1023u) & ~1023u) - a;
  }
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem);

  const int tid = threadIdx.x;
  const int grp = tid / T;
  const int lt = tid % T;
  const int warp = lt / 32, lane = lt % 32;
  const int it = warp / C::NT, jt = warp % C::NT;
  const int r = lane / 4, q = lane % 4;
  const int j = 8 * jt + r;          // accumulator row
  const int i0 = 8 * it + 2 * q;     // accumulator columns i0, i0 + 1
  const bool vj = j < N;
  const bool v0 = vj && i0 < N, v1 = vj && i0 + 1 < N;

  double *gb = reinterpret_cast<double *>(smem + L::bars +
                                          (size_t)grp * L::grp_bytes);
  double *ust0 = gb;                          // u of the element (+ lead)
  double *slabs = ust0 + L::UST;              // SGS x KS x 6 N^2
  double *wrr = slabs + SGS * KS * C::SLAB;   // wr: 2 padded slices
  double *wsr = wrr + 2 * SL;                 // ws: 2 padded slices
  uint64_t *ubar = bars + grp * (1 + SGS);
  uint64_t *gbar = ubar + 1;

  const int64_t q0 = (int64_t)blockIdx.x * G + grp;
  const int64_t Q = (int64_t)gridDim.x * G;
  const int64_t mine = nelt > q0 ? (nelt - q0 + Q - 1) / Q : 0;
  auto elem = [&](int64_t m) -> int64_t { return q0 + m * Q; };

  if (tid == 0) {
    for (int x = 0; x < G * (1 + SGS); ++x) mbar_init(&bars[x], 1);
    fence_mbar_init();
  }
  // zero all group smem once: padded / out-of-element fragment reads are
  // then finite (they meet zero d entries or feed unstored rows)
  for (int x = lt; x < (int)(L::grp_bytes / 8); x += T) gb[x] = 0.0;
  __syncthreads();

  const uint64_t pol = policy_evict_first();
  const int64_t u_bytes_total = nelt * NP * 8;
  auto u_lead = [&](int64_t e) -> int { return (int)((e * NP) & 1); };
  auto u_span = [&](int64_t e) -> int64_t {
    return ((int64_t)(u_lead(e) + NP) * 8 + 15) / 16 * 16;
  };
  auto u_bulk_ok = [&](int64_t e) -> bool {
    return (e * NP - u_lead(e)) * 8 + u_span(e) <= u_bytes_total;
  };
  auto issue_u = [&](int64_t m) {
    const int64_t e = elem(m);
    if constexpr (SWZ) {  // rows e N^2 .. e N^2 + N^2 - 1 of the (16 x rows) map
      mbar_arrive_expect_tx(ubar, (uint32_t)(NP * 8));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::"
          "complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(ust0)),
          "l"(&umap), "r"(0), "r"((int)(e * N2)), "r"(smem_u32(ubar))
          : "memory");
      return;
    }
    if (u_bulk_ok(e)) {
      mbar_arrive_expect_tx(ubar, (uint32_t)u_span(e));
      bulk_g2s_stream(ust0, u + e * NP - u_lead(e), (uint32_t)u_span(e),
                      ubar, pol);
    } else {
      mbar_arrive_expect_tx(ubar, 0);
    }
  };
  auto issue_slab = [&](int64_t sq) {
    const int64_t e = elem(sq / (N / KS));
    const int k0 = (int)(sq % (N / KS)) * KS;
    const int slot = (int)(sq % SGS);
    mbar_arrive_expect_tx(&gbar[slot], (uint32_t)(KS * C::SLAB * 8));
    bulk_g2s_stream(slabs + (size_t)slot * KS * C::SLAB,
                    g + e * 6 * NP + (int64_t)k0 * 6 * N2, KS * C::SLAB * 8,
                    &gbar[slot], pol);
  };
  const int64_t nslabs = mine * (N / KS);
  if (lt == 0) {
    if (mine > 0) issue_u(0);
    for (int64_t x = 0; x < SGS && x < nslabs; ++x) issue_slab(x);
  }

  // the contraction index of the phase-1 products for k-step ks, lane q:
  // 4 ks + q, or for odd n with four k-steps (13, 15) 4 q + ks -- then the
  // four q of a half warp read u rows 4 apart, and N x {0, 4, 8, 12} hits
  // four different bank quarters for odd N (the plain order was 2-way
  // conflicted in both fragment loads, ncu source view)
  constexpr bool RHO = KT == 4 && (N % 2 == 1);
  auto lk = [&](int ks) -> int { return RHO ? 4 * q + ks : 4 * ks + q; };
  double fa_r[KT], fb_s[KT], fa_t[KT], fb_t[KT];
#pragma unroll
  for (int ks = 0; ks < KT; ++ks) {
    fa_r[ks] = dtc<N, ROW>(8 * it + r, lk(ks));
    fb_s[ks] = dtc<N, ROW>(8 * jt + r, lk(ks));
    fa_t[ks] = dtc<N, ROW>(4 * ks + q, 8 * it + r);
    fb_t[ks] = dtc<N, ROW>(4 * ks + q, 8 * jt + r);
  }

  double acc_sq = 0.0;
  for (int64_t m = 0; m < mine; ++m) {
    const int64_t e = elem(m);
    mbar_wait(ubar, (uint32_t)(m & 1));
    const double *ust = SWZ ? ust0 : ust0 + u_lead(e);
    if (!SWZ && !u_bulk_ok(e)) {
      for (int x = lt; x < NP; x += T) ust0[u_lead(e) + x] = u[e * NP + x];
      named_bar_sync(1 + grp, T);
    }
    // ut for every k from the own columns (2N independent DFMA chains)
    double t0[N], t1[N];
    {
      double uc0[N], uc1[N];
#pragma unroll
      for (int l = 0; l < N; ++l) {
        uc0[l] = v0 ? ust[uidx<N, SWZ>(i0, j + N * l)] : 0.0;
        uc1[l] = v1 ? ust[uidx<N, SWZ>(i0 + 1, j + N * l)] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < N; ++k) t0[k] = t1[k] = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double dk = c_dtc[ROW][k + N * l];
          t0[k] = __fma_rn(dk, uc0[l], t0[k]);
          t1[k] = __fma_rn(dk, uc1[l], t1[k]);
        }
      }
    }

    double wt0[N], wt1[N], p0[N], p1[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int64_t s = m * N + k;
      // ---- phase 1, slice k: ur^T / us^T from the staged u (row stride N)
      double r0 = 0.0, r1 = 0.0, s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KT; ++ks) {
        dmma(r0, r1, ust[uidx<N, SWZ>(lk(ks), 8 * jt + r + N * k)],
             fa_r[ks]);
        dmma(s0, s1, fb_s[ks],
             ust[uidx<N, SWZ>(8 * it + r, lk(ks) + N * k)]);
      }
      if (k % KS == 0)
        mbar_wait(&gbar[(s / KS) % SGS], (uint32_t)((s / KS / SGS) & 1));
      const double *gs = slabs + (size_t)((s / KS) % SGS) * KS * C::SLAB +
                         (size_t)(k % KS) * C::SLAB;
      double *wr_k = wrr + (k & 1) * SL;
      double *ws_k = wsr + (k & 1) * SL;
      if (v0) {
        const double2 *g2 =
            reinterpret_cast<const double2 *>(gs + 6 * (i0 + N * j));
        const double2 g01 = g2[0], g23 = g2[1], g45 = g2[2];
        wr_k[i0 + P * j] = comb3<true>(g01.x, r0, g01.y, s0, g23.x, t0[k]);
        ws_k[i0 + P * j] = comb3<true>(g01.y, r0, g23.y, s0, g45.x, t0[k]);
        wt0[k] = comb3<true>(g23.x, r0, g45.x, s0, g45.y, t0[k]);
      } else {
        wt0[k] = 0.0;
      }
      if (v1) {
        const double2 *g2 =
            reinterpret_cast<const double2 *>(gs + 6 * (i0 + 1 + N * j));
        const double2 g01 = g2[0], g23 = g2[1], g45 = g2[2];
        wr_k[i0 + 1 + P * j] =
            comb3<true>(g01.x, r1, g01.y, s1, g23.x, t1[k]);
        ws_k[i0 + 1 + P * j] =
            comb3<true>(g01.y, r1, g23.y, s1, g45.x, t1[k]);
        wt1[k] = comb3<true>(g23.x, r1, g45.x, s1, g45.y, t1[k]);
      } else {
        wt1[k] = 0.0;
      }
      named_bar_sync(1 + grp, T);  // wr / ws of slice k complete
      if (k % KS == KS - 1) {       // slab consumed: refill
        const int64_t slab = s / KS;
        if (lt == 0 && slab + SGS < nslabs) {
          fence_proxy_async_smem();
          issue_slab(slab + SGS);
        }
      }
      if (k == N - 1 && lt == 0 && m + 1 < mine) {
        fence_proxy_async_smem();
        issue_u(m + 1);  // u consumed by every warp (barrier above)
      }
      // ---- phase 2 sums over wr / ws of slice k (tensor cores): two
      // independent accumulator chains (d^T.wr and ws.d), added at the end,
      // so the DMMA latency is paid over KT steps, not 2 KT
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KT; ++ks) {
        dmma(a0, a1, wr_k[(4 * ks + q) + P * (8 * jt + r)], fa_t[ks]);
        dmma(b0, b1, fb_t[ks], ws_k[(8 * it + r) + P * (4 * ks + q)]);
      }
      p0[k] = a0 + b0;
      p1[k] = a1 + b1;
    }
    // ---- the own-column sum over wt (needs every slice), then w
    double *we = w + e * NP;
#pragma unroll
    for (int l = 0; l < N; ++l) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double dk = c_dtc[ROW][l + N * k];
        p0[k] = __fma_rn(dk, wt0[l], p0[k]);
        p1[k] = __fma_rn(dk, wt1[l], p1[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      if (N % 2 == 0 && v1) {
        *reinterpret_cast<double2 *>(we + i0 + N * j + N2 * k) =
            make_double2(p0[k], p1[k]);
      } else {
        if (v0) we[i0 + N * j + N2 * k] = p0[k];
        if (v1) we[i0 + 1 + N * j + N2 * k] = p1[k];
      }
      if constexpr (SUMSQ) {
        if (v0) acc_sq = dadd(acc_sq, dmul(p0[k], p0[k]));
        if (v1) acc_sq = dadd(acc_sq, dmul(p1[k], p1[k]));
      }
    }
  }

  if constexpr (SUMSQ) block_sumsq_partial(acc_sq, partials);
}

// the (16 x rows) view of u for the swizzled staging (n = 16)
bool sem_u16_map(CUtensorMap *map, const double *u, int64_t nelt) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p,
                                    cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
               ? reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p)
               : nullptr;
  }();
  if (!encode || !aligned(u, 16) || nelt * 256 >= (int64_t(1) << 31))
    return false;
  cuuint64_t dims[2] = {16, (cuuint64_t)(nelt * 256)};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {16, 256};
  cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                const_cast<double *>(u), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int N>
static int slot_row(int slot) { return slot == 0 ? N : N + 10; }

template <int N, int G, int SGS, int KS, int ROW>
static void tc2_launch_row(bool sumsq, bool swz, int grid, size_t bytes,
                           double *w, const double *u, const double *g,
                           int64_t nelt, const lfb_launch *geom,
                           const CUtensorMap &umap, cudaStream_t s) {
  auto k = sumsq ? semlap_tc2_kernel<N, G, SGS, KS, true, false, ROW>
                 : semlap_tc2_kernel<N, G, SGS, KS, false, false, ROW>;
  auto ks = sumsq ? semlap_tc2_kernel<N, G, SGS, KS, true, N == 16, ROW>
                  : semlap_tc2_kernel<N, G, SGS, KS, false, N == 16, ROW>;
  cudaFuncSetAttribute(swz ? ks : k,
                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)bytes);
  (swz ? ks : k)<<<grid, G * TcCfg<N>::T, bytes, s>>>(
      w, u, g, nelt, sumsq ? geom->workspace : nullptr, umap);
}

template <int N, int G, int SGS, int KS>
static int launch_tc2(double *w, const double *u, const double *d,
                      const double *g, int64_t nelt, const lfb_launch *geom,
                      cudaStream_t s, int64_t *grid_out) {
  using L = Tc2Smem<N, G, SGS, KS>;
  using LS = Tc2Smem<N, G, SGS, KS, N == 16>;
  static_assert(L::total <= 227 * 1024 && LS::total <= 227 * 1024, "smem");
  int sms = sm_count(geom);
  if (sms <= 0) sms = 148;
  const int per_sm = (geom && geom->ctas_per_sm > 0) ? geom->ctas_per_sm : 1;
  int64_t grid64 = (int64_t)sms * per_sm;
  if (grid64 * G > nelt) grid64 = (nelt + G - 1) / G;
  const int grid = (int)(grid64 < 1 ? 1 : grid64);
  if (grid_out) {
    *grid_out = grid;
    return LFB_OK;
  }
  const bool sumsq = geom && geom->sumsq;
  if (sumsq && (!geom->workspace || geom->workspace_len < grid))
    return fail(LFB_ERR_ARG, "semlap: sumsq workspace too small");
  // n = 16: swizzled u staging when the tensor map encodes (geom->variant
  // 54 forces the plain staging, for the tests)
  alignas(64) CUtensorMap umap;
  memset(&umap, 0, sizeof(umap));
  const bool swz = N == 16 && !(geom && geom->variant == 54) &&
                   sem_u16_map(&umap, u, nelt);
  const size_t bytes = swz ? LS::total : L::total;
  {
    // two rotating constant slots per order (rows N and N + 10): one ring
    // per order, tag 8 + N
    std::unique_lock<std::mutex> lk;
    bool capturing = false;
    int slot = -2;
    if (int rc = dconst_acquire(c_dtc, 256 * 8, 8 + N, &slot, d, N, s, &lk,
                                &capturing, slot_row<N>))
      return rc;
    if (slot == 0)
      tc2_launch_row<N, G, SGS, KS, N>(sumsq, swz, grid, bytes, w, u, g,
                                       nelt, geom, umap, s);
    else
      tc2_launch_row<N, G, SGS, KS, N + 10>(sumsq, swz, grid, bytes, w, u,
                                            g, nelt, geom, umap, s);
    dconst_release(8 + N, slot, s, capturing);
  }
  if (int rc = check_launch("lfb_semlap_f64(dmma2)")) return rc;
  return sumsq ? sem_sumsq_finish(geom->workspace, grid, geom->sumsq, s)
               : LFB_OK;
}

// }}}

template <int N, int G, int SGS, int KS>
static int launch_tc(double *w, const double *u, const double *d,
                     const double *g, int64_t nelt, const lfb_launch *geom,
                     cudaStream_t s, int64_t *grid_out) {
  using L = TcSmem<N, G, SGS, KS>;
  static_assert(L::total <= 227 * 1024, "smem");
  int sms = sm_count(geom);
  if (sms <= 0) sms = 148;
  const int per_sm = (geom && geom->ctas_per_sm > 0) ? geom->ctas_per_sm : 1;
  int64_t grid64 = (int64_t)sms * per_sm;
  if (grid64 * G > nelt) grid64 = (nelt + G - 1) / G;
  const int grid = (int)(grid64 < 1 ? 1 : grid64);
  if (grid_out) {
    *grid_out = grid;
    return LFB_OK;
  }
  const bool sumsq = geom && geom->sumsq;
  if (sumsq && (!geom->workspace || geom->workspace_len < grid))
    return fail(LFB_ERR_ARG, "semlap: sumsq workspace too small");
  if (!aligned(u, 16) || !aligned(g, 16))
    return fail(LFB_ERR_UNSUPPORTED, "semlap(tc): u, g not 16-byte aligned");
  auto k = sumsq ? semlap_tc_kernel<N, G, SGS, KS, true>
                 : semlap_tc_kernel<N, G, SGS, KS, false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)L::total);
  {
    std::unique_lock<std::mutex> lk;
    bool capturing = false;
    int slot = 0;  // row N: slot 0 of the order's ring (launch_tc2)
    if (int rc = dconst_acquire(c_dtc, 256 * 8, 8 + N, &slot, d, N, s, &lk,
                                &capturing, slot_row<N>))
      return rc;
    k<<<grid, G * TcCfg<N>::T, L::total, s>>>(
        w, u, g, nelt, sumsq ? geom->workspace : nullptr);
    dconst_release(8 + N, slot, s, capturing);
  }
  if (int rc = check_launch("lfb_semlap_f64(dmma)")) return rc;
  return sumsq ? sem_sumsq_finish(geom->workspace, grid, geom->sumsq, s)
               : LFB_OK;
}

// (n, variant) -> (groups per CTA, g-slab ring depth, k-slices per slab).  Variant 51: the
// DMMA kernel; -1 when there is none for n.
#define LFB_TC_TABLE(X) \
  X(9, 51, 2, 3, 1)     \
  X(10, 51, 2, 2, 2)    \
  X(11, 51, 1, 4, 1)    \
  X(12, 51, 1, 3, 2)    \
  X(13, 51, 1, 4, 1)    \
  X(14, 51, 1, 2, 2)    \
  X(15, 51, 1, 4, 1)    \
  X(16, 51, 1, 2, 2)

// variant 52: the interleaved-phase kernel (groups, slab ring, slices/slab),
// tuned per n on B200 (3 groups = 12 warps/SM beat 2 despite small spills
// up to n = 15); 53: alternatives
#define LFB_TC2_TABLE(X) \
  X(7, 52, 12, 4, 1)     \
  X(8, 52, 6, 4, 2)      \
  X(8, 53, 7, 4, 2)      \
  X(9, 52, 3, 3, 1)      \
  X(10, 52, 3, 2, 2)     \
  X(11, 52, 3, 3, 1)     \
  X(12, 52, 3, 2, 2)     \
  X(13, 52, 3, 2, 1)     \
  X(14, 52, 3, 2, 1)     \
  X(15, 52, 3, 2, 1)     \
  X(16, 52, 2, 4, 1)     \
  X(16, 54, 2, 4, 1)     \
  X(12, 53, 2, 3, 2)     \
  X(13, 53, 2, 3, 1)     \
  X(14, 53, 2, 3, 1)     \
  X(15, 53, 2, 3, 1)     \
  X(16, 53, 2, 3, 1)

int sem_tc_dispatch(int n, int variant, double *w, const double *u,
                    const double *d, const double *g, int64_t nelt,
                    const lfb_launch *geom, cudaStream_t s,
                    int64_t *grid_out) {
#define X(NN, VV, GG, SS, KK)                                               \
  if (n == NN && variant == VV)                                             \
    return launch_tc<NN, GG, SS, KK>(w, u, d, g, nelt, geom, s, grid_out);
  LFB_TC_TABLE(X)
#undef X
#define X(NN, VV, GG, SS, KK)                                               \
  if (n == NN && variant == VV)                                             \
    return launch_tc2<NN, GG, SS, KK>(w, u, d, g, nelt, geom, s, grid_out);
  LFB_TC2_TABLE(X)
#undef X
  return -1;
}

}  // namespace lfb
