// SEM Laplacian, orders n = 9..16: phase 1 by *line owners* (variant 70
// bitwise -- the bitwise default at n = 13, 15, 16 --, 71 DFMA mode, 72 / 73
// other group counts and g-ring depths).
//
// Same reference arithmetic as every bitwise SEM kernel (SURVEY.md
// Appendix A, lf/interp.py:169-187; oracle/lf_oracle.c:59-94): ur, us, ut
// are separately rounded chains over l ascending, the combine is
// (g0 ur + g1 us) + g2 ut, and phase 2 is one chain per point with the three
// terms of each l interleaved.
//
// Why a new mapping: the column kernels (semlap_slab/gen, one k-column per
// thread) read one shared-memory operand per multiply-add in BOTH phases --
// the u row / column of ur / us and the wr row / ws column of phase 2 -- so
// at n >= 12 the L1 LSU pipe is as busy as the FP64 pipe (ncu n = 16: LSU
// 70 %, FP64 54 %, one 8-warp group per SM, profiles/r01_sem_hi_16_0.md).
// The three contractions of phase 1 are independent chains, so here each is
// computed by the thread that owns the whole input *line*:
//   thread t, (a, b) = (t % n, t / n):
//     i-line u(:, a, b) -> ur(:, a, b)   (n loads, n^2 multiply-adds)
//     j-line u(a, :, b) -> us(a, :, b)
//     k-line u(a, b, :) -> ut(a, b, :)   (the line kept in registers)
// Every d(x, l) of these is warp-uniform -- x and l are unrolled -- so it
// comes from the constant bank (dconst.cuh; sm_100a's DMUL takes no c-bank
// operand, ptxas loads it with LDCU / LDC), and each thread runs n
// independent chains: phase 1 costs n loads per n^2 multiply-adds instead of
// one per multiply-add.  ur / us go to shared memory; the point owner (i, j)
// (= the k-line owner) walks the slices k: it contracts its k-line for
// ut(i, j, k) (n < 16: this FP64 work hides the wait for the g slice; at
// n = 16 ut is contracted in phase 1, inside the combine ptxas spilled phase
// 2), combines with g, writes wr / ws in place and keeps wt(i, j, :) in
// registers for phase 2, which stays a point chain (bitwise parity fixes
// its interleaving): wr row + ws column from shared memory, d(l, i),
// d(l, j) from shared memory per l, d(l, k) from the constant bank.
//
// Shared memory per element group:
//   ua  u of the element (1-D bulk copy with the odd-n 8-byte lead, or for
//       n = 16 a 2-D TMA tensor load with the 128-B swizzle), reused as g
//       slots SD..S-1 once phase 1 has read u;
//   gd  SD dedicated g slots (prefetched for the next element during
//       phase 2 and phase 1);
//   rr, ss  ur -> wr and us -> ws, row = (j + n k), padded row stride P
//       (P = 2 mod 4 doubles: the lines of 8 lanes land on 8 distinct
//       16-byte bank groups) or, at n = 16, P = 16 with an XOR swizzle of
//       the 16-byte column chunks (the padding would not fit two groups).
// g is streamed one k-slice (6 n^2 doubles) per bulk copy through the S-slot
// ring during the combine; the next element's u is issued after the last
// slice, so it lands during phase 2 (and the TMA engine prefetches the next
// element's g and u into L2 at the start of each element: +2 %).
#include <string.h>

#include "dconst.cuh"
#include "lfb_common.cuh"
#include "semlap_common.cuh"

namespace lfb {

// d(a,b) at c_dline[N - 9][a + N b] for the order being launched
// (dconst.cuh)
__constant__ double c_dline[8][256];
#define LINE_D(a_plus_nb) c_dline[N - 9][a_plus_nb]

constexpr int line_pad(int n) {  // even, = 2 mod 4, >= n
  return (n + (n & 1)) % 4 == 2 ? n + (n & 1) : n + (n & 1) + 2;
}

template <int N>
struct LineCfg {
  static constexpr int N2 = N * N;
  static constexpr int NP = N * N * N;
  static constexpr int T = ((N2 + 31) / 32) * 32;
  static constexpr bool RSW = N == 16;              // rr/ss XOR swizzle
  static constexpr int P = RSW ? 16 : line_pad(N);  // rr/ss row stride
  static constexpr int RS = P * N2;                 // one of rr / ss
  static constexpr int SLAB = 6 * N2;               // g of one k-slice
};

template <int N, int G, bool USW, int SD = 1>
struct LineSmem {
  using C = LineCfg<N>;
  static constexpr int UST = USW ? C::NP : (C::NP + 2 + 1) / 2 * 2;
  static constexpr int SGU = UST / C::SLAB;  // g slots inside ua
  // SD dedicated slots (prefetched for the next element during phase 2 and
  // phase 1), then the slots inside the dead u stage
  static constexpr int S = (SD + SGU) < N ? SD + SGU : N;
  static constexpr size_t align = USW ? 1024 : 128;
  static constexpr size_t ua_off = 0;
  static constexpr size_t gd_off = ((size_t)UST * 8 + 127) / 128 * 128;
  static constexpr size_t rr_off = gd_off + (size_t)SD * C::SLAB * 8;
  static constexpr size_t ss_off = rr_off + (size_t)C::RS * 8;
  static constexpr size_t grp_bytes =
      (ss_off + (size_t)C::RS * 8 + align - 1) / align * align;
  static constexpr size_t head =  // mbarriers (512 B) + d (N^2 doubles)
      (512 + (size_t)C::N2 * 8 + align - 1) / align * align;
  static constexpr size_t total = head + G * grp_bytes + (USW ? 1024 : 0);
};

// u(c, R), R = j + N k the row, in the staged element: plain, or (USW) the
// TMA 128-B swizzle (16-byte chunk c/2 of row R XOR R mod 8)
template <int N, bool USW>
__device__ __forceinline__ int line_uidx(int c, int R) {
  if constexpr (USW)
    return R * 16 + ((((c >> 1) ^ (R & 7)) << 1) | (c & 1));
  else
    return c + N * R;
}

// ur / us / wr / ws (c, row) in rr / ss
template <int N>
__device__ __forceinline__ int line_ridx(int c, int row) {
  using C = LineCfg<N>;
  if constexpr (C::RSW)
    return row * 16 + ((((c >> 1) ^ (row & 7)) << 1) | (c & 1));
  else
    return c + C::P * row;
}

// out[a] = sum_l d(a, l) in[l], l ascending: N independent chains, every
// d(a, l) a constant-bank operand
template <int N, bool F>
__device__ __forceinline__ void line_contract(const double (&in)[N],
                                              double (&out)[N]) {
#pragma unroll
  for (int a = 0; a < N; ++a) out[a] = mac0<F>(LINE_D(a), in[0]);
#pragma unroll
  for (int l = 1; l < N; ++l) {
#pragma unroll
    for (int a = 0; a < N; ++a)
      out[a] = mac<F>(out[a], LINE_D(a + N * l), in[l]);
  }
}

template <int N, int G, bool USW, bool SUMSQ, bool F, bool PF, int SD>
__global__ void __launch_bounds__(G *LineCfg<N>::T, 1)
    semlap_line_kernel(double *__restrict__ w, const double *__restrict__ u,
                       const double *__restrict__ d,
                       const double *__restrict__ g, int64_t nelt,
                       double *__restrict__ partials,
                       const __grid_constant__ CUtensorMap umap) {
  using C = LineCfg<N>;
  using L = LineSmem<N, G, USW, SD>;
  constexpr int N2 = C::N2, NP = C::NP, T = C::T, S = L::S;
  static_assert(SD >= 1 && SD <= S, "dedicated slots");
  constexpr bool UTC = N < 16;  // ut contracted inside the combine
  static_assert(N >= 9 && N <= 16, "n = 9..16");
  static_assert(G * (1 + S) <= 63 && G <= 15, "mbarriers, barrier ids");
  static_assert(!USW || N == 16, "swizzled u staging: 128-B rows");

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = smem_raw;
  if constexpr (USW) {  // the swizzle pattern is of the absolute address
    const uint32_t a = smem_u32(smem_raw);
    smem += ((a + 1023u) & ~1023u) - a;
  }
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem);
  double *dn = reinterpret_cast<double *>(smem + 512);  // d(a,b) @ b + N a

  const int tid = threadIdx.x;
  const int grp = tid / T;
  const int lt = tid % T;
  const bool active = lt < N2;
  const int ta = lt % N, tb = lt / N;  // the thread's line / point (a, b)

  unsigned char *gbase = smem + L::head + (size_t)grp * L::grp_bytes;
  double *ua = reinterpret_cast<double *>(gbase + L::ua_off);
  double *gd = reinterpret_cast<double *>(gbase + L::gd_off);
  double *rr = reinterpret_cast<double *>(gbase + L::rr_off);
  double *ss = reinterpret_cast<double *>(gbase + L::ss_off);
  uint64_t *ubar = bars + grp * (1 + S);
  uint64_t *zero = bars + 63;  // holds 0 (see phase 2)
  uint64_t *gbar = ubar + 1;
  auto slot_ptr = [&](int s) -> double * {
    return s < SD ? gd + (size_t)s * C::SLAB : ua + (size_t)(s - SD) * C::SLAB;
  };

  const int64_t q0 = (int64_t)blockIdx.x * G + grp;
  const int64_t Q = (int64_t)gridDim.x * G;
  const int64_t mine = nelt > q0 ? (nelt - q0 + Q - 1) / Q : 0;
  auto elem = [&](int64_t m) -> int64_t { return q0 + m * Q; };

  if (tid == 0) {
    for (int x = 0; x < G * (1 + S); ++x) mbar_init(&bars[x], 1);
    *zero = 0;
    fence_mbar_init();
  }
  for (int x = tid; x < N2; x += G * T) dn[(x / N) + N * (x % N)] = d[x];
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
    if constexpr (USW) {  // rows e N^2 .. of the (16 x rows) map
      mbar_arrive_expect_tx(ubar, (uint32_t)(NP * 8));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::"
          "complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(ua)),
          "l"(&umap), "r"(0), "r"((int)(e * N2)), "r"(smem_u32(ubar))
          : "memory");
    } else if (u_bulk_ok(e)) {
      mbar_arrive_expect_tx(ubar, (uint32_t)u_span(e));
      bulk_g2s_stream(ua, u + e * NP - u_lead(e), (uint32_t)u_span(e), ubar,
                      pol);
    } else {
      mbar_arrive_expect_tx(ubar, 0);  // the threads copy it themselves
    }
  };
  // ring: k-slice k of element m -> slot k % S
  auto issue_slice = [&](int64_t m, int k) {
    const int s = k % S;
    mbar_arrive_expect_tx(&gbar[s], (uint32_t)(C::SLAB * 8));
    bulk_g2s_stream(slot_ptr(s), g + elem(m) * 6 * NP + (int64_t)k * C::SLAB,
                    C::SLAB * 8, &gbar[s], pol);
  };
  auto slice_parity = [&](int64_t m, int k) -> uint32_t {
    const int s = k % S;
    const int64_t per = (N - s + S - 1) / S;  // uses of slot s per element
    return (uint32_t)((m * per + k / S) & 1);
  };

  if (lt == 0 && mine > 0) {
    issue_u(0);
    for (int k = 0; k < SD; ++k) issue_slice(0, k);
  }

  double acc_sq = 0.0;
  for (int64_t m = 0; m < mine; ++m) {
    const int64_t e = elem(m);
    if (PF && lt == 0 && m + 1 < mine) {
      // the next element's g (and u) into L2 now: HBM streams evenly and the
      // burst of g reads in the next combine hits L2
      const int64_t e1 = elem(m + 1);
      bulk_prefetch_l2(g + e1 * 6 * NP, 6 * NP * 8);
      const int64_t u0 = (e1 * NP) & ~(int64_t)1;
      const int64_t u1 = ((e1 + 1) * NP + 1) & ~(int64_t)1;
      if (u1 * 8 <= u_bytes_total)
        bulk_prefetch_l2(u + u0, (uint32_t)((u1 - u0) * 8));
    }
    mbar_wait(ubar, (uint32_t)(m & 1));
    const double *ust = USW ? ua : ua + u_lead(e);
    if (!USW && !u_bulk_ok(e)) {
      for (int x = lt; x < NP; x += T) ua[u_lead(e) + x] = u[e * NP + x];
      named_bar_sync(1 + grp, T);
    }

    // ---- phase 1: the thread's three lines
    double uc[N];
    if (active) {
      double in[N], out[N];
      // i-line u(:, a, b), row R = lt
#pragma unroll
      for (int l = 0; l < N; l += 2) {
        if (N % 2 == 0) {
          const double2 v = *reinterpret_cast<const double2 *>(
              ust + line_uidx<N, USW>(l, lt));
          in[l] = v.x, in[l + 1] = v.y;
        } else {
          in[l] = ust[line_uidx<N, USW>(l, lt)];
          if (l + 1 < N) in[l + 1] = ust[line_uidx<N, USW>(l + 1, lt)];
        }
      }
      line_contract<N, F>(in, out);
#pragma unroll
      for (int x = 0; x < N; x += 2) {
        if (x + 1 < N) {
          *reinterpret_cast<double2 *>(rr + line_ridx<N>(x, lt)) =
              make_double2(out[x], out[x + 1]);
        } else {
          rr[line_ridx<N>(x, lt)] = out[x];
        }
      }
      // j-line u(a, :, b): rows l + N b
#pragma unroll
      for (int l = 0; l < N; ++l) in[l] = ust[line_uidx<N, USW>(ta, l + N * tb)];
      line_contract<N, F>(in, out);
#pragma unroll
      for (int x = 0; x < N; ++x) ss[line_ridx<N>(ta, x + N * tb)] = out[x];
      // k-line u(a, b, :): rows b + N l.  UTC: kept, its contraction runs
      // slice by slice inside the combine where it hides the g-slice
      // latency (n < 16: +1..13 %); n = 16: contracted here (inside the
      // combine ptxas spilled phase 2 under the 128-register cap)
#pragma unroll
      for (int l = 0; l < N; ++l) uc[l] = ust[line_uidx<N, USW>(ta, tb + N * l)];
      if constexpr (!UTC) {
        double t[N];
        line_contract<N, F>(uc, t);
#pragma unroll
        for (int l = 0; l < N; ++l) uc[l] = t[l];  // uc now holds ut
      }
    }
    named_bar_sync(1 + grp, T);  // u read by all; ur / us complete
    if (lt == 0) {
      fence_proxy_async_smem();
      for (int k = SD; k < S; ++k) issue_slice(m, k);  // slots inside ua
    }

    // ---- combine with g, slice by slice: wr / ws in place, wt in registers
    double wt[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int s = k % S;
      mbar_wait(&gbar[s], slice_parity(m, k));
      if (active) {
        const double2 *g2 =
            reinterpret_cast<const double2 *>(slot_ptr(s) + 6 * lt);
        const double2 g01 = g2[0], g23 = g2[1], g45 = g2[2];
        const int x = line_ridx<N>(ta, tb + N * k);
        const double ur = rr[x], us = ss[x];
        // ut(i, j, k) = sum_l d(k, l) u(i, j, l), l ascending
        double ut;
        if constexpr (UTC) {
          ut = mac0<F>(LINE_D(k), uc[0]);
#pragma unroll
          for (int l = 1; l < N; ++l) ut = mac<F>(ut, LINE_D(k + N * l), uc[l]);
        } else {
          ut = uc[k];
        }
        rr[x] = comb3<F>(g01.x, ur, g01.y, us, g23.x, ut);
        ss[x] = comb3<F>(g01.y, ur, g23.y, us, g45.x, ut);
        wt[k] = comb3<F>(g23.x, ur, g45.x, us, g45.y, ut);
      }
      named_bar_sync(1 + grp, T);  // slot s consumed (last: wr/ws complete)
      if (lt == 0) {
        if (k + S < N) {
          fence_proxy_async_smem();
          issue_slice(m, k + S);
        } else if (s < SD && m + 1 < mine) {
          fence_proxy_async_smem();
          issue_slice(m + 1, s);  // dedicated: the next element's first
        }
        if (k == N - 1 && m + 1 < mine) {
          fence_proxy_async_smem();
          issue_u(m + 1);  // lands during phase 2
        }
      }
    }

    // ---- phase 2: one chain per point, the three terms of each l in
    // turn; l outer, k inner: the thread's N chains advance together, only
    // wt, the accumulators and d(l, i), d(l, j) of the current l pair live
    if (active) {
      double sacc[N];
#pragma unroll
      for (int k = 0; k < N; ++k) sacc[k] = 0.0;
#pragma unroll
      for (int l = 0; l < N; l += 2) {
        constexpr int H = 2;
        double da[H], db[H];  // d(l + h, i), d(l + h, j)
        // wt(l) XOR a zero from a volatile shared load, per l pair
        // (bit-exact): ptxas would otherwise compute all n^2 products
        // d(l, k) wt(l) up front and spill them
        uint64_t z;
        asm volatile("ld.volatile.shared.u64 %0, [%1];"
                     : "=l"(z)
                     : "r"(smem_u32(zero)));
#pragma unroll
        for (int h = 0; h < H; ++h)
          if (l + h < N) {
            da[h] = dn[ta + N * (l + h)], db[h] = dn[tb + N * (l + h)];
            wt[l + h] = __longlong_as_double(
                __double_as_longlong(wt[l + h]) ^ (long long)z);
          }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const int rrow = tb + N * k;  // wr(:, j, k)
          double r0, r1 = 0.0;
          if (l + 1 < N) {
            const double2 v = *reinterpret_cast<const double2 *>(
                rr + line_ridx<N>(l, rrow));
            r0 = v.x, r1 = v.y;
          } else {
            r0 = rr[line_ridx<N>(l, rrow)];
          }
#pragma unroll
          for (int h = 0; h < H && l + h < N; ++h) {
            const int ll = l + h;
            sacc[k] = mac<F>(sacc[k], da[h], h ? r1 : r0);
            sacc[k] = mac<F>(sacc[k], db[h], ss[line_ridx<N>(ta, ll + N * k)]);
            sacc[k] = mac<F>(sacc[k], LINE_D(ll + N * k), wt[ll]);
          }
        }
      }
      double *we = w + e * NP + lt;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        we[N2 * k] = sacc[k];
        if constexpr (SUMSQ) acc_sq = dadd(acc_sq, dmul(sacc[k], sacc[k]));
      }
    }
    named_bar_sync(1 + grp, T);  // rr / ss read: free for the next element
  }

  if constexpr (SUMSQ) block_sumsq_partial(acc_sq, partials);
}

template <int N, int G, bool USW, bool F, bool PF, int SD>
static void line_launch(bool sumsq, int grid, double *w, const double *u,
                        const double *d, const double *g, int64_t nelt,
                        const lfb_launch *geom, const CUtensorMap &umap,
                        cudaStream_t s) {
  using L = LineSmem<N, G, USW, SD>;
  static_assert(L::total <= 227 * 1024, "smem");
  auto k = sumsq ? semlap_line_kernel<N, G, USW, true, F, PF, SD>
                 : semlap_line_kernel<N, G, USW, false, F, PF, SD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)L::total);
  k<<<grid, G * LineCfg<N>::T, L::total, s>>>(
      w, u, d, g, nelt, sumsq ? geom->workspace : nullptr, umap);
}

template <int N, int G, bool F, int SD = 1, bool PF = true>
static int launch_line(double *w, const double *u, const double *d,
                       const double *g, int64_t nelt, const lfb_launch *geom,
                       cudaStream_t s, int64_t *grid_out) {
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
  alignas(64) CUtensorMap umap;
  memset(&umap, 0, sizeof(umap));
  const bool usw = N == 16 && sem_u16_map(&umap, u, nelt);
  {
    std::unique_lock<std::mutex> lk;
    bool capturing = false;
    int slot = N - 9;  // one constant slot per order
    if (int rc = dconst_acquire(c_dline, 256 * 8, 3, &slot, d, N, s, &lk,
                                &capturing))
      return rc;
    if (usw)
      line_launch<N, G, N == 16, F, PF, SD>(sumsq, grid, w, u, d, g, nelt,
                                            geom, umap, s);
    else
      line_launch<N, G, false, F, PF, SD>(sumsq, grid, w, u, d, g, nelt,
                                          geom, umap, s);
    dconst_release(3, slot, s, capturing);
  }
  if (int rc = check_launch("lfb_semlap_f64(line)")) return rc;
  return sumsq ? sem_sumsq_finish(geom->workspace, grid, geom->sumsq, s)
               : LFB_OK;
}

// (n, variant) -> (groups per CTA, dedicated g slots).  70: bitwise, 71:
// the same in DFMA mode, 72: bitwise with (GB, SDB), 73: bitwise with one
// dedicated slot (the first ring)
#define LFB_LINE_TABLE(X)  \
  X(9, 4, 3, 6, 1)         \
  X(10, 4, 3, 6, 1)        \
  X(11, 3, 4, 4, 1)        \
  X(12, 3, 4, 4, 1)        \
  X(13, 2, 7, 3, 1)        \
  X(14, 2, 4, 3, 1)        \
  X(15, 2, 1, 1, 1)        \
  X(16, 2, 1, 1, 1)

int sem_line_dispatch(int n, int variant, double *w, const double *u,
                      const double *d, const double *g, int64_t nelt,
                      const lfb_launch *geom, cudaStream_t s,
                      int64_t *grid_out) {
#define X(NN, GA, SA, GB, SB)                                                \
  if (n == NN && variant == 70)                                              \
    return launch_line<NN, GA, false, SA>(w, u, d, g, nelt, geom, s,         \
                                          grid_out);                         \
  if (n == NN && variant == 71)                                              \
    return launch_line<NN, GA, true, SA>(w, u, d, g, nelt, geom, s,          \
                                         grid_out);                          \
  if (n == NN && variant == 72)                                              \
    return launch_line<NN, GB, false, SB>(w, u, d, g, nelt, geom, s,         \
                                          grid_out);                         \
  if (n == NN && variant == 73)                                              \
    return launch_line<NN, GA, false, 1>(w, u, d, g, nelt, geom, s,          \
                                         grid_out);
  LFB_LINE_TABLE(X)
#undef X
  return -1;
}

}  // namespace lfb
