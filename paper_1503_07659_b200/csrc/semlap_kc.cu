// SEM Laplacian, even orders: d in the constant bank (BASELINE configs 3/4,
// n = 8 default).
//
// Same reference arithmetic as semlap.cu (every * and +
// rounded separately, l ascending, left-associative sums), so the result is
// bitwise the reference's.
//
// Why a second n = 8 kernel: ncu on semlap_kernel (profiles/r01_sem65k.md)
// shows the L1 LSU data pipe at 95 % of peak -- the kernel is bound by
// shared-memory *instructions*, not bytes (bank reads 20 %).  Every warp-wide
// LDS costs >= 2 wavefronts however few distinct addresses it touches, and a
// third of them were broadcasts of d(k,.) / d(.,k) that are identical in all
// lanes.  This kernel removes those and the other avoidable wavefronts:
//  * d lives in a __constant__ slot; the unrolled loops index it with
//    compile-time offsets, so d(k,l) comes through the constant cache
//    (LDCU into a uniform register, dconst.cuh) -- no LDS on the LSU data
//    pipe.  The slot is filled by a
//    stream-ordered device-to-device copy before the launch; a ring of
//    KC_SLOTS slots with one event each keeps launches on other streams
//    from overwriting a slot a running kernel still reads (dconst.cuh).
//  * the per-thread d rows d(i,.), d(j,.) (phase 1) and d(.,i), d(.,j)
//    (phase 2) are registers, loaded per phase from the constant slot;
//  * u is transposed once per element into uT so the u(i,.,k) columns are
//    16-byte pairs, and ws is stored transposed the same way (row stride
//    N + 2: conflict-free for a half warp's 8 i values);
//  * wr is stored unpadded (row stride N): a half warp's two j rows then
//    fill the 16 double slots of a 128-byte line exactly, no conflict.
// Everything else follows semlap_kernel: persistent CTAs of G groups of n^2
// threads, thread (i,j) owns the k-column (i,j,*), u + g of a whole element
// by bulk copies (TMA engine) into an SG-deep per-group ring.
#include "dconst.cuh"
#include "lfb_common.cuh"
#include "semlap_common.cuh"

namespace lfb {

constexpr int KC_SLOTS = 4;
constexpr int KC_MAXN2 = 16 * 16;

__constant__ double c_dmat[KC_SLOTS][KC_MAXN2];  // d(a,b) at a + N b

template <int N>
struct KcCfg {
  static constexpr int N2 = N * N;
  static constexpr int NP = N * N * N;
  static constexpr int T = ((N2 + 31) / 32) * 32;
  static constexpr int R1 = N;      // wr row stride
  static constexpr int R2 = N + 2;  // wsT / uT row stride
  static constexpr int WR = N * N * N;
  static constexpr int WS = R2 * N * N;
  static constexpr int STAGE = 7 * NP;  // u then g
};

template <int N, int G, int SG>
struct KcSmem {
  using C = KcCfg<N>;
  static constexpr size_t bars = 128;
  static constexpr size_t scr_off = bars;
  static constexpr size_t grp_scr = (size_t)(C::WR + 2 * C::WS);  // doubles
  static constexpr size_t stage_off =
      ((scr_off + (size_t)G * grp_scr * 8) + 127) / 128 * 128;
  static constexpr size_t total = stage_off + (size_t)G * SG * C::STAGE * 8;
};

template <int SLOT, int N>
__device__ __forceinline__ double cd(int a, int b) {
  return c_dmat[SLOT][a + N * b];
}

template <int N, int G, int SG, int SLOT, bool SUMSQ, bool F>
__global__ void __launch_bounds__(G *KcCfg<N>::T, 1)
    semlap_kc_kernel(double *__restrict__ w, const double *__restrict__ u,
                     const double *__restrict__ g, int64_t nelt,
                     double *__restrict__ partials) {
  using C = KcCfg<N>;
  using L = KcSmem<N, G, SG>;
  constexpr int NP = C::NP, T = C::T, R1 = C::R1, R2 = C::R2;
  static_assert(G * SG <= 16, "too many stages");
  static_assert(N % 2 == 0, "paired loads need even n");

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem);
  double *scr = reinterpret_cast<double *>(smem + L::scr_off);
  double *stages = reinterpret_cast<double *>(smem + L::stage_off);

  const int tid = threadIdx.x;
  const int grp = tid / T;
  const int lt = tid % T;
  const int i = lt % N;
  const int j = lt / N;
  const bool active = lt < N * N;
  // interleaved persistent order: concurrently streamed elements are adjacent
  const int64_t ebase = blockIdx.x, estride = gridDim.x;
  const int64_t count =
      nelt > ebase ? (nelt - ebase + estride - 1) / estride : 0;

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
      if (t < count) issue(grp * SG + m, ebase + t * estride);
    }
  }


  double *wr = scr + (size_t)grp * L::grp_scr;  // wr(i,j,k) @ i + N j + N^2 k
  double *wsT = wr + C::WR;                     // ws(i,j,k) @ j + R2 i + R2 N k
  double *uT = wsT + C::WS;                     // u (i,j,k) @ j + R2 i + R2 N k
  double acc = 0.0;

  for (int m = 0;; ++m) {
    const int64_t t = grp + (int64_t)G * m;
    if (t >= count) break;
    const int64_t e = ebase + t * estride;
    const int st = grp * SG + (m % SG);
    mbar_wait(&bars[st], (uint32_t)((m / SG) & 1));
    const double *su = stages + (size_t)st * C::STAGE;
    const double *sg = su + NP;

    double ucol[N], wt[N];
    if (active) {
#pragma unroll
      for (int l = 0; l < N; ++l) ucol[l] = su[i + N * j + N * N * l];
#pragma unroll
      for (int k = 0; k < N; ++k) uT[j + R2 * i + R2 * N * k] = ucol[k];
    }
    named_bar_sync(1 + grp, T);  // uT complete

    if (active) {
      // per-thread d rows for phase 1 (constant-cache loads, no LSU traffic)
      double d1a[N], d1b[N];
#pragma unroll
      for (int l = 0; l < N; ++l) {
        d1a[l] = cd<SLOT, N>(i, l);  // d(i,l)
        d1b[l] = cd<SLOT, N>(j, l);  // d(j,l)
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double ur, us, ut;
        const double *row = su + N * j + N * N * k;    // u(.,j,k)
        const double *col = uT + R2 * i + R2 * N * k;  // u(i,.,k)
#pragma unroll
        for (int l = 0; l < N; l += 2) {
          const double2 r2 = *reinterpret_cast<const double2 *>(row + l);
          const double2 c2 = *reinterpret_cast<const double2 *>(col + l);
          if (l == 0) {  // ur = 0 + d*u ... (the reference's s = 0 start)
            ur = mac0<F>(d1a[0], r2.x);
            us = mac0<F>(d1b[0], c2.x);
            ut = mac0<F>(cd<SLOT, N>(k, 0), ucol[0]);
          } else {
            ur = mac<F>(ur, d1a[l], r2.x);
            us = mac<F>(us, d1b[l], c2.x);
            ut = mac<F>(ut, cd<SLOT, N>(k, l), ucol[l]);
          }
          ur = mac<F>(ur, d1a[l + 1], r2.y);
          us = mac<F>(us, d1b[l + 1], c2.y);
          ut = mac<F>(ut, cd<SLOT, N>(k, l + 1), ucol[l + 1]);
        }
        const double2 *g2 =
            reinterpret_cast<const double2 *>(sg + 6 * (i + N * j + N * N * k));
        const double2 g01 = g2[0], g23 = g2[1], g45 = g2[2];
        wr[i + N * j + N * N * k] =
            comb3<F>(g01.x, ur, g01.y, us, g23.x, ut);
        wsT[j + R2 * i + R2 * N * k] = comb3<F>(g01.y, ur, g23.y, us, g45.x, ut);
        wt[k] = comb3<F>(g23.x, ur, g45.x, us, g45.y, ut);
      }
    }
    named_bar_sync(1 + grp, T);  // stage consumed, scratch complete

    if (lt == 0) {
      const int64_t tn = t + (int64_t)G * SG;
      if (tn < count) {
        fence_proxy_async_smem();
        issue(st, ebase + tn * estride);
      }
    }

    if (active) {
      double d2a[N], d2b[N];
#pragma unroll
      for (int l = 0; l < N; ++l) {
        d2a[l] = cd<SLOT, N>(l, i);  // d(l,i)
        d2b[l] = cd<SLOT, N>(l, j);  // d(l,j)
      }
      double *we = w + e * NP + i + N * j;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double *rr = wr + R1 * j + N * N * k;    // wr(.,j,k)
        const double *rs = wsT + R2 * i + R2 * N * k;  // ws(i,.,k)
        double s;
#pragma unroll
        for (int l = 0; l < N; l += 2) {
          const double2 r2 = *reinterpret_cast<const double2 *>(rr + l);
          const double2 s2 = *reinterpret_cast<const double2 *>(rs + l);
          s = mac<F>(mac<F>(l == 0 ? mac0<F>(d2a[0], r2.x)
                                   : mac<F>(s, d2a[l], r2.x),
                            d2b[l], s2.x),
                     cd<SLOT, N>(l, k), wt[l]);
          s = mac<F>(mac<F>(mac<F>(s, d2a[l + 1], r2.y), d2b[l + 1], s2.y),
                     cd<SLOT, N>(l + 1, k), wt[l + 1]);
        }
        we[N * N * k] = s;
        if constexpr (SUMSQ) acc = dadd(acc, dmul(s, s));
      }
    }
    named_bar_sync(1 + grp, T);  // scratch reads done before the next element
  }

  if constexpr (SUMSQ) block_sumsq_partial(acc, partials);
}

template <int N, int G, int SG, int SLOT, bool F>
static void kc_launch_slot(bool sumsq, int grid, size_t smem, double *w,
                           const double *u, const double *g, int64_t nelt,
                           double *partials, cudaStream_t s) {
  auto k = sumsq ? semlap_kc_kernel<N, G, SG, SLOT, true, F>
                 : semlap_kc_kernel<N, G, SG, SLOT, false, F>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  k<<<grid, G * KcCfg<N>::T, smem, s>>>(w, u, g, nelt, partials);
}

template <int N, int G, int SG, bool F>
static int launch_kc(double *w, const double *u, const double *d,
                     const double *g, int64_t nelt, const lfb_launch *geom,
                     cudaStream_t s, int64_t *grid_out) {
  using L = KcSmem<N, G, SG>;
  static_assert(L::total <= 227 * 1024, "smem");
  static_assert(N * N <= KC_MAXN2, "constant slot");
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
  double *part = sumsq ? geom->workspace : nullptr;
  std::unique_lock<std::mutex> lk;
  bool capturing = false;
  int slot = -KC_SLOTS;  // rotate over the slots
  if (int rc = dconst_acquire(c_dmat, KC_MAXN2 * 8, 0, &slot, d, N, s, &lk,
                              &capturing))
    return rc;
  switch (slot) {
    case 0: kc_launch_slot<N, G, SG, 0, F>(sumsq, grid, L::total, w, u, g, nelt, part, s); break;
    case 1: kc_launch_slot<N, G, SG, 1, F>(sumsq, grid, L::total, w, u, g, nelt, part, s); break;
    case 2: kc_launch_slot<N, G, SG, 2, F>(sumsq, grid, L::total, w, u, g, nelt, part, s); break;
    default: kc_launch_slot<N, G, SG, 3, F>(sumsq, grid, L::total, w, u, g, nelt, part, s); break;
  }
  dconst_release(0, slot, s, capturing);
  lk.unlock();
  if (int rc = check_launch("lfb_semlap_f64")) return rc;
  return sumsq ? sem_sumsq_finish(geom->workspace, grid, geom->sumsq, s)
               : LFB_OK;
}

// (n, variant) -> (G, SG, fma).  -1: no constant-bank entry.  Variant 55 =
// the default configuration in DFMA mode (semlap_common.cuh); the DFMA-mode
// default at n = 8 (variant 50) is the DMMA kernel (semlap_tc.cu), which
// draws less power in sustained runs.
#define LFB_KC_TABLE(X) \
  X(8, 0, 4, 1, false)  \
  X(8, 40, 4, 1, false) \
  X(8, 41, 5, 1, false) \
  X(8, 42, 3, 2, false) \
  X(8, 55, 4, 1, true)

int sem_kc_dispatch(int n, int variant, double *w, const double *u,
                    const double *d, const double *g, int64_t nelt,
                    const lfb_launch *geom, cudaStream_t s,
                    int64_t *grid_out) {

#define X(NN, VV, GG, SS, FF)                                               \
  if (n == NN && variant == VV)                                             \
    return launch_kc<NN, GG, SS, FF>(w, u, d, g, nelt, geom, s, grid_out);
  LFB_KC_TABLE(X)
#undef X
  return -1;
}

}  // namespace lfb
