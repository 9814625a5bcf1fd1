// sgemm on the 5th-generation tensor cores: tcgen05.mma kind::tf32 with the
// 3xTF32 split (BASELINE config 5, fast mode).
//
// Reference: c(i,j) = c(i,j) + alpha*b(k,j)*a(i,k), k ascending, fp32
// (test_fortran.py:72-103 in real*4).  Tensor cores cannot reproduce the
// reference's k-sequential rounding, so this path is tolerance parity
// (normwise fp32 error vs the reference; the bit-exact mode is
// gemm_simt.cu).  Accuracy: each fp32 operand x is split x = hi + lo with
// hi = rna_tf32(x), lo = x - hi (exact); the product a*b is formed as
// hi_a*hi_b + hi_a*lo_b + lo_a*hi_b on the tensor pipe (the lo*lo term is
// below fp32 resolution).  The tensor pipe's fp32 accumulation truncates,
// which biases long sums (measured: 8.6e-5 normwise at K = 8192), so TMEM
// accumulates only a K chunk of TC_CHUNK values into A (columns 0..255);
// the epilogue warps fold each finished chunk into a running total T
// (columns 256..511) with round-to-nearest FADDs (tcgen05.ld / tcgen05.st),
// which bounds the bias by the chunk length.  Epilogue:
// c = c + alpha*(T + A) on the CUDA cores.
//
// Layout: column-major a (m,l) is M-contiguous; the prologue writes hi/lo of
// a transposed (K-major, row i has l contiguous values) and hi/lo of b as is
// (b(l,n) column-major is already K-major: column j has l contiguous).
//
// Kernel (one 128 x 256 tile of c per CTA, full K):
//   warp 0     TMA producer: 4 boxes per k-slab (a_hi, a_lo 128x32, b_hi,
//              b_lo 256x32, 128-byte swizzle) into a 2-stage ring, full/empty
//              mbarriers;
//   warp 1     MMA issuer: one elected thread issues 3 tcgen05.mma
//              (M=128, N=256, K=8) per 8-wide k step, tcgen05.commit frees the
//              stage; the accumulator (128 lanes x 256 fp32 columns) lives in
//              TMEM;
//   warps 2-5  epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes
//              32*(w%4)..), c = c + alpha*acc, coalesced column stores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "lfb_common.cuh"

namespace lfb {

constexpr int TC_BM = 128, TC_BN = 256, TC_BK = 32, TC_STAGES = 2;
constexpr int TC_THREADS = 192;
constexpr uint32_t TC_TMEM_COLS = 512;     // A: 0..255, T: 256..511
constexpr int TC_CHUNK = 8;                // k-slabs per TMEM chunk (K=256)

struct TcSmem {
  static constexpr size_t a_bytes = TC_BM * TC_BK * 4;   // 16 KB
  static constexpr size_t b_bytes = TC_BN * TC_BK * 4;   // 32 KB
  static constexpr size_t stage_bytes = 2 * a_bytes + 2 * b_bytes;  // 96 KB
  static constexpr size_t stages_off = 0;
  static constexpr size_t bars_off = TC_STAGES * stage_bytes;
  static constexpr size_t total = bars_off + 256 + 1024;  // + align slack
};

// {{{ PTX wrappers (tcgen05, TMA tensor)

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map,
                                            int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::"
      "bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 "
      "[%0];" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t adesc,
                                            uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// K-major, 128-byte swizzle smem descriptor (cute make_umma_desc<K> with
// Layout_K_SW128: rows of 128 B, 8-row atoms 1024 B apart -> SBO = 1024 B,
// LBO unused (1), version 1 for sm100, layout type 2 = SWIZZLE_128B)
__device__ __forceinline__ uint64_t sw128_kmajor_desc(const void *smem) {
  const uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;        // start address
  d |= (uint64_t)1 << 16;              // leading byte offset (unused)
  d |= (uint64_t)(1024 >> 4) << 32;    // stride byte offset
  d |= (uint64_t)1 << 46;              // version (sm100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, M=128, N=256
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N) {
  return (1u << 4)                     // c_format F32
         | (2u << 7)                   // a_format TF32
         | (2u << 10)                  // b_format TF32
         | ((uint32_t)(N >> 3) << 17)  // n_dim
         | ((uint32_t)(M >> 4) << 24); // m_dim
}

#define LFB_TMEM_ST16(taddr, r)                                              \
  asm volatile(                                                              \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "                        \
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"            \
      ::"r"(taddr), "r"((r)[0]), "r"((r)[1]), "r"((r)[2]), "r"((r)[3]), "r"((r)[4]),   \
      "r"((r)[5]), "r"((r)[6]), "r"((r)[7]), "r"((r)[8]), "r"((r)[9]), "r"((r)[10]),     \
      "r"((r)[11]), "r"((r)[12]), "r"((r)[13]), "r"((r)[14]), "r"((r)[15])             \
      : "memory")

#define LFB_TMEM_LD16(taddr, r)                                              \
  asm volatile(                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "                              \
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"      \
      : "=r"((r)[0]), "=r"((r)[1]), "=r"((r)[2]), "=r"((r)[3]), "=r"((r)[4]),          \
        "=r"((r)[5]), "=r"((r)[6]), "=r"((r)[7]), "=r"((r)[8]), "=r"((r)[9]),          \
        "=r"((r)[10]), "=r"((r)[11]), "=r"((r)[12]), "=r"((r)[13]), "=r"((r)[14]),     \
        "=r"((r)[15])                                                          \
      : "r"(taddr))

// }}}

__global__ void __launch_bounds__(TC_THREADS, 1)
    sgemm_tc_kernel(const __grid_constant__ CUtensorMap map_ahi,
                    const __grid_constant__ CUtensorMap map_alo,
                    const __grid_constant__ CUtensorMap map_bhi,
                    const __grid_constant__ CUtensorMap map_blo, float alpha,
                    float *__restrict__ c, int l, int m, int n) {
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment for the 128-byte swizzle atoms
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + TcSmem::bars_off);
  uint64_t *empty = full + TC_STAGES;
  uint64_t *chunk_done = empty + TC_STAGES;   // MMA -> epilogue
  uint64_t *chunk_free = chunk_done + 1;      // epilogue -> MMA
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(chunk_free + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int i0 = blockIdx.x * TC_BM, j0 = blockIdx.y * TC_BN;
  const int nk = l / TC_BK;
  const int nchunks = (nk + TC_CHUNK - 1) / TC_CHUNK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(chunk_done, 1);
    mbar_init(chunk_free, 4);  // one arrive per epilogue warp
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
        ::"r"(smem_u32(tmem_slot)), "r"(TC_TMEM_COLS)
        : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"
                 ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto stage_ptr = [&](int s) { return smem + s * TcSmem::stage_bytes; };

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % TC_STAGES;
        mbar_wait(&empty[s], ((kb / TC_STAGES) & 1) ^ 1);
        unsigned char *st = stage_ptr(s);
        mbar_arrive_expect_tx(&full[s], (uint32_t)TcSmem::stage_bytes);
        const int k0 = kb * TC_BK;
        tma_load_2d(st, &map_ahi, k0, i0, &full[s]);
        tma_load_2d(st + TcSmem::a_bytes, &map_alo, k0, i0, &full[s]);
        tma_load_2d(st + 2 * TcSmem::a_bytes, &map_bhi, k0, j0, &full[s]);
        tma_load_2d(st + 2 * TcSmem::a_bytes + TcSmem::b_bytes, &map_blo, k0,
                    j0, &full[s]);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tf32_idesc(TC_BM, TC_BN);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % TC_STAGES;
      const int ch = kb / TC_CHUNK;
      const bool first_in_chunk = (kb % TC_CHUNK) == 0;
      if (first_in_chunk && ch > 0) {
        // A must have been folded into T before it is overwritten
        mbar_wait(chunk_free, (ch - 1) & 1);
      }
      mbar_wait(&full[s], (kb / TC_STAGES) & 1);
      tc_fence_after();
      if (lane == 0) {
        unsigned char *st = stage_ptr(s);
        const uint64_t ahi = sw128_kmajor_desc(st);
        const uint64_t alo = sw128_kmajor_desc(st + TcSmem::a_bytes);
        const uint64_t bhi = sw128_kmajor_desc(st + 2 * TcSmem::a_bytes);
        const uint64_t blo =
            sw128_kmajor_desc(st + 2 * TcSmem::a_bytes + TcSmem::b_bytes);
#pragma unroll
        for (int k = 0; k < TC_BK / 8; ++k) {
          // K advance inside the 128-byte swizzled rows: +32 bytes per step
          const uint64_t dk = (uint64_t)((k * 32) >> 4);
          tc_mma_tf32(tmem, alo + dk, bhi + dk, idesc,
                      !(first_in_chunk && k == 0));
          tc_mma_tf32(tmem, ahi + dk, blo + dk, idesc, 1);
          tc_mma_tf32(tmem, ahi + dk, bhi + dk, idesc, 1);
        }
        tc_commit(&empty[s]);  // stage free once these MMAs completed
        if (kb % TC_CHUNK == TC_CHUNK - 1 || kb == nk - 1)
          tc_commit(chunk_done);
      }
      __syncwarp();
    }
  } else {
    // epilogue: warps 2..5 -> TMEM lane quarter (warp % 4)
    const int q = warp % 4;
    const uint32_t lanes = (uint32_t)(q * 32) << 16;
    // fold finished chunks: T = A (first) or T = T + A, round to nearest
    for (int ch = 0; ch < nchunks - 1; ++ch) {
      mbar_wait(chunk_done, ch & 1);
      tc_fence_after();
#pragma unroll 1
      for (int cb = 0; cb < TC_BN; cb += 16) {
        uint32_t ra[16], rt[16];
        LFB_TMEM_LD16(tmem + lanes + cb, ra);
        if (ch > 0) LFB_TMEM_LD16(tmem + lanes + TC_BN + cb, rt);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int t = 0; t < 16; ++t)
          rt[t] = ch > 0 ? __float_as_uint(fadd(__uint_as_float(rt[t]),
                                                __uint_as_float(ra[t])))
                         : ra[t];
        LFB_TMEM_ST16(tmem + lanes + TC_BN + cb, rt);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                         smem_u32(chunk_free))
                     : "memory");
    }
    mbar_wait(chunk_done, (nchunks - 1) & 1);
    tc_fence_after();
    const int i = i0 + q * 32 + lane;
    float *crow = c + i;
#pragma unroll 1
    for (int cb = 0; cb < TC_BN; cb += 16) {
      uint32_t ra[16], rt[16];
      LFB_TMEM_LD16(tmem + lanes + cb, ra);
      if (nchunks > 1) LFB_TMEM_LD16(tmem + lanes + TC_BN + cb, rt);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const float acc = nchunks > 1 ? fadd(__uint_as_float(rt[t]),
                                             __uint_as_float(ra[t]))
                                      : __uint_as_float(ra[t]);
        const int j = j0 + cb + t;
        float *p = crow + (int64_t)m * j;
        *p = fadd(*p, fmul(alpha, acc));
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(
                     tmem),
                 "r"(TC_TMEM_COLS)
                 : "memory");
  }
}

// {{{ persistent kernel: double-buffered TMEM accumulator, overlapped epilogue
//
// sgemm_tc_kernel above leaves the tensor pipe idle twice per tile: at every
// chunk boundary the MMA warp waits until the epilogue has folded A into T
// (A is about to be overwritten), and every tile ends with a serial C
// read-modify-write (ncu: tensor pipe 49 % active, profiles/r01_sgemm.md).
// Here
//  * TMEM holds two chunk accumulators, A0 (columns 0..255) and A1
//    (256..511): chunk g accumulates into A(g % 2) while the epilogue folds
//    chunk g - 1 out of the other, so the MMA warp never waits for a fold;
//  * the running total T lives in registers: 16 epilogue warps, warp w
//    reads TMEM lane quarter w % 4 and column quarter (w - 2) / 4, 64 fp32
//    of T per thread;
//  * CTAs are persistent (one per SM) over a grouped tile order, so the C
//    read-modify-write of tile t overlaps the MMAs of tile t + 1.
// Numerics are unchanged: T = A_0, T = T + A_1, ... (round-to-nearest FADD),
// c = c + alpha*T.
constexpr int TC2_EPI_WARPS = 16;
constexpr int TC2_THREADS = 32 * (2 + TC2_EPI_WARPS);  // producer, MMA, epi
constexpr int TC2_GROUP_M = 8;  // M tiles per raster group

// BK = 32: 128-byte swizzled K rows, 2 stages of 96 KB; BK = 16: 64-byte
// swizzled rows, 4 stages of 48 KB -- the same bytes in flight, but a stage
// is refilled after 6 instead of 12 MMAs, which gives the TMA loads three
// stages of slack instead of one.
template <int BK>
struct Tc2Cfg {
  static constexpr int STAGES = BK == 32 ? 2 : 4;
  static constexpr int CHUNK = 256 / BK;  // k-slabs per TMEM chunk (K = 256)
  static constexpr size_t a_bytes = (size_t)TC_BM * BK * 4;
  static constexpr size_t b_bytes = (size_t)TC_BN * BK * 4;
  static constexpr size_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  static constexpr size_t bars_off = STAGES * stage_bytes;
  static constexpr size_t total = bars_off + 256 + 1024;
  // K-major smem descriptor: rows of BK*4 bytes, 8-row swizzle atoms
  // (SBO = 8 rows), layout type 2 = SWIZZLE_128B, 4 = SWIZZLE_64B (sm100)
  __device__ static uint64_t desc(const void *smem) {
    const uint64_t addr = smem_u32(smem);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((8 * BK * 4) >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(BK == 32 ? 2 : 4) << 61;
    return d;
  }
};

__device__ __forceinline__ void tc2_tile(int t, int mt_count, int nt_count,
                                         int *mt, int *nt) {
  const int per_group = TC2_GROUP_M * nt_count;
  const int grp = t / per_group;
  const int r = t % per_group;
  const int m0 = grp * TC2_GROUP_M;
  const int gm = min(TC2_GROUP_M, mt_count - m0);
  *mt = m0 + r % gm;
  *nt = r / gm;
}

template <int BK>
__global__ void __launch_bounds__(TC2_THREADS, 1)
    sgemm_tc2_kernel(const __grid_constant__ CUtensorMap map_ahi,
                     const __grid_constant__ CUtensorMap map_alo,
                     const __grid_constant__ CUtensorMap map_bhi,
                     const __grid_constant__ CUtensorMap map_blo, float alpha,
                     float *__restrict__ c, int l, int m, int n) {
  using C = Tc2Cfg<BK>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::bars_off);
  uint64_t *empty = full + C::STAGES;
  uint64_t *acc_full = empty + C::STAGES;  // [2] MMA -> epilogue
  uint64_t *acc_empty = acc_full + 2;      // [2] epilogue -> MMA
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nk = l / BK;
  const int nchunks = (nk + C::CHUNK - 1) / C::CHUNK;
  const int mt_count = m / TC_BM, nt_count = n / TC_BN;
  const int ntiles = mt_count * nt_count;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], TC2_EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
        ::"r"(smem_u32(tmem_slot)), "r"(TC_TMEM_COLS)
        : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"
                 ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto stage_ptr = [&](int s) { return smem + s * C::stage_bytes; };

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;  // k-slab counter over all tiles of this CTA
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int mt, nt;
        tc2_tile(t, mt_count, nt_count, &mt, &nt);
        const int i0 = mt * TC_BM, j0 = nt * TC_BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait(&empty[s], ((it / C::STAGES) & 1) ^ 1);
          unsigned char *st = stage_ptr(s);
          mbar_arrive_expect_tx(&full[s], (uint32_t)C::stage_bytes);
          const int k0 = kb * BK;
          tma_load_2d(st, &map_ahi, k0, i0, &full[s]);
          tma_load_2d(st + C::a_bytes, &map_alo, k0, i0, &full[s]);
          tma_load_2d(st + 2 * C::a_bytes, &map_bhi, k0, j0, &full[s]);
          tma_load_2d(st + 2 * C::a_bytes + C::b_bytes, &map_blo,
                      k0, j0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tf32_idesc(TC_BM, TC_BN);
    int it = 0, g = 0;  // k-slab and chunk counters over all tiles
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % C::STAGES;
        const bool first_in_chunk = (kb % C::CHUNK) == 0;
        const bool last_in_chunk =
            kb % C::CHUNK == C::CHUNK - 1 || kb == nk - 1;
        const int b = g & 1;
        if (first_in_chunk)  // chunk g - 2 folded out of A(b)
          mbar_wait(&acc_empty[b], ((g >> 1) & 1) ^ 1);
        mbar_wait(&full[s], (it / C::STAGES) & 1);
        tc_fence_after();
        if (lane == 0) {
          unsigned char *st = stage_ptr(s);
          const uint64_t ahi = C::desc(st);
          const uint64_t alo = C::desc(st + C::a_bytes);
          const uint64_t bhi = C::desc(st + 2 * C::a_bytes);
          const uint64_t blo =
              C::desc(st + 2 * C::a_bytes + C::b_bytes);
          const uint32_t acc = tmem + (uint32_t)(b * TC_BN);
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const uint64_t dk = (uint64_t)((k * 32) >> 4);
            tc_mma_tf32(acc, alo + dk, bhi + dk, idesc,
                        !(first_in_chunk && k == 0));
            tc_mma_tf32(acc, ahi + dk, blo + dk, idesc, 1);
            tc_mma_tf32(acc, ahi + dk, bhi + dk, idesc, 1);
          }
          tc_commit(&empty[s]);
          if (last_in_chunk) tc_commit(&acc_full[b]);
        }
        __syncwarp();
        if (last_in_chunk) ++g;
      }
    }
  } else {
    const int q = warp % 4;
    const int cq = (warp - 2) / 4;  // column quarter
    const uint32_t lanes = (uint32_t)(q * 32) << 16;
    int g = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int mt, nt;
      tc2_tile(t, mt_count, nt_count, &mt, &nt);
      float T[64];
      for (int ch = 0; ch < nchunks; ++ch, ++g) {
        const int b = g & 1;
        mbar_wait(&acc_full[b], (g >> 1) & 1);
        tc_fence_after();
        const uint32_t base = tmem + lanes + (uint32_t)(b * TC_BN + cq * 64);
#pragma unroll
        for (int cb = 0; cb < 64; cb += 16) {
          uint32_t r[16];
          LFB_TMEM_LD16(base + cb, r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (ch == 0) {
#pragma unroll
            for (int x = 0; x < 16; ++x) T[cb + x] = __uint_as_float(r[x]);
          } else {
#pragma unroll
            for (int x = 0; x < 16; ++x)
              T[cb + x] = fadd(T[cb + x], __uint_as_float(r[x]));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                           smem_u32(&acc_empty[b]))
                       : "memory");
      }
      // c = c + alpha*T: lane = row, 32 consecutive rows per warp
      const int i = mt * TC_BM + q * 32 + lane;
      float *cp = c + i + (int64_t)m * (nt * TC_BN + cq * 64);
#pragma unroll
      for (int cb = 0; cb < 64; cb += 16) {
        float cv[16];
#pragma unroll
        for (int x = 0; x < 16; ++x) cv[x] = cp[(int64_t)m * (cb + x)];
#pragma unroll
        for (int x = 0; x < 16; ++x)
          cp[(int64_t)m * (cb + x)] = fadd(cv[x], fmul(alpha, T[cb + x]));
        asm volatile("" ::: "memory");
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(
                     tmem),
                 "r"(TC_TMEM_COLS)
                 : "memory");
  }
}

// }}}

// {{{ prologue: tf32 hi/lo split (a transposed to K-major)

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// a (m,l) column major -> hi/lo as [m][l] row major (K contiguous)
__global__ void split_transpose_a_kernel(const float *__restrict__ a,
                                         float *__restrict__ hi,
                                         float *__restrict__ lo, int m,
                                         int l) {
  __shared__ float tile[32][33];
  const int i0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y)
    tile[r][threadIdx.x] = a[(i0 + threadIdx.x) + (int64_t)m * (k0 + r)];
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const float x = tile[threadIdx.x][r];  // a(i0 + r, k0 + tx)
    const float h = rna_tf32(x);
    const int64_t o = (int64_t)(i0 + r) * l + k0 + threadIdx.x;
    hi[o] = h;
    lo[o] = x - h;
  }
}

__global__ void split_kernel(const float *__restrict__ b,
                             float *__restrict__ hi, float *__restrict__ lo,
                             int64_t count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count;
       q += stride) {
    const float x = b[q];
    const float h = rna_tf32(x);
    hi[q] = h;
    lo[q] = x - h;
  }
}

// }}}

static PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn() {
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

static bool make_kmajor_map(CUtensorMap *map, const float *base, int rows,
                            int kdim, int box_rows, int bk = TC_BK) {
  auto encode = tc_encode_fn();
  if (!encode) return false;
  cuuint64_t dims[2] = {(cuuint64_t)kdim, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kdim * 4};
  cuuint32_t box[2] = {(cuuint32_t)bk, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                const_cast<float *>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE,
                bk == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t sgemm_tc_workspace_floats(int l, int m, int n) {
  return 2 * ((int64_t)m * l + (int64_t)l * n);
}

bool sgemm_tc_shape_ok(int l, int m, int n) {
  return m % TC_BM == 0 && n % TC_BN == 0 && l % TC_BK == 0 && l > 0 &&
         m > 0 && n > 0;
}

// returns < 0 when the shape/workspace does not allow the tensor-core path
template <int BK>
static int launch_tc2(const float *ahi, const float *alo, const float *bhi,
                      const float *blo, float alpha, float *c, int l, int m,
                      int n, cudaStream_t s) {
  using C = Tc2Cfg<BK>;
  CUtensorMap mah, mal, mbh, mbl;
  if (!make_kmajor_map(&mah, ahi, m, l, TC_BM, BK) ||
      !make_kmajor_map(&mal, alo, m, l, TC_BM, BK) ||
      !make_kmajor_map(&mbh, bhi, n, l, TC_BN, BK) ||
      !make_kmajor_map(&mbl, blo, n, l, TC_BN, BK))
    return fail(LFB_ERR_LAUNCH, "sgemm: tensor map encode failed");
  cudaFuncSetAttribute(sgemm_tc2_kernel<BK>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)C::total);
  int sms = sm_count(nullptr);
  if (sms <= 0) sms = 148;
  const int tiles = (m / TC_BM) * (n / TC_BN);
  sgemm_tc2_kernel<BK><<<tiles < sms ? tiles : sms, TC2_THREADS, C::total,
                         s>>>(mah, mal, mbh, mbl, alpha, c, l, m, n);
  return check_launch("lfb_sgemm_f32(tcgen05 persistent)");
}

// variant: 0/2 persistent BK=16 (default), 3 the first non-persistent
// kernel, 4 persistent BK=32
int sgemm_tc(float alpha, const float *a, const float *b, float *c, int l,
             int m, int n, float *ws, int64_t ws_floats, cudaStream_t s,
             int variant) {
  if (!sgemm_tc_shape_ok(l, m, n) || !ws ||
      ws_floats < sgemm_tc_workspace_floats(l, m, n) || !aligned(ws, 16))
    return -1;
  float *ahi = ws, *alo = ahi + (int64_t)m * l;
  float *bhi = alo + (int64_t)m * l, *blo = bhi + (int64_t)l * n;
  split_transpose_a_kernel<<<dim3(m / 32, l / 32), dim3(32, 8), 0, s>>>(
      a, ahi, alo, m, l);
  const int64_t nb = (int64_t)l * n;
  split_kernel<<<sm_count(nullptr) * 8, 256, 0, s>>>(b, bhi, blo, nb);
  if (variant == 4)
    return launch_tc2<32>(ahi, alo, bhi, blo, alpha, c, l, m, n, s);
  if (variant != 3)
    return launch_tc2<16>(ahi, alo, bhi, blo, alpha, c, l, m, n, s);
  CUtensorMap mah, mal, mbh, mbl;
  if (!make_kmajor_map(&mah, ahi, m, l, TC_BM) ||
      !make_kmajor_map(&mal, alo, m, l, TC_BM) ||
      !make_kmajor_map(&mbh, bhi, n, l, TC_BN) ||
      !make_kmajor_map(&mbl, blo, n, l, TC_BN))
    return fail(LFB_ERR_LAUNCH, "sgemm: tensor map encode failed");
  cudaFuncSetAttribute(sgemm_tc_kernel,
                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)TcSmem::total);
  dim3 grid(m / TC_BM, n / TC_BN);
  sgemm_tc_kernel<<<grid, TC_THREADS, TcSmem::total, s>>>(
      mah, mal, mbh, mbl, alpha, c, l, m, n);
  return check_launch("lfb_sgemm_f32(tcgen05)");
}

}  // namespace lfb
