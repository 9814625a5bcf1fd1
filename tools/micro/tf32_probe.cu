// tcgen05 kind::tf32 issue-rate probe: the MMA shape of the sgemm kernel
// (cta_group::1, M = 128, N = 256, K = 8, K-major SWIZZLE_128B operands,
// f32 accumulator in TMEM) issued back to back from smem-resident tiles by
// one thread per SM, no loads and no epilogue.  The TFLOP/s it reaches is
// the tensor-pipe ceiling the 3xTF32 sgemm (csrc/gemm_sm100.cu) runs
// against: 3 MMAs per fp32 product, so the fp32-equivalent ceiling is a
// third of the printed TF32 figure.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tf32_probe tf32_probe.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// K-major operand descriptor: sw128 = 128-byte rows (BK = 32 tf32), else
// 64-byte rows with the 64-byte swizzle (BK = 16, the sgemm default)
__device__ __forceinline__ uint64_t desc(const void *smem, bool sw128) {
  const uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sw128 ? 1024 : 512) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(sw128 ? 2 : 4) << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1) probe(int iters, int sw128, float *sink,
                                               long long *cyc) {
  const long long c0 = clock64();
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char *a = smem;                 // 128 x 32 tf32 = 16 KB
  unsigned char *b = smem + 16384;         // 256 x 32 tf32 = 32 KB
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 49152);
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x)
    reinterpret_cast<float *>(smem)[i] = 0.0f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;"
        ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const uint64_t ad = desc(a, sw128), bd = desc(b, sw128);
    constexpr uint32_t id = idesc(128, 256);
    const int steps = sw128 ? 4 : 2;   // K = 8 steps per row
    for (int it = 0; it < iters * (4 / steps); ++it) {
#pragma unroll 2
      for (int dk = 0; dk < steps; ++dk) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
            ::"r"(tmem), "l"(ad + 2 * dk), "l"(bd + 2 * dk), "r"(id),
            "r"((uint32_t)(it | dk))
            : "memory");
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster."
        "b64 [%0];" ::"r"(smem_u32(bar))
        : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\n"
                   "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                   "selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(smem_u32(bar)) : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                 : "=r"(v) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (threadIdx.x == 0) {
      sink[blockIdx.x] = __uint_as_float(v);
      cyc[blockIdx.x] = clock64() - c0;
    }
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;"
                 ::"r"(tmem));
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *sink;
  cudaMalloc(&sink, sms * sizeof(float));
  long long *cyc;
  cudaMalloc(&cyc, sms * sizeof(long long));
  long long hc[1024];
  const int smem = 49152 + 1024 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int sw : {1, 0})
  for (int iters : {1000, 20000, 20000}) {
    cudaEventRecord(e0);
    probe<<<sms, 128, smem>>>(iters, sw, sink, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 128 * 256 * 8 * 4.0 * iters * sms;
    const cudaError_t err = cudaGetLastError();
    cudaMemcpy(hc, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    const double mhz = (double)hc[0] / (ms * 1e3);
    printf("%s iters %d: %.3f ms  %.1f TFLOP/s tf32  (%.1f fp32-equivalent "
           "for 3xTF32)  SM clock %.0f MHz  %s\n", sw ? "SW128" : "SW64 ",
           iters, ms, flops / ms / 1e9, flops / ms / 1e9 / 3, mhz,
           cudaGetErrorString(err));
  }
  return 0;
}
