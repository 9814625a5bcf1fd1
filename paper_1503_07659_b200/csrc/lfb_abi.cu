// ABI core: version, thread-local error text, device queries, FP64 probe.
#include <stdarg.h>

#include "lfb_common.cuh"

namespace lfb {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_launch(const char *what) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return fail(LFB_ERR_LAUNCH, "%s: CUDA launch failed: %s", what,
                cudaGetErrorString(err));
  return LFB_OK;
}

int sm_count(const lfb_launch *geom) {
  if (geom && geom->sm_count > 0) return geom->sm_count;
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) !=
      cudaSuccess)
    return -1;
  return n;
}

// 8 independent chains of separately rounded multiply + add per thread: the
// instruction mix of the SEM contractions, used to measure the FP64 issue
// ceiling on the box the bench runs on.
__global__ void probe_fp64_kernel(double *out, int iters) {
  double a[8], m = 1.0000001 + threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = c * 0.5 + blockIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = dadd(dmul(a[c], m), 1e-3);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += a[c];
  if (s == 123.456) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// The SEM kernel's HBM traffic without its arithmetic: per point read u (8 B)
// and the 6 g values (48 B), write w (8 B) -- the ceiling of that access mix
// at a given footprint (bench.py reports it beside the roofline).
__global__ void probe_stream_kernel(double *__restrict__ w,
                                    const double *__restrict__ u,
                                    const double *__restrict__ g,
                                    int64_t npoints) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
       2 * p + 1 < npoints; p += stride) {
    const double2 uv = __ldcs(reinterpret_cast<const double2 *>(u) + p);
    const double2 *gp = reinterpret_cast<const double2 *>(g) + 6 * p;
    double2 a = __ldcs(gp), b = __ldcs(gp + 1), c = __ldcs(gp + 2);
    double2 d = __ldcs(gp + 3), e = __ldcs(gp + 4), f = __ldcs(gp + 5);
    double2 r;
    r.x = uv.x + a.x + b.y + d.x;
    r.y = uv.y + c.x + e.y + f.x;
    __stcs(reinterpret_cast<double2 *>(w) + p, r);
  }
}

}  // namespace lfb

extern "C" {

int lfb_probe_stream(double *w, const double *u, const double *g,
                     int64_t npoints, lfb_stream stream) {
  if (!w || !u || !g || npoints < 2)
    return lfb::fail(LFB_ERR_ARG, "lfb_probe_stream: bad arguments");
  int sms = lfb::sm_count(nullptr);
  lfb::probe_stream_kernel<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(
      w, u, g, npoints);
  return lfb::check_launch("lfb_probe_stream");
}

int lfb_abi_version(void) { return LFB_ABI_VERSION; }

const char *lfb_last_error(void) { return lfb::g_last_error.c_str(); }

int lfb_device_sm_count(void) { return lfb::sm_count(nullptr); }

int lfb_probe_fp64(double *out, int iters, int blocks, int threads,
                   lfb_stream stream) {
  if (!out || iters <= 0 || blocks <= 0 || threads <= 0 || threads > 1024)
    return lfb::fail(LFB_ERR_ARG, "lfb_probe_fp64: bad arguments");
  lfb::probe_fp64_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(out,
                                                                      iters);
  return lfb::check_launch("lfb_probe_fp64");
}

}  // extern "C"
