// Generic path: CUDA C++ generated from a kernel's
// schedule (paper_1503_07659_b200/cudagen.py) is compiled for sm_100a with
// NVRTC and launched through the driver API.
//
// The reference has no device target at all -- its OpenCL text is never
// compiled (lf/codegen.py:580-612) -- so this replaces that text
// emitter with a real one, for kernels the hand-written sm_100a kernels do not
// cover.  Neither NVRTC nor the driver library is a link-time dependency:
// libnvrtc is dlopen'ed on first compile, driver entry points come from
// cudaGetDriverEntryPoint, so the library still loads on a host without a GPU
// (the CPU tests compile generated code, they just cannot launch it).
#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "lfb_common.cuh"

namespace lfb {
namespace {

// {{{ NVRTC, resolved at run time

struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcGetErrorString) err = nullptr;
  bool ok = false;
  std::string why;
};

Nvrtc &nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *names[] = {"libnvrtc.so.12", "libnvrtc.so",
                           "/usr/local/cuda/lib64/libnvrtc.so.12"};
    void *h = nullptr;
    for (const char *nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) {
      n.why = std::string("cannot dlopen libnvrtc: ") + dlerror();
      return;
    }
#define LFB_SYM(field, sym)                                               \
  n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, #sym));          \
  if (!n.field) {                                                         \
    n.why = "libnvrtc lacks " #sym;                                       \
    return;                                                               \
  }
    LFB_SYM(create, nvrtcCreateProgram)
    LFB_SYM(compile, nvrtcCompileProgram)
    LFB_SYM(log_size, nvrtcGetProgramLogSize)
    LFB_SYM(log, nvrtcGetProgramLog)
    LFB_SYM(cubin_size, nvrtcGetCUBINSize)
    LFB_SYM(cubin, nvrtcGetCUBIN)
    LFB_SYM(destroy, nvrtcDestroyProgram)
    LFB_SYM(err, nvrtcGetErrorString)
#undef LFB_SYM
    n.ok = true;
  });
  return n;
}

// }}}

// {{{ driver API through the runtime's entry-point table

struct Driver {
  CUresult (*module_load)(CUmodule *, const void *) = nullptr;
  CUresult (*module_unload)(CUmodule) = nullptr;
  CUresult (*get_function)(CUfunction *, CUmodule, const char *) = nullptr;
  CUresult (*func_set_attr)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned,
                     unsigned, unsigned, unsigned, CUstream, void **,
                     void **) = nullptr;
  CUresult (*err_string)(CUresult, const char **) = nullptr;
  CUresult (*encode_tiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t,
                           void *, const cuuint64_t *, const cuuint64_t *,
                           const cuuint32_t *, const cuuint32_t *,
                           CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion,
                           CUtensorMapFloatOOBfill) = nullptr;
  bool ok = false;
  std::string why;
};

Driver &driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFree(nullptr);  // make the primary context current
#define LFB_DRV(field, sym)                                                \
  {                                                                        \
    void *fp = nullptr;                                                    \
    cudaDriverEntryPointQueryResult q;                                     \
    if (cudaGetDriverEntryPoint(#sym, &fp, cudaEnableDefault, &q) !=       \
            cudaSuccess ||                                                 \
        !fp) {                                                             \
      d.why = "driver entry point " #sym " unavailable";                   \
      return;                                                              \
    }                                                                      \
    d.field = reinterpret_cast<decltype(d.field)>(fp);                     \
  }
    LFB_DRV(module_load, cuModuleLoadData)
    LFB_DRV(module_unload, cuModuleUnload)
    LFB_DRV(get_function, cuModuleGetFunction)
    LFB_DRV(func_set_attr, cuFuncSetAttribute)
    LFB_DRV(launch, cuLaunchKernel)
    LFB_DRV(err_string, cuGetErrorString)
    LFB_DRV(encode_tiled, cuTensorMapEncodeTiled)
#undef LFB_DRV
    d.ok = true;
  });
  return d;
}

int drv_fail(const char *what, CUresult r) {
  const char *s = "unknown";
  if (driver().err_string) driver().err_string(r, &s);
  return fail(LFB_ERR_LAUNCH, "%s: %s", what, s);
}

// }}}

}  // namespace
}  // namespace lfb

struct lfb_module_st {
  CUmodule mod;
  CUfunction fn;
  int smem_set;
};

extern "C" {

int lfb_rtc_compile(const char *src, const char *prog_name,
                    const char *const *opts, int nopts, void *cubin,
                    int64_t *cubin_len) {
  using namespace lfb;
  if (!src || !cubin_len)
    return fail(LFB_ERR_ARG, "lfb_rtc_compile: null argument");
  Nvrtc &n = nvrtc();
  if (!n.ok) return fail(LFB_ERR_UNSUPPORTED, "%s", n.why.c_str());
  nvrtcProgram prog;
  nvrtcResult r = n.create(&prog, src, prog_name ? prog_name : "lfb_gen.cu",
                           0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS)
    return fail(LFB_ERR_UNSUPPORTED, "nvrtcCreateProgram: %s", n.err(r));
  r = n.compile(prog, nopts, opts);
  size_t log_len = 0;
  n.log_size(prog, &log_len);
  std::string log(log_len, '\0');
  if (log_len) n.log(prog, &log[0]);
  if (r != NVRTC_SUCCESS) {
    n.destroy(&prog);
    return fail(LFB_ERR_UNSUPPORTED, "NVRTC compile failed: %s\n%s",
                n.err(r), log.c_str());
  }
  size_t len = 0;
  n.cubin_size(prog, &len);
  if (cubin) {
    if ((int64_t)len > *cubin_len) {
      n.destroy(&prog);
      return fail(LFB_ERR_ARG, "lfb_rtc_compile: cubin buffer too small");
    }
    n.cubin(prog, static_cast<char *>(cubin));
  }
  *cubin_len = (int64_t)len;
  n.destroy(&prog);
  set_error(log);  // warnings, if any, stay readable via lfb_last_error
  return LFB_OK;
}

int lfb_module_load(const void *cubin, int64_t len, const char *kernel_name,
                    lfb_module *out) {
  using namespace lfb;
  (void)len;
  if (!cubin || !kernel_name || !out)
    return fail(LFB_ERR_ARG, "lfb_module_load: null argument");
  Driver &d = driver();
  if (!d.ok) return fail(LFB_ERR_LAUNCH, "%s", d.why.c_str());
  CUmodule mod;
  CUresult r = d.module_load(&mod, cubin);
  if (r != CUDA_SUCCESS) return drv_fail("cuModuleLoadData", r);
  CUfunction fn;
  r = d.get_function(&fn, mod, kernel_name);
  if (r != CUDA_SUCCESS) {
    d.module_unload(mod);
    return drv_fail("cuModuleGetFunction", r);
  }
  *out = new lfb_module_st{mod, fn, 0};
  return LFB_OK;
}

int lfb_module_launch(lfb_module m, const int64_t *grid, const int32_t *block,
                      int32_t smem, void **args, lfb_stream stream) {
  using namespace lfb;
  if (!m || !grid || !block)
    return fail(LFB_ERR_ARG, "lfb_module_launch: null argument");
  for (int a = 0; a < 3; ++a)
    if (grid[a] < 0 || grid[a] > (a ? 65535 : 2147483647) || block[a] < 1)
      return fail(LFB_ERR_UNSUPPORTED,
                  "lfb_module_launch: grid (%lld,%lld,%lld) block (%d,%d,%d) "
                  "outside CUDA limits",
                  (long long)grid[0], (long long)grid[1], (long long)grid[2],
                  block[0], block[1], block[2]);
  if ((int64_t)block[0] * block[1] * block[2] > 1024)
    return fail(LFB_ERR_UNSUPPORTED,
                "lfb_module_launch: %d threads per block (work-group size "
                "from the l.N tags) exceeds 1024",
                block[0] * block[1] * block[2]);
  if (grid[0] == 0 || grid[1] == 0 || grid[2] == 0) return LFB_OK;  // empty
  Driver &d = driver();
  if (smem > 48 * 1024 && m->smem_set < smem) {
    CUresult r = d.func_set_attr(
        m->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem);
    if (r != CUDA_SUCCESS) return drv_fail("cuFuncSetAttribute", r);
    m->smem_set = smem;
  }
  CUresult r = d.launch(m->fn, (unsigned)grid[0], (unsigned)grid[1],
                        (unsigned)grid[2], (unsigned)block[0],
                        (unsigned)block[1], (unsigned)block[2],
                        (unsigned)smem, (CUstream)stream, args, nullptr);
  if (r != CUDA_SUCCESS) return drv_fail("cuLaunchKernel", r);
  return LFB_OK;
}

int lfb_tmap_encode(void *map, int dtype, int rank, const int64_t *dims,
                    const int64_t *strides_bytes, const int32_t *box,
                    int swizzle_bytes, const void *base) {
  using namespace lfb;
  if (!map || !dims || !box || !base || (rank > 1 && !strides_bytes))
    return fail(LFB_ERR_ARG, "lfb_tmap_encode: null argument");
  if (rank < 1 || rank > 5)
    return fail(LFB_ERR_UNSUPPORTED, "lfb_tmap_encode: rank %d", rank);
  static const CUtensorMapDataType types[] = {
      CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
      CU_TENSOR_MAP_DATA_TYPE_INT32};
  static const int esize[] = {8, 4, 4};
  if (dtype < 0 || dtype > 2)
    return fail(LFB_ERR_ARG, "lfb_tmap_encode: dtype %d", dtype);
  // the tensor-map rules, checked here so an unsuitable footprint is an
  // UNSUPPORTED status (the caller then runs the kernel's cooperative fetch)
  if (reinterpret_cast<uintptr_t>(base) % 16)
    return fail(LFB_ERR_UNSUPPORTED, "tensor map: base not 16-B aligned");
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t bdim[5], estride[5];
  for (int d = 0; d < rank; ++d) {
    if (dims[d] < 1 || dims[d] >= (int64_t(1) << 31) || box[d] < 1 ||
        box[d] > 256)
      return fail(LFB_ERR_UNSUPPORTED, "tensor map: dim %d extent %lld box %d",
                  d, (long long)dims[d], box[d]);
    gdim[d] = (cuuint64_t)dims[d];
    bdim[d] = (cuuint32_t)box[d];
    estride[d] = 1;
    if (d > 0) {
      int64_t st = strides_bytes[d - 1];
      if (st <= 0 || st % 16 || st >= (int64_t(1) << 40))
        return fail(LFB_ERR_UNSUPPORTED,
                    "tensor map: stride %lld B of dim %d not a positive "
                    "multiple of 16", (long long)st, d);
      gstride[d - 1] = (cuuint64_t)st;
    }
  }
  if ((box[0] * esize[dtype]) % 16)
    return fail(LFB_ERR_UNSUPPORTED, "tensor map: inner box %d B",
                box[0] * esize[dtype]);
  CUtensorMapSwizzle sw;
  switch (swizzle_bytes) {
    case 0: sw = CU_TENSOR_MAP_SWIZZLE_NONE; break;
    case 32: sw = CU_TENSOR_MAP_SWIZZLE_32B; break;
    case 64: sw = CU_TENSOR_MAP_SWIZZLE_64B; break;
    case 128: sw = CU_TENSOR_MAP_SWIZZLE_128B; break;
    default:
      return fail(LFB_ERR_ARG, "lfb_tmap_encode: swizzle %d", swizzle_bytes);
  }
  Driver &d = driver();
  if (!d.ok) return fail(LFB_ERR_LAUNCH, "%s", d.why.c_str());
  alignas(64) CUtensorMap tm;
  CUresult r = d.encode_tiled(&tm, types[dtype], (cuuint32_t)rank,
                              const_cast<void *>(base), gdim, gstride, bdim,
                              estride, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    const char *str = "unknown";
    if (d.err_string) d.err_string(r, &str);
    return fail(LFB_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled: %s", str);
  }
  memcpy(map, &tm, sizeof(tm));
  return LFB_OK;
}

int lfb_module_unload(lfb_module m) {
  using namespace lfb;
  if (!m) return LFB_OK;
  CUresult r = driver().module_unload(m->mod);
  delete m;
  if (r != CUDA_SUCCESS) return drv_fail("cuModuleUnload", r);
  return LFB_OK;
}

}  // extern "C"
