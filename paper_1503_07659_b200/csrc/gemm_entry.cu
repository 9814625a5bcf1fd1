// lfb_sgemm_f32: dispatch between the tensor-core path and the bit-exact
// CUDA-core path (geom->variant: 0 = default, 1 = exact, 2 = tensor only,
// 3 = the first, non-persistent tensor-core kernel, 4 = persistent BK=32).
// The tensor-core path needs m % 128 == 0, n % 256 == 0, l % 32 == 0 and a
// caller-provided workspace (lfb_sgemm_workspace doubles) for the tf32 hi/lo
// operand split; otherwise the default falls back to the exact kernel (a
// different kernel of the same sm_100a library, not a CPU path).
#include "lfb_common.cuh"

namespace lfb {
int sgemm_exact(float alpha, const float *a, const float *b, float *c, int l,
                int m, int n, cudaStream_t s);
int sgemm_tc(float alpha, const float *a, const float *b, float *c, int l,
             int m, int n, float *ws, int64_t ws_floats, cudaStream_t s,
             int variant);
int64_t sgemm_tc_workspace_floats(int l, int m, int n);
bool sgemm_tc_shape_ok(int l, int m, int n);
}  // namespace lfb

extern "C" {

int64_t lfb_sgemm_workspace(int l, int m, int n) {
  if (!lfb::sgemm_tc_shape_ok(l, m, n)) return 0;
  return (lfb::sgemm_tc_workspace_floats(l, m, n) + 1) / 2;
}

int lfb_sgemm_f32(float alpha, const float *a, const float *b, float *c,
                  int l, int m, int n, const lfb_launch *geom,
                  lfb_stream stream) {
  if (l < 0 || m < 0 || n < 0)
    return lfb::fail(LFB_ERR_ARG, "lfb_sgemm_f32: negative extent");
  if (m == 0 || n == 0) return LFB_OK;
  if (!a || !b || !c)
    return lfb::fail(LFB_ERR_ARG, "lfb_sgemm_f32: null array");
  if (geom && geom->abi_version != LFB_ABI_VERSION)
    return lfb::fail(LFB_ERR_ARG, "lfb_sgemm_f32: bad lfb_launch version");
  const int variant = geom ? geom->variant : 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (variant != 1) {
    float *ws = geom ? reinterpret_cast<float *>(geom->workspace) : nullptr;
    const int64_t wsf = geom ? 2 * geom->workspace_len : 0;
    int rc = lfb::sgemm_tc(alpha, a, b, c, l, m, n, ws, wsf, s, variant);
    if (rc >= 0) return rc;
    if (variant >= 2)
      return lfb::fail(LFB_ERR_UNSUPPORTED,
                       "lfb_sgemm_f32: tensor-core path needs m %% 128, "
                       "n %% 256, l %% 32 == 0 and a workspace of "
                       "lfb_sgemm_workspace() doubles (m=%d n=%d l=%d)",
                       m, n, l);
  }
  return lfb::sgemm_exact(alpha, a, b, c, l, m, n, s);
}

}  // extern "C"
