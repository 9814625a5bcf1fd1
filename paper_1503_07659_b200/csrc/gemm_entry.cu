// lfb_sgemm_f32: dispatch between the tensor-core path and the bit-exact
// CUDA-core path (geom->variant: 0 = default, 1 = exact, 2 = tensor).
#include "lfb_common.cuh"

namespace lfb {
int sgemm_exact(float alpha, const float *a, const float *b, float *c, int l,
                int m, int n, cudaStream_t s);
int sgemm_tc(float alpha, const float *a, const float *b, float *c, int l,
             int m, int n, cudaStream_t s);  // < 0: shape not supported
}  // namespace lfb

extern "C" int lfb_sgemm_f32(float alpha, const float *a, const float *b,
                             float *c, int l, int m, int n,
                             const lfb_launch *geom, lfb_stream stream) {
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
    int rc = lfb::sgemm_tc(alpha, a, b, c, l, m, n, s);
    if (rc >= 0) return rc;
    if (variant == 2)
      return lfb::fail(LFB_ERR_UNSUPPORTED,
                       "lfb_sgemm_f32: tensor-core path needs m, n multiples "
                       "of 128 and l of 32 (got m=%d n=%d l=%d)",
                       m, n, l);
  }
  return lfb::sgemm_exact(alpha, a, b, c, l, m, n, s);
}
