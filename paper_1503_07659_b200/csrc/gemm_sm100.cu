// sgemm on the 5th-generation tensor cores (placeholder until the tcgen05
// kernel lands: reports "shape not supported" so the dispatcher uses the
// bit-exact CUDA-core kernel).
#include "lfb_common.cuh"

namespace lfb {

int sgemm_tc(float, const float *, const float *, float *, int, int, int,
             cudaStream_t) {
  return -1;
}

}  // namespace lfb
