// K6 / K7 / K8: QAT attention backward (placeholder until the tcgen05 kernel lands).
#include <cuda_runtime.h>
#include "attn.h"
namespace aq {
cudaError_t launch_attn_bwd(const BwdParams&, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_bwd_pre(const void*, int, const void*, int, int64_t, int64_t, int, float*, uint8_t*, float*,
                           cudaStream_t) {
  return cudaErrorNotSupported;
}
cudaError_t launch_dq_convert(const float*, void*, int, int64_t, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace aq
