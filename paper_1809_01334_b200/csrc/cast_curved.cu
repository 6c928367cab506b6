// cast_curved.cu -- segment kernel for curved (R=2) trees.  (placeholder)
#include "kernels.cuh"

namespace rc {
cudaError_t launch_cast_curved(const CamConst&, const TreeConst*, DevLeafView, int, const int32_t*, const Rect16*,
                               const int64_t*, const int32_t*, int64_t, uint32_t, rc_seg*, int64_t, int32_t*,
                               int64_t*, int, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace rc
