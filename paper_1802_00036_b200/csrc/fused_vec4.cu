// Instantiations of the fused kernel for 4-column vector access (see fused_impl.cuh).
#include "fused_impl.cuh"

namespace dfc {

cudaError_t fused_dispatch_vec4(bool full, int blur, bool pre, bool dense, const void* params, size_t smem, int grid,
                                 cudaStream_t s) {
  const Params& p = *static_cast<const Params*>(params);
  if (dense && full) {
    if (blur == DFC_BLUR_GAUSSIAN) return dispatch_dense<DFC_BLUR_GAUSSIAN>(pre, p, smem, grid, s);
    if (blur == DFC_BLUR_NONE) return dispatch_dense<DFC_BLUR_NONE>(pre, p, smem, grid, s);
    return dispatch_dense<kBlurRaw>(pre, p, smem, grid, s);
  }
  (void)dense;
  if (full && p.regdense) {
    if (blur == DFC_BLUR_GAUSSIAN) return dispatch_regdense<DFC_BLUR_GAUSSIAN>(pre, p, smem, grid, s);
    if (blur == DFC_BLUR_NONE) return dispatch_regdense<DFC_BLUR_NONE>(pre, p, smem, grid, s);
    return dispatch_regdense<kBlurRaw>(pre, p, smem, grid, s);
  }
  return full ? dispatch_blur<4, true>(blur, pre, p, smem, grid, s) : dispatch_blur<4, false>(blur, pre, p, smem, grid, s);
}

}  // namespace dfc
