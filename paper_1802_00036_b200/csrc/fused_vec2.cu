// Instantiations of the fused kernel for 2-column vector access (see fused_impl.cuh).
#include "fused_impl.cuh"

namespace dfc {

cudaError_t fused_dispatch_vec2(bool full, int blur, bool pre, bool dense, const void* params, size_t smem, int grid,
                                 cudaStream_t s) {
  const Params& p = *static_cast<const Params*>(params);
  (void)dense;
  return full ? dispatch_blur<2, true>(blur, pre, p, smem, grid, s) : dispatch_blur<2, false>(blur, pre, p, smem, grid, s);
}

}  // namespace dfc
