// Instantiations of the fused kernel with 16-bit KITTI raw at the boundary
// (kitti_io.py:36-66): IO 1 = raw in / float32 out, IO 2 = raw in / raw out.
// W % 4 == 0 (8-byte lane accesses), single-kernel stage 2 (no multiscale).
#include "fused_impl.cuh"

namespace dfc {

cudaError_t fused_dispatch_raw16(int io, bool full, int blur, const void* params, size_t smem, int grid,
                                 cudaStream_t s) {
  const Params& p = *static_cast<const Params*>(params);
  if (io == 1) {
    if (blur == DFC_BLUR_GAUSSIAN)
      return full ? launch_t<4, true, DFC_BLUR_GAUSSIAN, false, false, 1>(p, smem, grid, s)
                  : launch_t<4, false, DFC_BLUR_GAUSSIAN, false, false, 1>(p, smem, grid, s);
    if (blur == DFC_BLUR_NONE)
      return full ? launch_t<4, true, DFC_BLUR_NONE, false, false, 1>(p, smem, grid, s)
                  : launch_t<4, false, DFC_BLUR_NONE, false, false, 1>(p, smem, grid, s);
    return full ? launch_t<4, true, kBlurRaw, false, false, 1>(p, smem, grid, s)
                : launch_t<4, false, kBlurRaw, false, false, 1>(p, smem, grid, s);
  }
  // io 2 is never the raw blur mode: there the blur tail encodes
  if (blur == DFC_BLUR_GAUSSIAN)
    return full ? launch_t<4, true, DFC_BLUR_GAUSSIAN, false, false, 2>(p, smem, grid, s)
                : launch_t<4, false, DFC_BLUR_GAUSSIAN, false, false, 2>(p, smem, grid, s);
  return full ? launch_t<4, true, DFC_BLUR_NONE, false, false, 2>(p, smem, grid, s)
              : launch_t<4, false, DFC_BLUR_NONE, false, false, 2>(p, smem, grid, s);
}

}  // namespace dfc
