// Fused streaming pipeline kernel -- placeholder until the sm_100a kernel lands.
#include "dfc_common.cuh"

namespace dfc {
bool fused_supported(const dfc_config&, int, int) { return false; }
size_t fused_workspace_bytes(const dfc_config&, int64_t, int, int) { return 0; }
cudaError_t launch_fused(const float*, float*, int64_t, int, int, const dfc_config&, uint32_t*, int32_t*, void*,
                         size_t, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace dfc
