// Shared device helpers and internal launcher declarations for libdfc.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>
#include <vector>

#include "dfc.h"

namespace dfc {

// Validity threshold: the reference compares float32 maps against the
// Python float 0.1, which numpy-2 evaluates as float32(0.1) = 0x3DCCCCCD
// (depth_core.py:20,151).
constexpr float kValid = 0.1f;

__device__ __forceinline__ bool is_valid(float v) { return v > kValid; }
__device__ __forceinline__ int clampi(int i, int n) { return i < 0 ? 0 : (i >= n ? n - 1 : i); }
__device__ __forceinline__ float max3(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }
__device__ __forceinline__ float min3(float a, float b, float c) { return fminf(fminf(a, b), c); }

struct MaxOp {
  static __device__ __forceinline__ float identity() { return 0.0f; }  // all maps are >= 0
  static __device__ __forceinline__ float apply(float a, float b) { return fmaxf(a, b); }
};
struct MinOp {
  static __device__ __forceinline__ float identity() { return 3.402823466e38f; }
  static __device__ __forceinline__ float apply(float a, float b) { return fminf(a, b); }
};

// make_kernel + kernel_offsets (kernels.py:45-78): row-major (dy,dx) list of
// the Fig. 3 shape; *is_full when every cell of the size x size square is on
inline std::vector<int32_t> kernel_offsets(int shape, int size, bool* is_full) {
  std::vector<int32_t> o;
  const int r = size / 2;
  bool full = true;
  for (int dy = -r; dy <= r; ++dy)
    for (int dx = -r; dx <= r; ++dx) {
      bool on;
      switch (shape) {
        case DFC_SHAPE_FULL: on = true; break;
        case DFC_SHAPE_DIAMOND: on = std::abs(dx) + std::abs(dy) <= r; break;
        case DFC_SHAPE_CROSS: on = dx == 0 || dy == 0; break;
        default: on = 4 * (dx * dx + dy * dy) <= size * size; break;
      }
      if (on) {
        o.push_back(dy);
        o.push_back(dx);
      } else {
        full = false;
      }
    }
  *is_full = full;
  return o;
}

// process-wide count of kernels launched by libdfc (diagnostics for the bench)
extern std::atomic<unsigned long long> g_kernel_launches;
inline void note_launch(unsigned long long n = 1) { g_kernel_launches.fetch_add(n, std::memory_order_relaxed); }

// ---- internal launchers (ops_kernels.cu) ---------------------------------
cudaError_t launch_line_minmax(const float* in, float* out, int64_t B, int H, int W, int radius, bool is_min,
                               int axis, cudaStream_t s);
cudaError_t launch_offsets_minmax(const float* in, float* out, int64_t B, int H, int W, const int32_t* offs, int n,
                                  bool is_min, cudaStream_t s);
cudaError_t launch_median(const float* in, float* out, int64_t B, int H, int W, int size, cudaStream_t s);
cudaError_t launch_gauss_line(const float* in, void* out, int64_t B, int H, int W, const double* w, int k,
                              int axis, bool exact, bool in_is_f64, bool out_is_f64, cudaStream_t s);
cudaError_t launch_bilateral(const float* in, float* out, int64_t B, int H, int W, int size, double sv, double ss,
                             bool exact, cudaStream_t s);
cudaError_t launch_invert(const float* in, float* out, int64_t n_per_frame, int64_t B, float offset,
                          uint32_t* status, cudaStream_t s);
cudaError_t launch_validate(const float* in, int64_t n_per_frame, int64_t B, uint32_t* status, int64_t* n_valid,
                            cudaStream_t s);
cudaError_t launch_masked_fill(const float* cur, const float* dil, float* out, int64_t n, cudaStream_t s);
cudaError_t launch_extend_to_top(const float* in, float* out, int64_t B, int H, int W, cudaStream_t s);
cudaError_t launch_count_empty(const float* in, int64_t n_per_frame, int64_t B, int64_t* counts, cudaStream_t s);
cudaError_t launch_decode_raw16(const uint16_t* raw, float* out, int64_t n, cudaStream_t s);
cudaError_t launch_encode_raw16(const float* in, uint16_t* out, int64_t n_per_frame, int64_t n, uint32_t* status,
                                cudaStream_t s);
cudaError_t launch_error_sums(const float* pred, const float* gt, int64_t B, int64_t HW, double* sums,
                              int64_t* counts, cudaStream_t s);
cudaError_t launch_colormap(const float* values, uint8_t* rgb, int64_t n, double lo, double hi, cudaStream_t s);
cudaError_t launch_error_map(const float* pred, const float* gt, float* out, int64_t n, cudaStream_t s);
cudaError_t launch_reimpose(const float* blurred, const float* mask_src, float* out, int64_t n, cudaStream_t s);
cudaError_t launch_bin_select(const float* direct, const float* inv, float* out, int64_t n, float lo, float hi,
                              cudaStream_t s);
cudaError_t launch_max2(const float* a, const float* b, float* out, int64_t n, cudaStream_t s);
cudaError_t launch_iter_update(const int64_t* counts, int32_t* iters, int64_t B, unsigned long long* total,
                               cudaStream_t s);
cudaError_t launch_or_status(uint32_t* status, uint32_t bits, cudaStream_t s);
cudaError_t launch_finalize_status(const int64_t* n_valid, uint32_t* status, int64_t B, cudaStream_t s);
// large_fill.cu: device-gated multi-iteration large fill, frame gather / scatter
bool large_fill_tiled_supported(int r);
size_t large_fill_scratch_bytes(int64_t B);
cudaError_t launch_large_fill_loop(float* buf0, float* buf1, int64_t B, int H, int W, int r, int max_iters,
                                   int32_t* iters, void* scratch, cudaStream_t s);
cudaError_t launch_gather_frames(const float* src, float* dst, int64_t HW, const int64_t* idx, int64_t C, bool scatter,
                                 cudaStream_t s);
cudaError_t launch_scatter_status(const uint32_t* st, const int32_t* it, const unsigned* vc, const int64_t* idx,
                                  int64_t C, uint32_t* status, int32_t* iters, unsigned* vcount, uint32_t bits,
                                  cudaStream_t s);
cudaError_t launch_valid_counts(const float* out, int64_t HW, int64_t C, const int64_t* n_valid, unsigned* vcount,
                                cudaStream_t s);

// ---- blur stage + invert back in one tiled kernel (blur_tail.cu) ---------
bool blur_tail_supported(const dfc_config& c);
cudaError_t launch_blur_tail(const float* in, void* out, int64_t B, int H, int W, const dfc_config& c, bool out_raw,
                             uint32_t* status, unsigned* vcount, cudaStream_t s);

// ---- multiscale stage 1 + 2 (multiscale.cu) -------------------------------
bool multiscale_stage2_supported(const dfc_config& c);
cudaError_t launch_multiscale_stage2(const float* in, float* out, int64_t B, int H, int W, const dfc_config& c,
                                     const int32_t* const offs[3], const int n[3], unsigned* umax, unsigned* vcount,
                                     unsigned* work, cudaStream_t s);  // work: a zeroed device counter (item queue)

// ---- fused pipeline (fused.cu) -------------------------------------------
struct FusedPlan;
bool fused_supported(const dfc_config& c, int H, int W);
size_t fused_workspace_bytes(const dfc_config& c, int64_t B, int H, int W);
cudaError_t launch_fused(const void* in, void* out, int64_t B, int H, int W, const dfc_config& c,
                         uint32_t* status, int32_t* iters, unsigned* vcount, void* ws, size_t ws_bytes,
                         cudaStream_t s, int io = 0);
bool fused_supports_raw16(const dfc_config& c, int H, int W);

}  // namespace dfc
