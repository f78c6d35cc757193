// Depth-completion error metrics on the GPU.
//
// metrics._error_sums (metrics.py:119-137): over pixels where prediction and
// ground truth are both valid (> 0.1f), float64 sums of err^2, |err|,
// (1/d - 1/g)^2, |1/d - 1/g| with err = d - g, the count of such pixels, and
// the count of ground-truth-valid pixels the prediction leaves empty.
// error_map (metrics.py:101-108): |f64(d) - f64(g)| rounded to float32 where
// both are valid, 0 elsewhere.
//
// colormap: the visualisation of kitti_io.write_colormap_png.
//
// One CTA per frame, fixed reduction order (per-thread strided sums, warp
// butterfly, then the warps in order), so a frame's sums are reproducible run
// to run.  The reference's np.dot / np.sum order is unspecified (BLAS /
// pairwise); the float64 sums agree to ~1e-12 relative, the counts exactly.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dfc_common.cuh"

namespace dfc {
namespace {

constexpr int kMetThreads = 512;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kMetThreads) error_sums_kernel(const float* __restrict__ pred,
                                                                 const float* __restrict__ gt, int64_t HW,
                                                                 double* __restrict__ sums,
                                                                 int64_t* __restrict__ counts) {
  const int64_t b = blockIdx.x;
  const float* d = pred + b * HW;
  const float* g = gt + b * HW;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  long long n = 0, skipped = 0;
  for (int64_t i = threadIdx.x; i < HW; i += kMetThreads) {
    const float dv = __ldcs(d + i), gv = __ldcs(g + i);
    const bool gvld = gv > kValid, dvld = dv > kValid;
    skipped += gvld && !dvld;
    if (gvld && dvld) {
      const double dd = dv, gg = gv;
      const double e = dd - gg;
      const double ie = 1.0 / dd - 1.0 / gg;
      s[0] = fma(e, e, s[0]);
      s[1] += fabs(e);
      s[2] = fma(ie, ie, s[2]);
      s[3] += fabs(ie);
      ++n;
    }
  }
  __shared__ double ws[kMetThreads / 32][4];
  __shared__ long long wc[kMetThreads / 32][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 4; ++k) s[k] = warp_sum(s[k]);
  for (int o = 16; o > 0; o >>= 1) {
    n += __shfl_xor_sync(0xffffffffu, n, o);
    skipped += __shfl_xor_sync(0xffffffffu, skipped, o);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) ws[warp][k] = s[k];
    wc[warp][0] = n;
    wc[warp][1] = skipped;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t[4] = {0.0, 0.0, 0.0, 0.0};
    long long tn = 0, ts = 0;
    for (int w = 0; w < kMetThreads / 32; ++w) {
#pragma unroll
      for (int k = 0; k < 4; ++k) t[k] += ws[w][k];
      tn += wc[w][0];
      ts += wc[w][1];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) sums[b * 4 + k] = t[k];
    counts[b * 2] = tn;
    counts[b * 2 + 1] = ts;
  }
}

__global__ void error_map_kernel(const float* __restrict__ pred, const float* __restrict__ gt, float* __restrict__ out,
                                 int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float d = pred[i], g = gt[i];
    out[i] = (d > kValid && g > kValid) ? (float)fabs((double)d - (double)g) : 0.0f;
  }
}

// kitti_io.write_colormap_png's pixel arithmetic (kitti_io.py:69-85): t =
// clip((f64(v) - lo) / (hi - lo), 0, 1); per channel numpy.interp on the
// 5-stop ramp, i.e. slope_j * (t - x_j) + y_j for x_j <= t < x_{j+1} (y_4 at
// t == 1), each operation rounded separately; rint to uint8; black where
// v == 0.  float64 without contraction: bit-identical to numpy.
struct Ramp {
  double lo, span;
  double x[5];
  double y[3][5];
  double slope[3][4];
};

__global__ void colormap_kernel(const float* __restrict__ v, uint8_t* __restrict__ rgb, int64_t n,
                                const __grid_constant__ Ramp r) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float val = v[i];
    double t = __ddiv_rn(__dsub_rn((double)val, r.lo), r.span);
    t = fmin(fmax(t, 0.0), 1.0);
    const int j = t >= r.x[3] ? 3 : (t >= r.x[2] ? 2 : (t >= r.x[1] ? 1 : 0));
    uint8_t o[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double y = t >= r.x[4] ? r.y[c][4] : __dadd_rn(__dmul_rn(r.slope[c][j], __dsub_rn(t, r.x[j])), r.y[c][j]);
      o[c] = val == 0.0f ? (uint8_t)0 : (uint8_t)rint(y);
    }
    rgb[3 * i] = o[0];
    rgb[3 * i + 1] = o[1];
    rgb[3 * i + 2] = o[2];
  }
}

}  // namespace

cudaError_t launch_colormap(const float* values, uint8_t* rgb, int64_t n, double lo, double hi, cudaStream_t s) {
  Ramp r;
  r.lo = lo;
  r.span = hi - lo;
  const double x[5] = {0.0, 0.25, 0.5, 0.75, 1.0};
  const double y[3][5] = {{0.0, 0.0, 0.0, 255.0, 255.0}, {0.0, 255.0, 255.0, 255.0, 0.0},
                          {255.0, 255.0, 0.0, 0.0, 0.0}};  // kitti_io.py:27-31 ramp stops
  for (int k = 0; k < 5; ++k) r.x[k] = x[k];
  for (int c = 0; c < 3; ++c)
    for (int k = 0; k < 5; ++k) {
      r.y[c][k] = y[c][k];
      if (k < 4) r.slope[c][k] = (y[c][k + 1] - y[c][k]) / (x[k + 1] - x[k]);
    }
  const int64_t blocks = (n + 255) / 256;
  note_launch();
  colormap_kernel<<<(unsigned)(blocks < 148 * 32 ? blocks : 148 * 32), 256, 0, s>>>(values, rgb, n, r);
  return cudaGetLastError();
}

cudaError_t launch_error_sums(const float* pred, const float* gt, int64_t B, int64_t HW, double* sums,
                              int64_t* counts, cudaStream_t s) {
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
    note_launch();
    error_sums_kernel<<<(unsigned)nb, kMetThreads, 0, s>>>(pred + b0 * HW, gt + b0 * HW, HW, sums + b0 * 4,
                                                           counts + b0 * 2);
  }
  return cudaGetLastError();
}

cudaError_t launch_error_map(const float* pred, const float* gt, float* out, int64_t n, cudaStream_t s) {
  const int64_t blocks = (n + 255) / 256;
  note_launch();
  error_map_kernel<<<(unsigned)(blocks < 148 * 32 ? blocks : 148 * 32), 256, 0, s>>>(pred, gt, out, n);
  return cudaGetLastError();
}

}  // namespace dfc
