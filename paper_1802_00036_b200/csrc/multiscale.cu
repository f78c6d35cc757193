// Stage 1 + 2 of fill_in_multiscale in one tiled kernel: invert, depth-binned
// dilation (near / medium / far bins, each with its own kernel shape), max
// merge.  The composed oracle it follows is oracle/depthfill_oracle.py
// multiscale_dilate:
//   bin(p) = near   if d(p) <= edge_near     (empties carry 0 in every bin)
//            medium if edge_near < d(p) <= edge_far
//            far    if d(p) > edge_far
//   stage2 = max_k dilate_k(where(bin == k, invert(d), 0))
// with each dilation the reference's replicate-border offsets max
// (_native_ops.pyx:158-190): the CTA's input tile is loaded with
// frame-clamped coordinates, which is that border exactly.
//
// The kernel also records the largest input bit pattern per frame (the
// fused kernel's status check, fused.cu finalize_kernel), since the fused
// kernel that follows reads the stage-2 map, not the input.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "dfc_common.cuh"

namespace dfc {
namespace {

constexpr int kTX = 64, kTY = 16, kThreads = 256, kMaxR = 3;
constexpr int kMaxOffs = (2 * kMaxR + 1) * (2 * kMaxR + 1);

struct BinParams {
  float md, edge_near, edge_far;
  int n[3];                   // offsets per bin
  int8_t dy[3][kMaxOffs], dx[3][kMaxOffs];
};

template <int R>
__global__ void __launch_bounds__(kThreads) ms_stage2_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                             int H, int W, unsigned* __restrict__ umax,
                                                             const __grid_constant__ BinParams p) {
  constexpr int IW = kTX + 2 * R, IH = kTY + 2 * R;
  __shared__ float sb[3][IH * IW];
  __shared__ unsigned s_umax;
  const int64_t b = blockIdx.z;
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  const float* src = in + b * (int64_t)H * W;
  if (threadIdx.x == 0) s_umax = 0;
  unsigned um = 0;
  for (int i = threadIdx.x; i < IH * IW; i += kThreads) {
    const int iy = i / IW, ix = i - iy * IW;
    const int gy = y0 - R + iy, gx = x0 - R + ix;
    const float d = __ldg(src + (int64_t)clampi(gy, H) * W + clampi(gx, W));
    if (gy >= 0 && gy < H && gx >= 0 && gx < W) um = max(um, __float_as_uint(d));
    const float v = d > kValid ? p.md - d : 0.0f;  // depth_core.invert
    sb[0][i] = d <= p.edge_near ? v : 0.0f;
    sb[1][i] = (d > p.edge_near && d <= p.edge_far) ? v : 0.0f;
    sb[2][i] = d > p.edge_far ? v : 0.0f;
  }
  um = __reduce_max_sync(0xffffffffu, um);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicMax(&s_umax, um);
  float* dst = out + b * (int64_t)H * W;
  for (int i = threadIdx.x; i < kTX * kTY; i += kThreads) {
    const int oy = i / kTX, ox = i - oy * kTX;
    const int gy = y0 + oy, gx = x0 + ox;
    if (gy >= H || gx >= W) continue;
    const int c = (oy + R) * IW + ox + R;
    float m = 0.0f;  // all bin maps are >= 0
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float* t = sb[k] + c;
      for (int j = 0; j < p.n[k]; ++j) m = fmaxf(m, t[p.dy[k][j] * IW + p.dx[k][j]]);
    }
    __stcs(dst + (int64_t)gy * W + gx, m);
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(umax + b, s_umax);
}

}  // namespace

// kernel_offsets (capi.cu) for the three bins; false if a bin is wider than 7
bool multiscale_stage2_supported(const dfc_config& c) {
  return c.multiscale && c.near_size <= 2 * kMaxR + 1 && c.med_size <= 2 * kMaxR + 1 &&
         c.far_size <= 2 * kMaxR + 1;
}

cudaError_t launch_multiscale_stage2(const float* in, float* out, int64_t B, int H, int W, const dfc_config& c,
                                     const int32_t* const offs[3], const int n[3], unsigned* umax, cudaStream_t s) {
  BinParams p{};
  p.md = c.max_depth;
  p.edge_near = c.bin_edge_near;
  p.edge_far = c.bin_edge_far;
  int R = 0;
  for (int k = 0; k < 3; ++k) {
    if (n[k] > kMaxOffs) return cudaErrorInvalidValue;
    p.n[k] = n[k];
    for (int j = 0; j < n[k]; ++j) {
      p.dy[k][j] = (int8_t)offs[k][2 * j];
      p.dx[k][j] = (int8_t)offs[k][2 * j + 1];
      R = std::max(R, std::max(std::abs((int)p.dy[k][j]), std::abs((int)p.dx[k][j])));
    }
  }
  const dim3 grid((W + kTX - 1) / kTX, (H + kTY - 1) / kTY, (unsigned)B);
  note_launch();
  switch (R) {
    case 0:
    case 1: ms_stage2_kernel<1><<<grid, kThreads, 0, s>>>(in, out, H, W, umax, p); break;
    case 2: ms_stage2_kernel<2><<<grid, kThreads, 0, s>>>(in, out, H, W, umax, p); break;
    case 3: ms_stage2_kernel<3><<<grid, kThreads, 0, s>>>(in, out, H, W, umax, p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace dfc
