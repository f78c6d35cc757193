// Multi-iteration large hole fill without a host round trip per iteration
// (pipeline.py:176-187: while iters < large_fill_max_iters and any pixel is
// empty: cur = masked_fill_dilate(cur, FULL large_fill_size); iters += 1).
//
// One tiled kernel per iteration does the whole masked 31x31 (any radius
// <= kLFMaxR) fill of one frame tile: the tile plus its halo is staged in
// shared memory with clamped coordinates (max over a clamped window == the
// reference's replicate border), tiles without an empty pixel are copied,
// the others take vertical then horizontal window maxima, and the empties
// left in the output are counted per frame.  The kernel is gated per frame
// on the device: a frame whose count reached zero (or that never had an
// empty pixel) returns at once, so the host launches iterations in groups
// and synchronises once per group instead of once per iteration, and frames
// of one batch iterate independently (each keeps its own iteration count).
//
// Ping-pong: active frames of iteration k read buf[k & 1] and write
// buf[(k + 1) & 1] (a frame is active for a prefix of the iterations, so every
// active frame has done exactly k of them); after the loop, frames with an odd
// iteration count are copied back to buf[0].
//
// Per-frame counts rotate over three arrays: iteration k reads cnt[k % 3],
// adds to cnt[(k + 1) % 3] and zeroes cnt[(k + 2) % 3] (read at k - 1, written
// at k + 1); the batch totals the host polls rotate the same way.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dfc_common.cuh"

namespace dfc {
namespace {

constexpr int kLFTX = 64, kLFTY = 16, kLFThreads = 256, kLFMaxR = 32;

__global__ void lf_count_kernel(const float* __restrict__ in, int64_t HW, int64_t* cnt0, unsigned long long* tot0) {
  const int64_t b = blockIdx.y;
  const float* src = in + b * HW;
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW; i += (int64_t)gridDim.x * blockDim.x)
    c += !(src[i] > kValid);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) {
    atomicAdd((unsigned long long*)(cnt0 + b), c);
    atomicAdd(tot0, c);
  }
}

// grid: (tiles per frame, frames); dynamic smem (TY + 2r) x (TX + 2r) input + TY x (TX + 2r) vertical maxima
__global__ void __launch_bounds__(kLFThreads) lf_iter_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                                             int H, int W, int r, int tiles_x, int k,
                                                             const int64_t* __restrict__ cnt_in, int64_t* cnt_out,
                                                             int64_t* cnt_zero, unsigned long long* tot_out,
                                                             unsigned long long* tot_zero, int32_t* iters) {
  extern __shared__ float sm[];
  const int64_t b = blockIdx.y;
  const int t = blockIdx.x;
  if (threadIdx.x == 0) {
    if (t == 0) cnt_zero[b] = 0;
    if (t == 0 && b == 0) *tot_zero = 0;
  }
  if (cnt_in[b] == 0) return;  // frame done (uniform over the CTA)
  if (t == 0 && threadIdx.x == 0) iters[b] = k + 1;
  const int x0 = (t % tiles_x) * kLFTX, y0 = (t / tiles_x) * kLFTY;
  const int IW = kLFTX + 2 * r, IH = kLFTY + 2 * r;
  float* sIn = sm;
  float* sV = sm + IH * IW;
  const int64_t HW = (int64_t)H * W;
  const float* f = src + b * HW;
  float* o = dst + b * HW;
  for (int i = threadIdx.x; i < IH * IW; i += kLFThreads) {
    const int iy = i / IW, ix = i - iy * IW;
    sIn[i] = __ldg(f + (int64_t)clampi(y0 - r + iy, H) * W + clampi(x0 - r + ix, W));
  }
  __syncthreads();
  bool empty = false;
  for (int i = threadIdx.x; i < kLFTX * kLFTY; i += kLFThreads) {
    const int y = i / kLFTX, x = i - y * kLFTX;
    if (y0 + y < H && x0 + x < W) empty |= !(sIn[(y + r) * IW + x + r] > kValid);
  }
  if (!__syncthreads_or(empty)) {  // nothing to fill: copy the tile
    for (int i = threadIdx.x; i < kLFTX * kLFTY; i += kLFThreads) {
      const int y = i / kLFTX, x = i - y * kLFTX;
      if (y0 + y < H && x0 + x < W) o[(int64_t)(y0 + y) * W + x0 + x] = sIn[(y + r) * IW + x + r];
    }
    return;
  }
  // vertical maxima over rows [y, y + 2r] of every staged column
  for (int i = threadIdx.x; i < kLFTY * IW; i += kLFThreads) {
    const int y = i / IW, x = i - y * IW;
    const float* c = sIn + y * IW + x;
    float m = c[0];
    for (int d = 1; d <= 2 * r; ++d) m = fmaxf(m, c[d * IW]);
    sV[i] = m;
  }
  __syncthreads();
  unsigned long long left = 0;
  for (int i = threadIdx.x; i < kLFTX * kLFTY; i += kLFThreads) {
    const int y = i / kLFTX, x = i - y * kLFTX;
    if (y0 + y >= H || x0 + x >= W) continue;
    float v = sIn[(y + r) * IW + x + r];
    if (!(v > kValid)) {
      const float* c = sV + y * IW + x;
      float m = c[0];
      for (int d = 1; d <= 2 * r; ++d) m = fmaxf(m, c[d]);
      v = m;
      left += !(v > kValid);
    }
    o[(int64_t)(y0 + y) * W + x0 + x] = v;
  }
  for (int s = 16; s > 0; s >>= 1) left += __shfl_xor_sync(0xffffffffu, left, s);
  if ((threadIdx.x & 31) == 0 && left) {
    atomicAdd((unsigned long long*)(cnt_out + b), left);
    atomicAdd(tot_out, left);
  }
}

// frames whose iteration count is odd hold their result in buf1: copy it to buf0
__global__ void lf_settle_kernel(float* __restrict__ buf0, const float* __restrict__ buf1, int64_t HW,
                                 const int32_t* __restrict__ n) {
  const int64_t b = blockIdx.y;
  if (!(n[b] & 1)) return;
  const float* s = buf1 + b * HW;
  float* d = buf0 + b * HW;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

__global__ void gather_frames_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t HW,
                                     const int64_t* __restrict__ idx, bool scatter) {
  const int64_t b = blockIdx.y, f = idx[b];
  const float4* s = reinterpret_cast<const float4*>(src + (scatter ? b : f) * HW);
  float4* d = reinterpret_cast<float4*>(dst + (scatter ? f : b) * HW);
  const float* s1 = src + (scatter ? b : f) * HW;
  float* d1 = dst + (scatter ? f : b) * HW;
  const bool vec = HW % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  if (vec) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW / 4; i += (int64_t)gridDim.x * blockDim.x)
      d[i] = s[i];
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW; i += (int64_t)gridDim.x * blockDim.x)
      d1[i] = s1[i];
  }
}

__global__ void scatter_status_kernel(const uint32_t* __restrict__ st, const int32_t* __restrict__ it,
                                      const unsigned* __restrict__ vc, const int64_t* __restrict__ idx, int64_t C,
                                      uint32_t* status, int32_t* iters, unsigned* vcount, uint32_t bits) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= C) return;
  const int64_t f = idx[b];
  status[f] = st[b] | bits;
  if (iters) iters[f] = it[b];
  if (vcount) vcount[2 * f] = vc[2 * b], vcount[2 * f + 1] = vc[2 * b + 1];
}

// [b][0] = n_valid[b] (inputs > 0.1, from the validate pass), [b][1] = outputs > 0.1
__global__ void valid_counts_kernel(const float* __restrict__ out, int64_t HW, const int64_t* __restrict__ n_valid,
                                    unsigned* vcount) {
  const int64_t b = blockIdx.y;
  const float* src = out + b * HW;
  unsigned c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW; i += (int64_t)gridDim.x * blockDim.x)
    c += src[i] > kValid;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(vcount + 2 * b + 1, c);
  if (blockIdx.x == 0 && threadIdx.x == 0) vcount[2 * b] = (unsigned)n_valid[b];
}

unsigned frames_grid_x(int64_t HW) {
  const int64_t g = (HW + 1023) / 1024;
  return (unsigned)(g < 1 ? 1 : (g > 64 ? 64 : g));
}

}  // namespace

bool large_fill_tiled_supported(int r) { return r >= 1 && r <= kLFMaxR; }

size_t large_fill_scratch_bytes(int64_t B) { return (size_t)(3 * B + 3) * 8 + (size_t)B * 4; }

// Runs the large-fill loop on B frames in buf0 (result in buf0; buf1 is
// scratch).  iters[b] (may be null) receives the frame's iteration count.
// scratch: large_fill_scratch_bytes(B).  Batches of more than 65535 frames
// are chunked by the caller (run_staged chunks by memory).
cudaError_t launch_large_fill_loop(float* buf0, float* buf1, int64_t B, int H, int W, int r, int max_iters,
                                   int32_t* iters, void* scratch, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  if (B > 65535 || !large_fill_tiled_supported(r)) return cudaErrorInvalidValue;
  const int64_t HW = (int64_t)H * W;
  int64_t* cnt = static_cast<int64_t*>(scratch);  // [3][B]
  unsigned long long* tot = reinterpret_cast<unsigned long long*>(cnt + 3 * B);  // [3]
  int32_t* nit = reinterpret_cast<int32_t*>(tot + 3);                             // [B]
  cudaError_t e = cudaMemsetAsync(scratch, 0, large_fill_scratch_bytes(B), s);
  if (e != cudaSuccess) return e;
  note_launch();
  lf_count_kernel<<<dim3(frames_grid_x(HW), (unsigned)B), 256, 0, s>>>(buf0, HW, cnt, tot);
  const int tiles_x = (W + kLFTX - 1) / kLFTX, tiles_y = (H + kLFTY - 1) / kLFTY;
  const size_t smem = (size_t)((kLFTY + 2 * r) * (kLFTX + 2 * r) + kLFTY * (kLFTX + 2 * r)) * 4;
  if ((e = cudaFuncSetAttribute(lf_iter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  float* buf[2] = {buf0, buf1};
  int k = 0;
  // first group of 2 (generated frames need one iteration), then groups of 4
  for (int group = 2; k < max_iters; group = 4) {
    const int kend = k + group < max_iters ? k + group : max_iters;
    for (; k < kend; ++k) {
      note_launch();
      lf_iter_kernel<<<dim3(tiles_x * tiles_y, (unsigned)B), kLFThreads, smem, s>>>(
          buf[k & 1], buf[(k + 1) & 1], H, W, r, tiles_x, k, cnt + (k % 3) * B, cnt + ((k + 1) % 3) * B,
          cnt + ((k + 2) % 3) * B, tot + (k + 1) % 3, tot + (k + 2) % 3, nit);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    unsigned long long left = 0;
    if ((e = cudaMemcpyAsync(&left, tot + k % 3, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    if (left == 0) break;
  }
  note_launch();
  lf_settle_kernel<<<dim3(frames_grid_x(HW), (unsigned)B), 256, 0, s>>>(buf0, buf1, HW, nit);
  if (iters && (e = cudaMemcpyAsync(iters, nit, B * 4, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_gather_frames(const float* src, float* dst, int64_t HW, const int64_t* idx, int64_t C, bool scatter,
                                 cudaStream_t s) {
  for (int64_t b0 = 0; b0 < C; b0 += 65535) {
    const int64_t nb = C - b0 < 65535 ? C - b0 : 65535;
    note_launch();
    gather_frames_kernel<<<dim3(frames_grid_x(HW), (unsigned)nb), 256, 0, s>>>(
        scatter ? src + b0 * HW : src, scatter ? dst : dst + b0 * HW, HW, idx + b0, scatter);
  }
  return cudaGetLastError();
}

cudaError_t launch_scatter_status(const uint32_t* st, const int32_t* it, const unsigned* vc, const int64_t* idx,
                                  int64_t C, uint32_t* status, int32_t* iters, unsigned* vcount, uint32_t bits,
                                  cudaStream_t s) {
  note_launch();
  scatter_status_kernel<<<(unsigned)((C + 255) / 256), 256, 0, s>>>(st, it, vc, idx, C, status, iters, vcount, bits);
  return cudaGetLastError();
}

cudaError_t launch_valid_counts(const float* out, int64_t HW, int64_t C, const int64_t* n_valid, unsigned* vcount,
                                cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(vcount, 0, (size_t)C * 8, s);
  if (e != cudaSuccess) return e;
  for (int64_t b0 = 0; b0 < C; b0 += 65535) {
    const int64_t nb = C - b0 < 65535 ? C - b0 : 65535;
    note_launch();
    valid_counts_kernel<<<dim3(frames_grid_x(HW), (unsigned)nb), 256, 0, s>>>(out + b0 * HW, HW, n_valid + b0,
                                                                               vcount + 2 * b0);
  }
  return cudaGetLastError();
}

}  // namespace dfc
