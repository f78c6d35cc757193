// Operator-surface and stage kernels (batched [B][H][W] float32).
//
// These implement the reference's 7-function backend surface
// (_native_ops.pyx / _numpy_ops.py) and the numpy-side pipeline stages one op
// per launch.  They back the `cuda` plug-in backend, the op-level parity
// tests, and the staged pipeline used for configurations the fused kernel
// does not cover (and for the rare frames needing >1 large-fill iteration).
// The hot path is fused.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "dfc_common.cuh"
#include "median_networks.cuh"

namespace dfc {

std::atomic<unsigned long long> g_kernel_launches{0};

namespace {

constexpr int kRowTile = 256;
constexpr int kColTileX = 32;
constexpr int kColTileY = 64;
constexpr int kMaxSmemFloats = 12 * 1024;  // 48 KB default dynamic smem

inline unsigned ceil_div(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// ---------------------------------------------------------------------------
// 1-D running min/max along rows (axis=1) or columns (axis=0).  Replicate
// border == clipped window for min/max, so indices are
// simply clamped.  The radius is clamped to the line length (a window wider
// than the line sees the whole line either way).
// ---------------------------------------------------------------------------
template <class Op>
__global__ void row_minmax_kernel(const float* __restrict__ in, float* __restrict__ out, int W, int r,
                                  int64_t nrows, bool use_smem) {
  extern __shared__ float seg[];
  const int ntiles = (W + kRowTile - 1) / kRowTile;
  const int64_t bid = blockIdx.x;
  const int64_t row = bid / ntiles;
  if (row >= nrows) return;
  const int x0 = (int)(bid % ntiles) * kRowTile;
  const float* src = in + row * W;
  const int x = x0 + threadIdx.x;
  if (use_smem) {
    const int S = kRowTile + 2 * r;
    for (int i = threadIdx.x; i < S; i += blockDim.x) seg[i] = __ldg(src + clampi(x0 - r + i, W));
    __syncthreads();
    if (x < W) {
      float m = seg[threadIdx.x];
      for (int d = 1; d <= 2 * r; ++d) m = Op::apply(m, seg[threadIdx.x + d]);
      out[row * W + x] = m;
    }
  } else if (x < W) {
    float m = __ldg(src + clampi(x - r, W));
    for (int d = -r + 1; d <= r; ++d) m = Op::apply(m, __ldg(src + clampi(x + d, W)));
    out[row * W + x] = m;
  }
}

template <class Op>
__global__ void col_minmax_kernel(const float* __restrict__ in, float* __restrict__ out, int H, int W, int r,
                                  bool use_smem) {
  extern __shared__ float seg[];  // [(kColTileY + 2r)][kColTileX]
  const int64_t b = blockIdx.z;
  const int x = blockIdx.x * kColTileX + threadIdx.x;
  const int y0 = blockIdx.y * kColTileY;
  const float* src = in + b * (int64_t)H * W;
  float* dst = out + b * (int64_t)H * W;
  const int xc = min(x, W - 1);
  if (use_smem) {
    const int S = kColTileY + 2 * r;
    for (int i = threadIdx.y; i < S; i += blockDim.y)
      seg[i * kColTileX + threadIdx.x] = __ldg(src + (int64_t)clampi(y0 - r + i, H) * W + xc);
    __syncthreads();
    if (x >= W) return;
    for (int j = threadIdx.y; j < kColTileY && y0 + j < H; j += blockDim.y) {
      float m = seg[j * kColTileX + threadIdx.x];
      for (int d = 1; d <= 2 * r; ++d) m = Op::apply(m, seg[(j + d) * kColTileX + threadIdx.x]);
      dst[(int64_t)(y0 + j) * W + x] = m;
    }
  } else {
    if (x >= W) return;
    for (int j = threadIdx.y; j < kColTileY && y0 + j < H; j += blockDim.y) {
      const int y = y0 + j;
      float m = __ldg(src + (int64_t)clampi(y - r, H) * W + x);
      for (int d = -r + 1; d <= r; ++d) m = Op::apply(m, __ldg(src + (int64_t)clampi(y + d, H) * W + x));
      dst[(int64_t)y * W + x] = m;
    }
  }
}

// ---------------------------------------------------------------------------
// Max/min over an arbitrary (dy,dx) offset list, replicate border
// (_native_ops.pyx:158-195).  Offsets travel as kernel parameters.
// ---------------------------------------------------------------------------
constexpr int kMaxOffsets = 4096;
struct OffsetList {
  int n, ry, rx;
  int8_t dy[kMaxOffsets];
  int8_t dx[kMaxOffsets];
};

template <class Op>
__global__ void offsets_kernel(const float* __restrict__ in, float* __restrict__ out, int H, int W,
                               const __grid_constant__ OffsetList offs) {
  extern __shared__ float tile[];  // [(16 + 2ry)][(32 + 2rx)]
  const int64_t b = blockIdx.z;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 16;
  const float* src = in + b * (int64_t)H * W;
  const int TW = 32 + 2 * offs.rx, TH = 16 + 2 * offs.ry;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int i = tid; i < TW * TH; i += 32 * 16) {
    const int ty = i / TW, tx = i % TW;
    tile[i] = __ldg(src + (int64_t)clampi(y0 - offs.ry + ty, H) * W + clampi(x0 - offs.rx + tx, W));
  }
  __syncthreads();
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  if (x >= W || y >= H) return;
  const int cy = threadIdx.y + offs.ry, cx = threadIdx.x + offs.rx;
  float m = tile[(cy + offs.dy[0]) * TW + cx + offs.dx[0]];
  for (int t = 1; t < offs.n; ++t) m = Op::apply(m, tile[(cy + offs.dy[t]) * TW + cx + offs.dx[t]]);
  out[b * (int64_t)H * W + (int64_t)y * W + x] = m;
}

// ---------------------------------------------------------------------------
// Median of the size x size replicate-clamped window (duplicates counted).
// Sizes 3 and 5 run the pruned Batcher network on registers; other sizes use
// an exact rank test (value whose rank interval contains the middle index).
// ---------------------------------------------------------------------------
#define DFC_CSWAP(a, b)            \
  do {                             \
    const float lo_ = fminf(a, b); \
    const float hi_ = fmaxf(a, b); \
    a = lo_;                       \
    b = hi_;                       \
  } while (0)

template <int S>
__global__ void median_net_kernel(const float* __restrict__ in, float* __restrict__ out, int H, int W) {
  const int64_t b = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= W || y >= H) return;
  const float* src = in + b * (int64_t)H * W;
  constexpr int R = S / 2;
  float v[S * S];
#pragma unroll
  for (int dy = -R; dy <= R; ++dy)
#pragma unroll
    for (int dx = -R; dx <= R; ++dx)
      v[(dy + R) * S + dx + R] = __ldg(src + (int64_t)clampi(y + dy, H) * W + clampi(x + dx, W));
  if constexpr (S == 3) {
    DFC_MEDNET9_APPLY(v);
  } else {
    DFC_MEDNET25_APPLY(v);
  }
  out[b * (int64_t)H * W + (int64_t)y * W + x] = v[(S * S) / 2];
}

__global__ void median_rank_kernel(const float* __restrict__ in, float* __restrict__ out, int H, int W, int size) {
  const int64_t b = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= W || y >= H) return;
  const float* src = in + b * (int64_t)H * W;
  const int r = size / 2, n = size * size, mid = n / 2;
  float result = 0.0f;
  for (int i = 0; i < n; ++i) {
    const float vi = __ldg(src + (int64_t)clampi(y + i / size - r, H) * W + clampi(x + i % size - r, W));
    int less = 0, le = 0;
    for (int j = 0; j < n; ++j) {
      const float vj = __ldg(src + (int64_t)clampi(y + j / size - r, H) * W + clampi(x + j % size - r, W));
      less += vj < vi;
      le += vj <= vi;
    }
    if (less <= mid && mid < le) {
      result = vi;
      break;
    }
  }
  out[b * (int64_t)H * W + (int64_t)y * W + x] = result;
}

// ---------------------------------------------------------------------------
// Separable Gaussian line pass.  EXACT: float64 with explicit non-fused
// multiply and add in tap order (the reference's numpy order,
// _numpy_ops.py:61-73: tmp = 0; tmp += w_t * v_t).  Fast: float32 FMA.
// ---------------------------------------------------------------------------
struct Taps {
  int k;
  double w[64];
  float wf[64];
};

template <bool EXACT, typename TIn, typename TOut>
__global__ void gauss_row_kernel(const TIn* __restrict__ in, TOut* __restrict__ out, int W, int64_t nrows,
                                 const __grid_constant__ Taps taps) {
  const int ntiles = (W + kRowTile - 1) / kRowTile;
  const int64_t row = blockIdx.x / ntiles;
  if (row >= nrows) return;
  const int x = (int)(blockIdx.x % ntiles) * kRowTile + threadIdx.x;
  if (x >= W) return;
  const TIn* src = in + row * W;
  const int r = taps.k / 2;
  if constexpr (EXACT) {
    double a = 0.0;
    for (int t = 0; t < taps.k; ++t) a = __dadd_rn(a, __dmul_rn(taps.w[t], (double)src[clampi(x + t - r, W)]));
    out[row * W + x] = (TOut)a;
  } else {
    float a = 0.0f;
    for (int t = 0; t < taps.k; ++t) a = fmaf(taps.wf[t], (float)src[clampi(x + t - r, W)], a);
    out[row * W + x] = (TOut)a;
  }
}

template <bool EXACT, typename TIn>
__global__ void gauss_col_kernel(const TIn* __restrict__ in, float* __restrict__ out, int H, int W,
                                 const __grid_constant__ Taps taps) {
  const int64_t b = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= W || y >= H) return;
  const TIn* src = in + b * (int64_t)H * W;
  const int r = taps.k / 2;
  if constexpr (EXACT) {
    double a = 0.0;
    for (int t = 0; t < taps.k; ++t)
      a = __dadd_rn(a, __dmul_rn(taps.w[t], (double)src[(int64_t)clampi(y + t - r, H) * W + x]));
    out[b * (int64_t)H * W + (int64_t)y * W + x] = __double2float_rn(a);
  } else {
    float a = 0.0f;
    for (int t = 0; t < taps.k; ++t) a = fmaf(taps.wf[t], (float)src[(int64_t)clampi(y + t - r, H) * W + x], a);
    out[b * (int64_t)H * W + (int64_t)y * W + x] = a;
  }
}

// ---------------------------------------------------------------------------
// Bilateral (_native_ops.pyx:340-369 / _numpy_ops.py:76-95).  EXACT follows
// the numpy backend in float64: w = exp(s*inv2_space + diff^2*inv2_value),
// num += w*q, den += w, (float)(num/den).  Fast: float32 centre-relative
// c + sum w (q-c) / sum w with exp2.
// ---------------------------------------------------------------------------
template <bool EXACT>
__global__ void bilateral_kernel(const float* __restrict__ in, float* __restrict__ out, int H, int W, int size,
                                 double inv2_value, double inv2_space) {
  const int64_t b = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= W || y >= H) return;
  const float* src = in + b * (int64_t)H * W;
  const int r = size / 2;
  const float c = src[(int64_t)y * W + x];
  if constexpr (EXACT) {
    const double c64 = (double)c;
    double num = 0.0, den = 0.0;
    for (int dy = -r; dy <= r; ++dy) {
      const float* rowp = src + (int64_t)clampi(y + dy, H) * W;
      for (int dx = -r; dx <= r; ++dx) {
        const double q = (double)rowp[clampi(x + dx, W)];
        const double diff = __dadd_rn(q, -c64);
        const double e = __dadd_rn((double)(dy * dy + dx * dx) * inv2_space,
                                   __dmul_rn(__dmul_rn(diff, diff), inv2_value));
        const double wgt = exp(e);
        num = __dadd_rn(num, __dmul_rn(wgt, q));
        den = __dadd_rn(den, wgt);
      }
    }
    out[b * (int64_t)H * W + (int64_t)y * W + x] = __double2float_rn(num / den);
  } else {
    const float kl = 1.4426950408889634f;
    const float ks = (float)inv2_space * kl, kv = (float)inv2_value * kl;
    float acc = 0.0f, den = 0.0f;
    for (int dy = -r; dy <= r; ++dy) {
      const float* rowp = src + (int64_t)clampi(y + dy, H) * W;
      for (int dx = -r; dx <= r; ++dx) {
        const float d = rowp[clampi(x + dx, W)] - c;
        const float wgt = exp2f(fmaf(kv * d, d, ks * (float)(dy * dy + dx * dx)));
        acc = fmaf(wgt, d, acc);
        den += wgt;
      }
    }
    out[b * (int64_t)H * W + (int64_t)y * W + x] = c + acc / den;
  }
}

// ---------------------------------------------------------------------------
// Stage kernels
// ---------------------------------------------------------------------------
__global__ void invert_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n_per_frame,
                              int64_t total, float off, uint32_t* status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = in[i];
    out[i] = v > kValid ? off - v : 0.0f;
    if (v >= off && status) atomicOr(status + i / n_per_frame, DFC_ST_RANGE);
  }
}

// per-frame: blockIdx.y = frame, blockIdx.x strides pixels
__global__ void validate_kernel(const float* __restrict__ in, int64_t n_per_frame, uint32_t* status,
                                int64_t* n_valid) {
  const int64_t b = blockIdx.y;
  const float* src = in + b * n_per_frame;
  unsigned long long cnt = 0;
  uint32_t bits = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_per_frame;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = src[i];
    if (!isfinite(v)) bits |= DFC_ST_NONFINITE;
    if (v < 0.0f) bits |= DFC_ST_NEGATIVE;
    cnt += v > kValid;
  }
  bits = __reduce_or_sync(0xffffffffu, bits);
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) {
    if (bits) atomicOr(status + b, bits);
    if (n_valid && cnt) atomicAdd((unsigned long long*)(n_valid + b), cnt);
  }
}

__global__ void count_empty_kernel(const float* __restrict__ in, int64_t n_per_frame, int64_t* counts) {
  const int64_t b = blockIdx.y;
  const float* src = in + b * n_per_frame;
  unsigned long long cnt = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_per_frame;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt += !(src[i] > kValid);
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd((unsigned long long*)(counts + b), cnt);
}

__global__ void masked_fill_kernel(const float* __restrict__ cur, const float* __restrict__ dil,
                                   float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = cur[i];
    out[i] = v > kValid ? v : dil[i];
  }
}

__global__ void reimpose_kernel(const float* __restrict__ bl, const float* __restrict__ m, float* __restrict__ out,
                                int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = m[i] > kValid ? bl[i] : 0.0f;
}

__global__ void bin_select_kernel(const float* __restrict__ d, const float* __restrict__ inv, float* __restrict__ out,
                                  int64_t n, float lo, float hi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = d[i];
    out[i] = (v > lo && v <= hi) ? inv[i] : 0.0f;
  }
}

__global__ void max2_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out,
                            int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = fmaxf(a[i], b[i]);
}

// extend_to_top (morphology.py:81-96): one thread per (frame, column)
__global__ void extend_kernel(const float* __restrict__ in, float* __restrict__ out, int H, int W) {
  const int64_t b = blockIdx.y;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= W) return;
  const float* src = in + b * (int64_t)H * W;
  float* dst = out + b * (int64_t)H * W;
  int r0 = H;
  float top = 0.0f;
  for (int y = 0; y < H; ++y) {
    const float v = src[(int64_t)y * W + x];
    if (v > kValid) {
      r0 = y;
      top = v;
      break;
    }
  }
  for (int y = 0; y < H; ++y) dst[(int64_t)y * W + x] = (y < r0 && r0 < H) ? top : src[(int64_t)y * W + x];
}

__global__ void iter_update_kernel(const int64_t* counts, int32_t* iters, int64_t B, unsigned long long* total) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B) return;
  const long long c = counts[b];
  if (c > 0) {
    if (iters) iters[b] += 1;
    atomicAdd(total, (unsigned long long)c);
  }
}

__global__ void finalize_status_kernel(const int64_t* n_valid, uint32_t* status, int64_t B) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b < B && n_valid[b] == 0) status[b] |= DFC_ST_DEGENERATE;
}

__global__ void or_status_kernel(uint32_t* status, uint32_t bits) { *status |= bits; }

unsigned grid1d(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (unsigned)(g > 148 * 32 ? 148 * 32 : (g < 1 ? 1 : g));
}

}  // namespace

// ===========================================================================
// launchers
// ===========================================================================
cudaError_t launch_line_minmax(const float* in, float* out, int64_t B, int H, int W, int radius, bool is_min,
                               int axis, cudaStream_t s) {
  if (axis == 1) {
    note_launch();
    const int r = radius < W - 1 ? radius : W - 1;
    const int64_t nrows = B * H;
    const bool smem = kRowTile + 2 * r <= kMaxSmemFloats;
    const size_t sm = smem ? (size_t)(kRowTile + 2 * r) * 4 : 0;
    const int64_t nblk = nrows * ((W + kRowTile - 1) / kRowTile);
    if (nblk > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    if (is_min)
      row_minmax_kernel<MinOp><<<(unsigned)nblk, kRowTile, sm, s>>>(in, out, W, r, nrows, smem);
    else
      row_minmax_kernel<MaxOp><<<(unsigned)nblk, kRowTile, sm, s>>>(in, out, W, r, nrows, smem);
  } else {
    const int r = radius < H - 1 ? radius : H - 1;
    const bool smem = (kColTileY + 2 * r) * kColTileX <= kMaxSmemFloats;
    const size_t sm = smem ? (size_t)(kColTileY + 2 * r) * kColTileX * 4 : 0;
    for (int64_t b0 = 0; b0 < B; b0 += 65535) {
      note_launch();
      const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
      dim3 grid(ceil_div(W, kColTileX), ceil_div(H, kColTileY), (unsigned)nb);
      dim3 block(kColTileX, 8);
      const float* i0 = in + b0 * (int64_t)H * W;
      float* o0 = out + b0 * (int64_t)H * W;
      if (is_min)
        col_minmax_kernel<MinOp><<<grid, block, sm, s>>>(i0, o0, H, W, r, smem);
      else
        col_minmax_kernel<MaxOp><<<grid, block, sm, s>>>(i0, o0, H, W, r, smem);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_offsets_minmax(const float* in, float* out, int64_t B, int H, int W, const int32_t* offs, int n,
                                  bool is_min, cudaStream_t s) {
  if (n < 1 || n > kMaxOffsets) return cudaErrorInvalidValue;
  OffsetList L;
  L.n = n;
  L.ry = 0;
  L.rx = 0;
  for (int t = 0; t < n; ++t) {
    int dy = offs[2 * t], dx = offs[2 * t + 1];
    if (dy < -127 || dy > 127 || dx < -127 || dx > 127) return cudaErrorInvalidValue;
    // clamp offsets to the frame: beyond the frame the clamped sample is the
    // edge pixel either way, so a clamped offset gives the identical sample.
    dy = dy < -(H - 1) ? -(H - 1) : (dy > H - 1 ? H - 1 : dy);
    dx = dx < -(W - 1) ? -(W - 1) : (dx > W - 1 ? W - 1 : dx);
    L.dy[t] = (int8_t)dy;
    L.dx[t] = (int8_t)dx;
    L.ry = abs(dy) > L.ry ? abs(dy) : L.ry;
    L.rx = abs(dx) > L.rx ? abs(dx) : L.rx;
  }
  const size_t sm = (size_t)(32 + 2 * L.rx) * (16 + 2 * L.ry) * 4;
  if (sm > 200 * 1024) return cudaErrorInvalidValue;
  auto kmax = offsets_kernel<MaxOp>;
  auto kmin = offsets_kernel<MinOp>;
  cudaFuncSetAttribute(is_min ? kmin : kmax, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    note_launch();
    const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
    dim3 grid(ceil_div(W, 32), ceil_div(H, 16), (unsigned)nb);
    dim3 block(32, 16);
    const float* i0 = in + b0 * (int64_t)H * W;
    float* o0 = out + b0 * (int64_t)H * W;
    if (is_min)
      kmin<<<grid, block, sm, s>>>(i0, o0, H, W, L);
    else
      kmax<<<grid, block, sm, s>>>(i0, o0, H, W, L);
  }
  return cudaGetLastError();
}

cudaError_t launch_median(const float* in, float* out, int64_t B, int H, int W, int size, cudaStream_t s) {
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    note_launch();
    const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
    dim3 block(32, 4);
    dim3 grid(ceil_div(W, 32), ceil_div(H, 4), (unsigned)nb);
    const float* i0 = in + b0 * (int64_t)H * W;
    float* o0 = out + b0 * (int64_t)H * W;
    if (size == 3)
      median_net_kernel<3><<<grid, block, 0, s>>>(i0, o0, H, W);
    else if (size == 5)
      median_net_kernel<5><<<grid, block, 0, s>>>(i0, o0, H, W);
    else
      median_rank_kernel<<<grid, block, 0, s>>>(i0, o0, H, W, size);
  }
  return cudaGetLastError();
}

cudaError_t launch_gauss_line(const float* in, void* out, int64_t B, int H, int W, const double* w, int k, int axis,
                              bool exact, bool in_is_f64, bool out_is_f64, cudaStream_t s) {
  if (k < 1 || k > 64) return cudaErrorInvalidValue;
  Taps T;
  T.k = k;
  for (int t = 0; t < k; ++t) {
    T.w[t] = w[t];
    T.wf[t] = (float)w[t];
  }
  if (axis == 1) {
    note_launch();
    const int64_t nrows = B * H;
    const int64_t nblk = nrows * ((W + kRowTile - 1) / kRowTile);
    const float* fin = in;
    if (exact && out_is_f64)
      gauss_row_kernel<true, float, double><<<(unsigned)nblk, kRowTile, 0, s>>>(fin, (double*)out, W, nrows, T);
    else if (!exact && !out_is_f64)
      gauss_row_kernel<false, float, float><<<(unsigned)nblk, kRowTile, 0, s>>>(fin, (float*)out, W, nrows, T);
    else
      return cudaErrorInvalidValue;
  } else {
    for (int64_t b0 = 0; b0 < B; b0 += 65535) {
      note_launch();
      const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
      dim3 block(32, 8);
      dim3 grid(ceil_div(W, 32), ceil_div(H, 8), (unsigned)nb);
      float* o0 = (float*)out + b0 * (int64_t)H * W;
      if (in_is_f64) {
        const double* i0 = (const double*)in + b0 * (int64_t)H * W;
        gauss_col_kernel<true, double><<<grid, block, 0, s>>>(i0, o0, H, W, T);
      } else {
        const float* i0 = in + b0 * (int64_t)H * W;
        if (exact)
          gauss_col_kernel<true, float><<<grid, block, 0, s>>>(i0, o0, H, W, T);
        else
          gauss_col_kernel<false, float><<<grid, block, 0, s>>>(i0, o0, H, W, T);
      }
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_bilateral(const float* in, float* out, int64_t B, int H, int W, int size, double sv, double ss,
                             bool exact, cudaStream_t s) {
  const double iv = -0.5 / (sv * sv), is = -0.5 / (ss * ss);
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    note_launch();
    const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
    dim3 block(32, 4);
    dim3 grid(ceil_div(W, 32), ceil_div(H, 4), (unsigned)nb);
    const float* i0 = in + b0 * (int64_t)H * W;
    float* o0 = out + b0 * (int64_t)H * W;
    if (exact)
      bilateral_kernel<true><<<grid, block, 0, s>>>(i0, o0, H, W, size, iv, is);
    else
      bilateral_kernel<false><<<grid, block, 0, s>>>(i0, o0, H, W, size, iv, is);
  }
  return cudaGetLastError();
}

cudaError_t launch_invert(const float* in, float* out, int64_t n_per_frame, int64_t B, float offset,
                          uint32_t* status, cudaStream_t s) {
  const int64_t n = n_per_frame * B;
  note_launch();
  invert_kernel<<<grid1d(n), 256, 0, s>>>(in, out, n_per_frame, n, offset, status);
  return cudaGetLastError();
}

static dim3 frame_grid(int64_t n_per_frame, int64_t nb) {
  int64_t gx = (n_per_frame + 1023) / 1024;
  if (gx > 64) gx = 64;
  return dim3((unsigned)(gx < 1 ? 1 : gx), (unsigned)nb);
}

cudaError_t launch_validate(const float* in, int64_t n_per_frame, int64_t B, uint32_t* status, int64_t* n_valid,
                            cudaStream_t s) {
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    note_launch();
    const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
    validate_kernel<<<frame_grid(n_per_frame, nb), 256, 0, s>>>(in + b0 * n_per_frame, n_per_frame, status + b0,
                                                                n_valid ? n_valid + b0 : nullptr);
  }
  return cudaGetLastError();
}

cudaError_t launch_count_empty(const float* in, int64_t n_per_frame, int64_t B, int64_t* counts, cudaStream_t s) {
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    note_launch();
    const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
    count_empty_kernel<<<frame_grid(n_per_frame, nb), 256, 0, s>>>(in + b0 * n_per_frame, n_per_frame, counts + b0);
  }
  return cudaGetLastError();
}

cudaError_t launch_masked_fill(const float* cur, const float* dil, float* out, int64_t n, cudaStream_t s) {
  note_launch();
  masked_fill_kernel<<<grid1d(n), 256, 0, s>>>(cur, dil, out, n);
  return cudaGetLastError();
}

cudaError_t launch_extend_to_top(const float* in, float* out, int64_t B, int H, int W, cudaStream_t s) {
  for (int64_t b0 = 0; b0 < B; b0 += 65535) {
    note_launch();
    const int64_t nb = B - b0 < 65535 ? B - b0 : 65535;
    extend_kernel<<<dim3(ceil_div(W, 128), (unsigned)nb), 128, 0, s>>>(in + b0 * (int64_t)H * W,
                                                                       out + b0 * (int64_t)H * W, H, W);
  }
  return cudaGetLastError();
}

namespace {
__global__ void decode_raw16_kernel(const uint16_t* __restrict__ raw, float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)raw[i] * 0.00390625f;  // exact (kitti_io.py:53)
}

__global__ void encode_raw16_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t n_per_frame,
                                    int64_t n, uint32_t* status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = in[i];
    // np.rint(f64(v) * 256) clipped (kitti_io.py:64-65); v * 256 is exact in float32
    out[i] = (uint16_t)fminf(fmaxf(rintf(v * 256.0f), 0.0f), 65535.0f);
    if (status && v >= 256.0f) atomicOr(status + i / n_per_frame, DFC_ST_ENCODE);
  }
}
}  // namespace

cudaError_t launch_decode_raw16(const uint16_t* raw, float* out, int64_t n, cudaStream_t s) {
  note_launch();
  decode_raw16_kernel<<<grid1d(n), 256, 0, s>>>(raw, out, n);
  return cudaGetLastError();
}

cudaError_t launch_encode_raw16(const float* in, uint16_t* out, int64_t n_per_frame, int64_t n, uint32_t* status,
                                cudaStream_t s) {
  note_launch();
  encode_raw16_kernel<<<grid1d(n), 256, 0, s>>>(in, out, n_per_frame, n, status);
  return cudaGetLastError();
}

cudaError_t launch_reimpose(const float* blurred, const float* mask_src, float* out, int64_t n, cudaStream_t s) {
  note_launch();
  reimpose_kernel<<<grid1d(n), 256, 0, s>>>(blurred, mask_src, out, n);
  return cudaGetLastError();
}

cudaError_t launch_bin_select(const float* direct, const float* inv, float* out, int64_t n, float lo, float hi,
                              cudaStream_t s) {
  note_launch();
  bin_select_kernel<<<grid1d(n), 256, 0, s>>>(direct, inv, out, n, lo, hi);
  return cudaGetLastError();
}

cudaError_t launch_max2(const float* a, const float* b, float* out, int64_t n, cudaStream_t s) {
  note_launch();
  max2_kernel<<<grid1d(n), 256, 0, s>>>(a, b, out, n);
  return cudaGetLastError();
}

cudaError_t launch_iter_update(const int64_t* counts, int32_t* iters, int64_t B, unsigned long long* total,
                               cudaStream_t s) {
  note_launch();
  iter_update_kernel<<<ceil_div(B, 256), 256, 0, s>>>(counts, iters, B, total);
  return cudaGetLastError();
}

cudaError_t launch_or_status(uint32_t* status, uint32_t bits, cudaStream_t s) {
  note_launch();
  or_status_kernel<<<1, 1, 0, s>>>(status, bits);
  return cudaGetLastError();
}

cudaError_t launch_finalize_status(const int64_t* n_valid, uint32_t* status, int64_t B, cudaStream_t s) {
  note_launch();
  finalize_status_kernel<<<ceil_div(B, 256), 256, 0, s>>>(n_valid, status, B);
  return cudaGetLastError();
}

}  // namespace dfc
