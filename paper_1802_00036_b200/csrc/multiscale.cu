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
#include "lane_ops.cuh"
#include "tmem.cuh"

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
                                                             unsigned* __restrict__ vcount,
                                                             const __grid_constant__ BinParams p) {
  constexpr int IW = kTX + 2 * R, IH = kTY + 2 * R;
  __shared__ float sb[3][IH * IW];
  __shared__ unsigned s_umax;
  const int64_t b = blockIdx.z;
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  const float* src = in + b * (int64_t)H * W;
  if (threadIdx.x == 0) s_umax = 0;
  unsigned um = 0, nv = 0;
  for (int i = threadIdx.x; i < IH * IW; i += kThreads) {
    const int iy = i / IW, ix = i - iy * IW;
    const int gy = y0 - R + iy, gx = x0 - R + ix;
    const float d = __ldg(src + (int64_t)clampi(gy, H) * W + clampi(gx, W));
    if (gy >= 0 && gy < H && gx >= 0 && gx < W) um = max(um, __float_as_uint(d));
    // valid inputs of the tile itself (each pixel in exactly one tile)
    if (iy >= R && iy < R + kTY && ix >= R && ix < R + kTX && gy < H && gx < W) nv += d > kValid;
    const float v = d > kValid ? p.md - d : 0.0f;  // depth_core.invert
    sb[0][i] = d <= p.edge_near ? v : 0.0f;
    sb[1][i] = (d > p.edge_near && d <= p.edge_far) ? v : 0.0f;
    sb[2][i] = d > p.edge_far ? v : 0.0f;
  }
  um = __reduce_max_sync(0xffffffffu, um);
  nv = __reduce_add_sync(0xffffffffu, nv);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicMax(&s_umax, um);
  if ((threadIdx.x & 31) == 0 && nv) atomicAdd(vcount + 2 * b, nv);
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

// ---------------------------------------------------------------------------
// Streaming variant for the default bin kernels (near FULL7, medium DIAMOND7,
// far DIAMOND5).  Each warp owns 120 columns (lanes 1..30 of 32 x 4 columns;
// one lane of halo per side covers the radius 3) and walks the frame top-down
// in 4-row blocks, warps independent.  FULL7 = vertical max7 then horizontal
// max7; DIAMOND(2r+1) = cross3 applied r times.  Out-of-frame rows and columns
// are zero between the stages (max identity for maps >= 0): for these
// rectangle-convex shapes the dilation clipped to the frame equals the
// reference's replicate border.  Outputs trail the input
// by 3 rows.
// ---------------------------------------------------------------------------
constexpr int kMsOwn = 120;
constexpr int kMsWarps = 4;

struct MsFastParams {
  float md, edge_near, edge_far;
  int64_t nframes;
  int nseg, seg_rows;  // row segments per column slice, rows per segment (a multiple of 4)
};

__device__ __forceinline__ F4 cross3(const F4& up, const F4& mid, const F4& dn) {
  const Ext<1> e = ext_row<1>(mid);
  F4 o;
#pragma unroll
  for (int c = 0; c < 4; ++c) o.v[c] = fmx3(fmx3(up.v[c], mid.v[c], dn.v[c]), e.e[c], e.e[c + 2]);
  return o;
}

// one cross3 stage over a 4-row block with 2 carried rows; zeroes rows outside
// [0, H) (row of output j: t0 - lag + j) and out-of-frame columns
template <bool EDGE, bool WOOB>
__device__ __forceinline__ void cross3_block(F4 carry[2], const F4 in4[kB], F4 out[kB], int row0, int H,
                                             unsigned oob) {
  const F4 in[kB + 2] = {carry[0], carry[1], in4[0], in4[1], in4[2], in4[3]};
#pragma unroll
  for (int j = 0; j < kB; ++j) {
    out[j] = cross3(in[j], in[j + 1], in[j + 2]);
    if (EDGE && (row0 + j < 0 || row0 + j >= H)) set_row(out[j], 0.f);
    if (WOOB) fix_oob(out[j], oob, 0.f);
  }
  carry[0] = in4[2];
  carry[1] = in4[3];
}

// Carried rows live in tensor memory (tmem.cuh): near-bin box rows nc (6)
// at TMEM columns 0..23, the cross3 carries m1 m2 m3 f1 f2 (2 rows each) at
// 24..63; fd (the far bin's one-row delay) and the prefetched rows stay in
// registers.  184 registers (2 CTAs / SM) became <= 128 (4 CTAs / SM).
constexpr int kTmNc = 0, kTmM1 = 24, kTmM2 = 32, kTmM3 = 40, kTmF1 = 48, kTmF2 = 56, kMsTmCols = 128;
struct MsState {
  F4 fd, nx[kB];
  unsigned um;
  float2 cnt[2];  // valid inputs (> 0.1) per column pair (RunStats.input_density, pipeline.py:138-141);
                  // out-of-frame columns load 0, so only the halo lanes 0 / 31 are left out at the end
  uint32_t tm;  // this thread's TMEM lane, column 0
};

// one 4-row block: input rows t0..t0+3 in, output rows t0-3..t0 out.  EDGE:
// rows may lie outside the frame; WOOB: the warp has out-of-frame columns.
// EDGE blocks also carry the row segment [ya, yb) the warp stores (rows outside
// it belong to the neighbouring segments, or are warm-up) and whether this
// block's input rows count towards the valid-input sum.
template <int VEC, bool EDGE, bool WOOB>
__device__ __forceinline__ void ms_block(MsState& S, const float* __restrict__ src, float* __restrict__ dst, int t0,
                                         int H, int W, int x0, unsigned oob, unsigned own, const MsFastParams& p,
                                         int ya = 0, int yb = 0, bool cnt_on = true) {
  F4 cur[kB];
#pragma unroll
  for (int j = 0; j < kB; ++j) {
    cur[j] = S.nx[j];
    if (!EDGE || t0 + kB + j < H)
      S.nx[j] = load4<VEC, true>(src + (int64_t)(t0 + kB + j) * W, x0, W);
    else
      set_row(S.nx[j], 0.f);
  }
  F4 nv[kB], mv[kB], fv[kB];
  // validity and bin membership as 1.0f / 0.0f (one FSET each, ALU pipe); the
  // selects and the valid-input count (RunStats.input_density, pipeline.py:138-141)
  // run on the FMA pipe in column pairs: x * 1 and x * 0 are exact, and the
  // medium bin inv - near - far is exactly inv or +0 (en < ef: one of near / far is 0)
#pragma unroll
  for (int j = 0; j < kB; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float2 v = make_float2(cur[j].v[2 * h], cur[j].v[2 * h + 1]);
      S.um = max(max(S.um, __float_as_uint(v.x)), __float_as_uint(v.y));
      const float2 q = make_float2(v.x > kValid ? 1.f : 0.f, v.y > kValid ? 1.f : 0.f);
      const float2 qn = make_float2(v.x <= p.edge_near ? 1.f : 0.f, v.y <= p.edge_near ? 1.f : 0.f);
      const float2 qf = make_float2(v.x > p.edge_far ? 1.f : 0.f, v.y > p.edge_far ? 1.f : 0.f);
      if (!EDGE || cnt_on) S.cnt[h] = __fadd2_rn(S.cnt[h], q);  // rows / columns outside the frame are 0
      // depth_core.invert: (md - v) * valid
      const float2 inv = __fmul2_rn(__ffma2_rn(v, make_float2(-1.f, -1.f), make_float2(p.md, p.md)), q);
      const float2 n2 = __fmul2_rn(inv, qn), f2 = __fmul2_rn(inv, qf);
      const float2 m2 = __fadd2_rn(__fadd2_rn(inv, make_float2(-n2.x, -n2.y)), make_float2(-f2.x, -f2.y));
      nv[j].v[2 * h] = n2.x, nv[j].v[2 * h + 1] = n2.y;
      fv[j].v[2 * h] = f2.x, fv[j].v[2 * h + 1] = f2.y;
      mv[j].v[2 * h] = m2.x, mv[j].v[2 * h + 1] = m2.y;
    }
  // near: FULL7 box (rows t0-3+j)
  F4 nb[kB];
  {
    F4 nc[6];
    tm_wait_st();  // the previous block's carry stores
    tm_ld_rows(S.tm + kTmNc, nc, 6);
    const F4 col[kB + 6] = {nc[0], nc[1], nc[2], nc[3], nc[4], nc[5], nv[0], nv[1], nv[2], nv[3]};
    F4 vv[kB];
    vwin3<OpMax>(col, vv);
#pragma unroll
    for (int j = 0; j < kB; ++j) nb[j] = hwin3<OpMax>(ext_row<3>(vv[j]));
    const F4 n6[6] = {nc[4], nc[5], nv[0], nv[1], nv[2], nv[3]};
    tm_st_rows(S.tm + kTmNc, n6, 6);
  }
  // medium: DIAMOND7 = cross3^3 (rows t0-1+j, t0-2+j, t0-3+j)
  F4 a1[kB], a2[kB], a3[kB];
  {
    F4 c[2];
    tm_ld_rows(S.tm + kTmM1, c, 2);
    cross3_block<EDGE, WOOB>(c, mv, a1, t0 - 1, H, oob);
    tm_st_rows(S.tm + kTmM1, c, 2);
    tm_ld_rows(S.tm + kTmM2, c, 2);
    cross3_block<EDGE, WOOB>(c, a1, a2, t0 - 2, H, oob);
    tm_st_rows(S.tm + kTmM2, c, 2);
    tm_ld_rows(S.tm + kTmM3, c, 2);
    cross3_block<EDGE, WOOB>(c, a2, a3, t0 - 3, H, oob);
    tm_st_rows(S.tm + kTmM3, c, 2);
  }
  // far: DIAMOND5 = cross3^2 (rows t0-2+j), delayed one row
  F4 b1[kB], b2[kB];
  {
    F4 c[2];
    tm_ld_rows(S.tm + kTmF1, c, 2);
    cross3_block<EDGE, WOOB>(c, fv, b1, t0 - 1, H, oob);
    tm_st_rows(S.tm + kTmF1, c, 2);
    tm_ld_rows(S.tm + kTmF2, c, 2);
    cross3_block<EDGE, WOOB>(c, b1, b2, t0 - 2, H, oob);
    tm_st_rows(S.tm + kTmF2, c, 2);
  }
  const F4 fr[kB] = {S.fd, b2[0], b2[1], b2[2]};
  S.fd = b2[3];
#pragma unroll
  for (int j = 0; j < kB; ++j) {
    const int y = t0 - 3 + j;
    if (EDGE && (y < ya || y >= yb)) continue;
    F4 o;
#pragma unroll
    for (int c = 0; c < 4; ++c) o.v[c] = fmx3(nb[j].v[c], a3[j].v[c], fr[j].v[c]);
    if (own) store4<VEC>(dst + (int64_t)y * W, x0, o, own);
  }
}

// Output rows [ya, yb) of the warp's columns (ya a multiple of 4; yb one too,
// or H).  A segment that starts inside the frame streams one warm-up block
// first: with zero carries, outputs from 3 rows below the first streamed row
// are exact (each output row depends on input rows y - 3 .. y + 3 only).
template <int VEC, bool WOOB>
__device__ __forceinline__ void ms_rows(MsState& S, const float* src, float* dst, int H, int W, int x0, unsigned oob,
                                        unsigned own, const MsFastParams& p, int ya, int yb) {
  // the lean body needs every row it touches inside the frame -- stages and
  // outputs down to t0 - 3 (t0 >= 4), the prefetch up to t0 + 7 (t0 + 8 <= H)
  // -- and its four output rows t0 - 3 .. t0 inside the segment
  int t0 = ya >= kB ? ya - kB : 0;
  const int tend = yb >= H ? H + 3 : yb + 1;  // the block at t0 = yb holds the segment's last rows
  const int lean0 = max(ya + kB, 4);
  for (; t0 < lean0 && t0 < tend; t0 += kB)
    ms_block<VEC, true, WOOB>(S, src, dst, t0, H, W, x0, oob, own, p, ya, yb, t0 >= ya && t0 < yb);
  for (; t0 + kB <= yb && t0 + 2 * kB <= H; t0 += kB) ms_block<VEC, false, WOOB>(S, src, dst, t0, H, W, x0, oob, own, p);
  for (; t0 < tend; t0 += kB)
    ms_block<VEC, true, WOOB>(S, src, dst, t0, H, W, x0, oob, own, p, ya, yb, t0 >= ya && t0 < yb);
}

template <int VEC>
__device__ __forceinline__ void ms_warp(const float* __restrict__ in, float* __restrict__ out, int H, int W,
                                        unsigned* __restrict__ umax, unsigned* __restrict__ vcount,
                                        const MsFastParams& p, int64_t b, int S0, int ya, int yb, int lane,
                                        uint32_t tm) {
  const float* src = in + b * (int64_t)H * W;
  float* dst = out + b * (int64_t)H * W;
  const int x0 = S0 - 4 + 4 * lane;
  unsigned oob = 0, own = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int x = x0 + c;
    oob |= (unsigned)(x < 0 || x >= W) << c;
    own |= (unsigned)(lane >= 1 && lane <= 30 && x < W) << c;
  }
  MsState S;
  S.tm = tm;
  tm_wait_st();  // the previous item's carry stores (persistent warps)
  {
    F4 z[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) set_row(z[i], 0.f);
    tm_st_rows(tm + kTmNc, z, 6);
    tm_st_rows(tm + kTmM1, z, 2);
    tm_st_rows(tm + kTmM2, z, 2);
    tm_st_rows(tm + kTmM3, z, 2);
    tm_st_rows(tm + kTmF1, z, 2);
    tm_st_rows(tm + kTmF2, z, 2);
  }
  set_row(S.fd, 0.f);
  S.um = 0;
  S.cnt[0] = S.cnt[1] = make_float2(0.f, 0.f);
  const int ts = ya >= kB ? ya - kB : 0;  // first streamed row (ms_rows)
#pragma unroll
  for (int j = 0; j < kB; ++j) {
    if (ts + j < H)
      S.nx[j] = load4<VEC, true>(src + (int64_t)(ts + j) * W, x0, W);
    else
      set_row(S.nx[j], 0.f);
  }
  if (__any_sync(kFull, oob != 0))
    ms_rows<VEC, true>(S, src, dst, H, W, x0, oob, own, p, ya, yb);
  else
    ms_rows<VEC, false>(S, src, dst, H, W, x0, oob, own, p, ya, yb);
  const unsigned um = __reduce_max_sync(kFull, S.um);
  // per-lane counts <= 4 H < 2^24: exact in float
  const unsigned mine = (unsigned)(S.cnt[0].x + S.cnt[0].y + S.cnt[1].x + S.cnt[1].y);
  const unsigned nv = __reduce_add_sync(kFull, lane >= 1 && lane <= 30 ? mine : 0u);
  if (lane == 0) atomicMax(umax + b, um);
  if (lane == 0 && nv) atomicAdd(vcount + 2 * b, nv);
}

template <int VEC>
__global__ void __launch_bounds__(kMsWarps * 32, 4) ms_fast_kernel(const float* __restrict__ in,
                                                                   float* __restrict__ out, int H, int W,
                                                                   unsigned* __restrict__ umax,
                                                                   unsigned* __restrict__ vcount,
                                                                   unsigned* __restrict__ work,
                                                                   const __grid_constant__ MsFastParams p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  static_assert(kMsWarps == 4, "one warp per TMEM lane quarter");
  __shared__ uint32_t s_tm;
  if (warp == 0) tm_alloc((uint32_t)__cvta_generic_to_shared(&s_tm), kMsTmCols);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tmbase = s_tm;
  // warps are numbered over (frame, 120-column slice) pairs, so a CTA may span
  // two frames and no warp of a CTA idles at the frame's right edge (with one
  // CTA per 480 columns, half the warps of the last CTA of a 1216-wide frame had
  // no columns and held their slot)
  // ... and over row segments: a round of 296 frames x 11 slices is 1.4 waves
  // of the 16 warps per SM, so whole-column items left the second wave 37 %
  // full (config 4: 9 %); with p.nseg segments per column the last wave is a
  // fraction of an item.  Items of a frame's segment are adjacent.
  const int nwf = (W + kMsOwn - 1) / kMsOwn;  // items per (frame, segment)
  // Warps are persistent and take items from a queue: a warp that finishes
  // (interior slices are ~20 % cheaper than the frame-edge ones) starts its
  // next item at once instead of holding its slot until the CTA's slowest
  // warp reaches the closing barrier.
  const unsigned total = (unsigned)(p.nframes * p.nseg * nwf);
  for (;;) {
    unsigned gw = 0;
    if (lane == 0) gw = atomicAdd(work, 1u);
    gw = __shfl_sync(kFull, gw, 0);
    if (gw >= total) break;
    const unsigned fs = gw / nwf;
    const int seg = (int)(fs % p.nseg);
    const int ya = seg * p.seg_rows, yb = min(H, ya + p.seg_rows);
    ms_warp<VEC>(in, out, H, W, umax, vcount, p, fs / p.nseg, (int)(gw % nwf) * kMsOwn, ya, yb, lane,
                 tmbase + ((uint32_t)(warp * 32) << 16));
  }
  tm_wait_st();
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (warp == 0) tm_dealloc(tmbase, kMsTmCols);
}


}  // namespace

bool multiscale_fast_kernels(const dfc_config& c) {
  return c.near_shape == DFC_SHAPE_FULL && c.near_size == 7 && c.med_shape == DFC_SHAPE_DIAMOND && c.med_size == 7 &&
         c.far_shape == DFC_SHAPE_DIAMOND && c.far_size == 5;
}

// kernel_offsets (capi.cu) for the three bins; false if a bin is wider than 7
bool multiscale_stage2_supported(const dfc_config& c) {
  return c.multiscale && c.near_size <= 2 * kMaxR + 1 && c.med_size <= 2 * kMaxR + 1 &&
         c.far_size <= 2 * kMaxR + 1;
}

cudaError_t launch_multiscale_stage2(const float* in, float* out, int64_t B, int H, int W, const dfc_config& c,
                                     const int32_t* const offs[3], const int n[3], unsigned* umax, unsigned* vcount,
                                     unsigned* work, cudaStream_t s) {
  if (multiscale_fast_kernels(c)) {
    MsFastParams q{c.max_depth, c.bin_edge_near, c.bin_edge_far, 0, 1, 0};
    q.nframes = B;
    // Row segments per column slice (each adds one 4-row warm-up block and the
    // per-item set-up).  Whole columns are best while they fill the GPU evenly
    // (measured: config 2's 1.4 waves lose 2.5 % to 4 segments -- a thin second
    // wave runs faster, the kernel is issue-bound per SM); segments pay when the
    // last wave is nearly empty (config 4: 1.09 waves, +4.5 % with 4 segments)
    // or the batch does not fill the SMs at all (single frames, small batches).
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t slots = (int64_t)sms * 4 * kMsWarps, items = B * ((W + kMsOwn - 1) / kMsOwn);
    int nseg = 1;
    if (items < slots)  // measured on 1216x352: 20 % off the whole call for batches of 1-16 frames, 13 % at 32
      nseg = (int)std::min<int64_t>(std::max<int64_t>(4, slots / (4 * items)), 16);
    else if (items > slots && items % slots != 0 && items % slots < slots / 4)
      nseg = 4;
    if (getenv("DFC_MS_NSEG")) nseg = atoi(getenv("DFC_MS_NSEG"));  // A/B runs
    q.nseg = std::max(1, std::min(nseg, H / 32));
    q.seg_rows = (((H + kB - 1) / kB + q.nseg - 1) / q.nseg) * kB;
    q.nseg = (H + q.seg_rows - 1) / q.seg_rows;
    const int64_t nw = B * q.nseg * ((W + kMsOwn - 1) / kMsOwn);
    const unsigned grid = (unsigned)std::min<int64_t>((nw + kMsWarps - 1) / kMsWarps, (int64_t)sms * 4);
    note_launch();
    if (W % 4 == 0)
      ms_fast_kernel<4><<<grid, kMsWarps * 32, 0, s>>>(in, out, H, W, umax, vcount, work, q);
    else if (W % 2 == 0)
      ms_fast_kernel<2><<<grid, kMsWarps * 32, 0, s>>>(in, out, H, W, umax, vcount, work, q);
    else
      ms_fast_kernel<1><<<grid, kMsWarps * 32, 0, s>>>(in, out, H, W, umax, vcount, work, q);
    return cudaGetLastError();
  }
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
    case 1: ms_stage2_kernel<1><<<grid, kThreads, 0, s>>>(in, out, H, W, umax, vcount, p); break;
    case 2: ms_stage2_kernel<2><<<grid, kThreads, 0, s>>>(in, out, H, W, umax, vcount, p); break;
    case 3: ms_stage2_kernel<3><<<grid, kThreads, 0, s>>>(in, out, H, W, umax, vcount, p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace dfc
