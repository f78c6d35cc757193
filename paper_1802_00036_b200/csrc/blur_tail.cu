// Blur tail: stage 7 + stage 8 of the pipeline in one tiled kernel.
//
//   [median KxK] -> [Gaussian | bilateral KxK] -> [partial re-impose] -> invert back
//
// (pipeline._blur_stage, pipeline.py:206-238; morphology.py:99-125;
// depth_core.invert_back :150-156.)  Input: the stage-6 (FULL) or stage-4
// (PARTIAL) map in the inverted encoding; output: the final direct-depth map.
// One CTA per output tile (64 x 64 minus the blur halo): the input tile (+
// median and blur halos, replicate-clamped) is staged in shared memory, the
// median is computed on the tile plus the blur halo -- each halo position
// outside the frame at its frame-clamped centre, which is exactly the
// replicate border the reference's blur sees -- then the blur, re-impose and
// re-inversion run two pixels per thread.  The 5x5 median uses one shared
// min/max network per 8x2 block of outputs (median_block.cuh, ~64 min/max per
// output instead of ~200 for a separate median-of-25 network).
//
// The median is exact (selection network, bit-identical to the reference's
// median_network).  The Gaussian is fp32 centre-relative c + sum w_i w_j (q - c) and the
// bilateral fp32 centre-relative c + sum w (q - c) / sum w with ex2.approx; both are
// within the 1e-4 m bar of the float64 reference (tests/test_gpu_pipeline.py).
// The exact float64 blurs (DFC_F_EXACT_BLUR) stay on the staged op kernels.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>

#include "dfc_common.cuh"
#include "median_block.cuh"
#include "median_networks.cuh"

namespace dfc {
namespace {

// The median region (output tile + blur halo) is kMW x kMH = 64 x 64: 256
// blocks of 8 x 2 medians, one per thread.  Output tile = region - 2 PR.
constexpr int kMW = 64, kMH = 64, kThreads = 256;
static_assert((kMW / kMedBlockW) * (kMH / kMedBlockH) == kThreads, "one median block per thread");
constexpr int kPostNone = 0, kPostGauss = 1, kPostBilateral = 2;
constexpr unsigned kFullMask = 0xffffffffu;
#ifndef DFC_TAIL_MINB
#define DFC_TAIL_MINB 3  // resident CTAs per SM the register allocation targets (<= 80 registers)
#endif

struct TailParams {
  float md;
  float w2[25];  // Gaussian 2-D taps w_i * w_j (row-major, radius PR)
  float ks[25];  // bilateral: log2(e) * spatial exponent per tap (dy^2 + dx^2) / (-2 sigma_s^2)
  float kv;      // bilateral: log2(e) / (-2 sigma_v^2)
  float bsc, bisc;  // bilateral: sqrt(-kv) and its inverse (bilateral5_sym prescales the values)
  unsigned* vcount;  // [B][2] (may be null): [1] += valid outputs (RunStats.output_density)
};

#define DFC_CSWAP(a, b)            \
  do {                             \
    const float lo_ = fminf(a, b); \
    const float hi_ = fmaxf(a, b); \
    a = lo_;                       \
    b = hi_;                       \
  } while (0)

// exact median of 5: med3(c, max(min(a, b), min(d, e)), min(max(a, b), max(d, e)))
__device__ __forceinline__ float med5(float a, float b, float c, float d, float e) {
  const float f = fmaxf(fminf(a, b), fminf(d, e)), g = fminf(fmaxf(a, b), fmaxf(d, e));
  return fmaxf(fminf(c, f), fminf(fmaxf(c, f), g));
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MR>
__device__ __forceinline__ float median_at(const float* __restrict__ t, int stride) {
  // t points at the window's top-left element
  constexpr int S = 2 * MR + 1;
  float v[S * S];
#pragma unroll
  for (int dy = 0; dy < S; ++dy)
#pragma unroll
    for (int dx = 0; dx < S; ++dx) v[dy * S + dx] = t[dy * stride + dx];
  if constexpr (S == 3) {
    DFC_MEDNET9_APPLY(v);
  } else {
    DFC_MEDNET25_APPLY(v);
  }
  return v[(S * S) / 2];
}

// OUT16: the output is 16-bit KITTI raw, rint(depth * 256) clipped (kitti_io.py:62-65)
__device__ __forceinline__ unsigned enc_raw16(float v) {
  return (unsigned)fminf(fmaxf(rintf(v * 256.0f), 0.0f), 65535.0f);
}

// Tile geometry per (median radius MR, blur radius PR).
template <int MR, int PR>
struct TileGeo {
  static constexpr int HI = MR + PR;  // input halo
  static constexpr int TX = kMW - 2 * PR, TY = kMH - 2 * PR;
  static constexpr int IW = TX + 2 * HI, IH = TY + 2 * HI;
  // shared row stride: odd, so the 8x2 median blocks of a warp (bases 8 bx +
  // 2 IWS by) fall on 16 distinct banks instead of 4 (2-way, not 8-way,
  // conflicts; config 2: 110k -> 114.5k frames/s)
  static constexpr int IWS = MR > 0 ? (IW | 1) : IW;  // MR = 0: 8-byte aligned rows (bilateral5_sym reads sIn)
  // Double-buffered persistent CTAs with the median or the 5x5 bilateral (long
  // ALU phases, few resident CTAs: the next tile's staging hides behind them);
  // otherwise one tile per CTA and more resident CTAs hide the loads better.
  static constexpr bool kDB = MR > 0;
  static constexpr size_t kSmem = (size_t)(2 * IH * IWS + kMW * kMH) * sizeof(float);
};

__device__ __forceinline__ void cp_async4(uint32_t sdst, const float* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sdst), "l"(g) : "memory");
}

// Stage tile t's input (+ halos, replicate-clamped) into sIn with 4-byte
// cp.async: the copies of the next tile fly while this one is computed.
template <int MR, int PR>
__device__ __forceinline__ void stage_tile(const float* __restrict__ in, int H, int W, int tx, int ty, int64_t t,
                                           float* sIn) {
  using G = TileGeo<MR, PR>;
  const unsigned per = (unsigned)(tx * ty), tu = (unsigned)t;  // tiles < 2^31 (launch_t chunks the batch)
  const unsigned b = tu / per, r = tu - b * per, byi = r / (unsigned)tx, bxi = r - byi * (unsigned)tx;
  const int x0 = (int)bxi * G::TX, y0 = (int)byi * G::TY;
  const float* src = in + b * (int64_t)H * W;
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sIn);
  if (x0 - G::HI >= 0 && y0 - G::HI >= 0 && x0 - G::HI + G::IW <= W && y0 - G::HI + G::IH <= H) {
    // interior tile: no clamping; each thread's (row, column) advances by a
    // fixed step, so the addresses are updated incrementally
    constexpr int DY = kThreads / G::IW, DX = kThreads % G::IW;
    int iy = threadIdx.x / G::IW, ix = threadIdx.x - iy * G::IW;
    const float* g = src + (int64_t)(y0 - G::HI + iy) * W + (x0 - G::HI + ix);
    uint32_t d = s0 + 4 * (iy * G::IWS + ix);
    const int64_t stepA = (int64_t)DY * W + DX, stepB = W - G::IW;
    for (int i = threadIdx.x; i < G::IH * G::IW; i += kThreads) {
      cp_async4(d, g);
      ix += DX;
      g += stepA;
      d += 4 * (DY * G::IWS + DX);
      if (ix >= G::IW) {
        ix -= G::IW;
        g += stepB;
        d += 4 * (G::IWS - G::IW);
      }
    }
    return;
  }
  for (int i = threadIdx.x; i < G::IH * G::IW; i += kThreads) {
    const int iy = i / G::IW, ix = i - iy * G::IW;
    const float* g = src + (int64_t)clampi(y0 - G::HI + iy, H) * W + clampi(x0 - G::HI + ix, W);
    cp_async4(s0 + 4 * (iy * G::IWS + ix), g);
  }
}

// Stage 7c (re-impose) + stage 8 for one output pair and its store:
// PARTIAL keeps the pre-blur validity (pipeline.py:212-214), then invert back
// (depth_core.py:150-156).
template <bool PARTIAL, bool OUT16, bool BLUR>
__device__ __forceinline__ void finish_pair(float2 r, float2 c, void* __restrict__ out_v, int64_t off, int gx, int W,
                                            const TailParams& p, bool& over, unsigned& nvalid) {
  float o[2] = {r.x, r.y};
  const float cc[2] = {c.x, c.y};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (PARTIAL && BLUR && !(cc[h] > kValid)) o[h] = 0.0f;
    o[h] = o[h] > kValid ? p.md - o[h] : 0.0f;
  }
  nvalid += (o[0] > kValid) + (gx + 1 < W && o[1] > kValid);
  if constexpr (OUT16) {
    uint16_t* q = static_cast<uint16_t*>(out_v) + off;
    over |= o[0] >= 256.0f || (gx + 1 < W && o[1] >= 256.0f);
    if (gx + 1 < W && (reinterpret_cast<uintptr_t>(q) & 3) == 0)
      __stcs(reinterpret_cast<unsigned*>(q), enc_raw16(o[0]) | enc_raw16(o[1]) << 16);
    else {
      q[0] = (uint16_t)enc_raw16(o[0]);
      if (gx + 1 < W) q[1] = (uint16_t)enc_raw16(o[1]);
    }
  } else {
    float* q = static_cast<float*>(out_v) + off;
    if (gx + 1 < W) {
      if ((reinterpret_cast<uintptr_t>(q) & 7) == 0)
        __stcs(reinterpret_cast<float2*>(q), make_float2(o[0], o[1]));
      else
        __stcs(q, o[0]), __stcs(q + 1, o[1]);
    } else {
      __stcs(q, o[0]);
    }
  }
}

// 5x5 bilateral (morphology.py:115-125, _numpy_ops.py:76-95) with the weights
// shared between the two pixels of every pair: w(p, p+d) = ex2(ks(d) - (sc
// (v(p+d) - v(p)))^2) is symmetric (ks(-d) = ks(d); float a - b = -(b - a)
// exactly, so both directions round identically), so each pixel evaluates the
// 12 forward offsets d (dy > 0, or dy = 0 and dx > 0) only: 12 ex2 per output
// instead of 24 (the MUFU pipe bounded this kernel).  Each weight adds w (q - p)
// to p's sums and is pushed, as -w (q - p), to the pixel q = p + d: into the
// pending sums of the row dy below (registers), through a shuffle when q lies
// in the neighbour lane.  Warp w sweeps a band of 8 output rows top-down over
// the whole 64-column region (lane l holds sM columns 2l, 2l+1 = output columns
// 2l-2, 2l-1; lanes 1..30 own outputs, lanes 0 / 31 evaluate the weights
// their neighbours take), starting with two warm-up rows that push only.
// Values are prescaled by sc = sqrt(-kv) (kv = log2(e) / (-2 sigma_v^2)), so
// the exponent is one FFMA2: ks - d'^2 with d' = sc d (prescaled differences
// round differently from d: ~1e-6 m at most in the output, the bar is 1e-4).
// fp32 centre-relative: out = c + sum w d / (1 + sum w).
template <bool PARTIAL, bool OUT16, int MW, bool CST>
__device__ __forceinline__ void bilateral5_sym(const float* __restrict__ sM, void* __restrict__ out_v, int H, int W,
                                               const TailParams& p, int64_t b, int x0, int y0, bool& over,
                                               unsigned& nvalid) {
  constexpr int TY = kMH - 4, NW = kThreads / 32;
  constexpr int kBand = (TY + NW - 1) / NW;  // 8 output rows per warp (bands overlap by <= 1 row)
  static_assert(MW % 2 == 0, "float2 rows");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // every warp sweeps exactly kBand rows (straight-line code: the shuffles need
  // no reconvergence); it stores only the rows below the next band's start
  const int ra = warp * (TY - kBand) / (NW - 1), rb = warp == NW - 1 ? TY : (warp + 1) * (TY - kBand) / (NW - 1);
  const int X0 = 2 * lane;
  // the first / last lane's outer columns are never used: clamp their loads into the region
  const int cA = max(X0 - 2, 0), cC = min(X0 + 2, kMW - 2);
  const float2 sc = make_float2(p.bsc, p.bsc);
  const int gx = x0 + X0 - 2;       // output column of the pair
  const bool Weven = (W & 1) == 0;  // gx is even: float2 stores are aligned
  const int64_t obase = b * (int64_t)H * W + (int64_t)y0 * W + gx;
  float* const fbase = static_cast<float*>(out_v) + b * (int64_t)H * W;
  int ooff = (y0 + ra) * W + gx;  // 32-bit in-frame offset of the output pair of sweep step i >= 2 (H W < 2^31)
  // V[r][k]: prescaled sM row s + r, column X0 - 2 + k; C[r]: the unscaled centre pair of that row
  float V[3][6];
  float2 C[3];
  auto load_row = [&](int s, float* v, float2& c) {
    const float* r = sM + s * MW;
    const float2 a = *reinterpret_cast<const float2*>(r + cA);
    const float2 m = *reinterpret_cast<const float2*>(r + X0);
    const float2 e = *reinterpret_cast<const float2*>(r + cC);
    c = m;
    const float2 a2 = __fmul2_rn(a, sc), m2 = __fmul2_rn(m, sc), e2 = __fmul2_rn(e, sc);
    v[0] = a2.x, v[1] = a2.y, v[2] = m2.x, v[3] = m2.y, v[4] = e2.x, v[5] = e2.y;
  };
  // pending (acc, den) pushed to rows s, s + 1, s + 2
  float2 Qa[3], Qd[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) Qa[k] = Qd[k] = make_float2(0.f, 0.f);
#pragma unroll
  for (int r = 0; r < 3; ++r) load_row(ra + r, V[r], C[r]);
  float2 last_r = make_float2(0.f, 0.f);  // the band's first output pair (replicated by the constant path)
  auto step = [&](const int i) {
    const int s = ra + i;  // sM row (output row s - 2)
    if (i > 0) {
#pragma unroll
      for (int k = 0; k < 6; ++k) V[0][k] = V[1][k], V[1][k] = V[2][k];
      C[0] = C[1], C[1] = C[2];
      load_row(s + 2, V[2], C[2]);
    }
    const bool outrow = i >= 2;
    float2 Fa = make_float2(0.f, 0.f), Fd = make_float2(0.f, 0.f);  // forward sums of this row's pixels
    const float2 c2 = make_float2(V[0][2], V[0][3]);
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
      // warm-up rows push only what reaches the band: row ra - 2 (i = 0) the dy = 2
      // offsets, row ra - 1 (i = 1) dy >= 1; dy = 0 only on output rows
      if ((i == 0 && dy < 2) || (i == 1 && dy < 1)) continue;
      float2 La = make_float2(0.f, 0.f), Ld = La, Ra = La, Rd = La;  // pushes to the left / right lane
      bool hasL = false;
#pragma unroll
      for (int dx = -2; dx <= 2; ++dx) {
        if (dy == 0 && dx <= 0) continue;
        const float ks = p.ks[(dy + 2) * 5 + dx + 2];
        const float2 n = make_float2(V[dy][2 + dx], V[dy][3 + dx]);
        const float2 d = __fadd2_rn(n, make_float2(-c2.x, -c2.y));
        const float2 e = __ffma2_rn(make_float2(-d.x, -d.y), d, make_float2(ks, ks));  // exponents <= 0
        const float2 w = make_float2(ex2_ftz(e.x), ex2_ftz(e.y));
        const float2 wd = __fmul2_rn(w, d);
        if (outrow) {
          Fa = __fadd2_rn(Fa, wd);
          Fd = __fadd2_rn(Fd, w);
        }
        // push -w d and w to q = p + (dy, dx): lane offset / component by (comp + dx)
        if (dx == 0) {
          Qa[dy] = __fadd2_rn(Qa[dy], make_float2(-wd.x, -wd.y));
          Qd[dy] = __fadd2_rn(Qd[dy], w);
        } else if (dx == -2) {
          La = make_float2(-wd.x, -wd.y), Ld = w, hasL = true;
        } else if (dx == 2) {
          Ra = __fadd2_rn(Ra, make_float2(-wd.x, -wd.y));
          Rd = __fadd2_rn(Rd, w);
        } else if (dx == -1) {  // x -> left lane's y; y -> own x
          La.y -= wd.x, Ld.y += w.x;
          Qa[dy].x -= wd.y, Qd[dy].x += w.y;
          hasL = true;
        } else {  // dx == 1: x -> own y; y -> right lane's x
          Qa[dy].y -= wd.x, Qd[dy].y += w.x;
          Ra.x -= wd.y, Rd.x += w.y;
        }
      }
      // receive: the right lane's left pushes and the left lane's right pushes
      if (hasL) {
        const float2 ra_ = make_float2(__shfl_down_sync(kFullMask, La.x, 1), __shfl_down_sync(kFullMask, La.y, 1));
        const float2 rd_ = make_float2(__shfl_down_sync(kFullMask, Ld.x, 1), __shfl_down_sync(kFullMask, Ld.y, 1));
        Qa[dy] = __fadd2_rn(Qa[dy], ra_);
        Qd[dy] = __fadd2_rn(Qd[dy], rd_);
      }
      {
        const float2 ra_ = make_float2(__shfl_up_sync(kFullMask, Ra.x, 1), __shfl_up_sync(kFullMask, Ra.y, 1));
        const float2 rd_ = make_float2(__shfl_up_sync(kFullMask, Rd.x, 1), __shfl_up_sync(kFullMask, Rd.y, 1));
        Qa[dy] = __fadd2_rn(Qa[dy], ra_);
        Qd[dy] = __fadd2_rn(Qd[dy], rd_);
      }
    }
    if (outrow) {
      const float2 acc = __fadd2_rn(Qa[0], Fa);
      const float2 den = __fadd2_rn(__fadd2_rn(Qd[0], Fd), make_float2(1.f, 1.f));  // centre tap: weight 1
      // den >= 1: rcp.approx.ftz needs no denormal handling; acc is in prescaled units
      const float2 q = __fmul2_rn(make_float2(rcp_approx(den.x), rcp_approx(den.y)), make_float2(p.bisc, p.bisc));
      const float2 c = C[0];
      const float2 r = __ffma2_rn(acc, q, c);
      last_r = r;
      const int oy = s - 2;
      if (lane != 0 && lane != 31 && oy < rb && y0 + oy < H && gx < W) {
        if (!OUT16 && Weven && gx + 1 < W) {
          // the common case: [re-impose,] invert back and one aligned 8-byte store
          float o0 = r.x > kValid ? p.md - r.x : 0.0f, o1 = r.y > kValid ? p.md - r.y : 0.0f;
          if (PARTIAL && !(c.x > kValid)) o0 = 0.0f;
          if (PARTIAL && !(c.y > kValid)) o1 = 0.0f;
          nvalid += (o0 > kValid) + (o1 > kValid);
          __stcs(reinterpret_cast<float2*>(fbase + ooff), make_float2(o0, o1));
        } else {
          finish_pair<PARTIAL, OUT16, true>(r, c, out_v, obase + (int64_t)oy * W, gx, W, p, over, nvalid);
        }
      }
      ooff += W;
    }
    Qa[0] = Qa[1], Qd[0] = Qd[1];
    Qa[1] = Qa[2], Qd[1] = Qd[2];
    Qa[2] = Qd[2] = make_float2(0.f, 0.f);
  };
  // A band whose input rows (sM rows ra .. ra + kBand + 3) are vertically
  // constant in every column -- the rows above every column's first valid row,
  // which extend_to_top made equal (morphology.py:81-96), or all-empty rows --
  // has equal output rows: sweep to the first one and store it kBand times.
  // (CST: without the median; after it, the check's registers cost the
  // median network more than the shortcut saves, config 2 measured.)
  bool cst = CST;
  if (CST) {
    const float* r0 = sM + ra * MW;
    const float2 a0 = *reinterpret_cast<const float2*>(r0 + cA), m0 = *reinterpret_cast<const float2*>(r0 + X0),
                 e0 = *reinterpret_cast<const float2*>(r0 + cC);
#pragma unroll
    for (int r = 1; r < kBand + 4; ++r) {
      const float* rr = r0 + r * MW;
      const float2 a1 = *reinterpret_cast<const float2*>(rr + cA), m1 = *reinterpret_cast<const float2*>(rr + X0),
                   e1 = *reinterpret_cast<const float2*>(rr + cC);
      cst &= __float_as_uint(a1.x) == __float_as_uint(a0.x) && __float_as_uint(a1.y) == __float_as_uint(a0.y) &&
             __float_as_uint(m1.x) == __float_as_uint(m0.x) && __float_as_uint(m1.y) == __float_as_uint(m0.y) &&
             __float_as_uint(e1.x) == __float_as_uint(e0.x) && __float_as_uint(e1.y) == __float_as_uint(e0.y);
    }
  }
  if (CST && __all_sync(kFullMask, cst)) {
#pragma unroll
    for (int i = 0; i < 3; ++i) step(i);
    const float2 c = C[0];  // = the centre pair of every row
    for (int oy = ra + 1; oy < rb && y0 + oy < H; ++oy) {
      if (lane != 0 && lane != 31 && gx < W)
        finish_pair<PARTIAL, OUT16, true>(last_r, c, out_v, obase + (int64_t)oy * W, gx, W, p, over, nvalid);
    }
  } else {
#pragma unroll
    for (int i = 0; i < kBand + 2; ++i) step(i);
  }
}

// One output tile from its staged input: median -> blur -> re-impose -> invert back -> store.
template <int MR, int POST, int PR, bool PARTIAL, bool OUT16>
__device__ __forceinline__ void tile_process(const float* __restrict__ sIn, float* __restrict__ sM,
                                             void* __restrict__ out_v, int H, int W, uint32_t* __restrict__ status,
                                             const TailParams& p, int64_t b, int x0, int y0) {
  using G = TileGeo<MR, PR>;
  constexpr int HI = G::HI, kTX = G::TX, kTY = G::TY, IWS = G::IWS;
  constexpr int MW = kMW, MH = kMH;
  bool over = false;  // OUT16: an output >= 256 m
  unsigned nvalid = 0;

  if constexpr (MR == 0 && POST == kPostBilateral && PR == 2) {
    // no median: the staged tile (frame-clamped positions = replicate border)
    // is the blur input as it is
    bilateral5_sym<PARTIAL, OUT16, IWS, true>(sIn, out_v, H, W, p, b, x0, y0, over, nvalid);
    if (OUT16 && over) atomicOr(status + b, DFC_ST_ENCODE);
    if (p.vcount) {
      nvalid = __reduce_add_sync(0xffffffffu, nvalid);
      if ((threadIdx.x & 31) == 0 && nvalid) atomicAdd(p.vcount + 2 * b + 1, nvalid);
    }
    return;
  }
  // stage-7a: median (or copy) on the tile + blur halo, at frame-clamped centres
  if constexpr (MR == 2) {
    // shared 8x2-block network on the regular grid; positions outside the
    // frame then take the value at their clamped position
    const int bx = threadIdx.x % (MW / kMedBlockW), by = threadIdx.x / (MW / kMedBlockW);
    const int mx = bx * kMedBlockW, my = by * kMedBlockH;
    float med[kMedBlockH][kMedBlockW];
    // The warp's blocks cover median rows 8w .. 8w + 7 of the region; when their
    // input window (rows 8w .. 8w + 11, all 68 columns) is vertically constant
    // in every column -- the rows above every column's first valid row, which
    // extend_to_top made equal (morphology.py:81-96), or empty rows -- each
    // 5x5 median is the median of its 5 column values (each counted 5 times):
    // 9 min/max per output instead of ~60.  Each lane checks two columns.
    bool cst = true;
    {
      const float* t = sIn + (threadIdx.x >> 5) * (4 * kMedBlockH) * IWS;
      const int l = threadIdx.x & 31, ca = 2 * l, cb = 2 * l + 1, cc = min(64 + l, 67);
      const unsigned b0 = __float_as_uint(t[ca]), b1 = __float_as_uint(t[cb]), b2 = __float_as_uint(t[cc]);
#pragma unroll
      for (int r = 1; r < 4 * kMedBlockH + 4; ++r)
        cst &= __float_as_uint(t[r * IWS + ca]) == b0 && __float_as_uint(t[r * IWS + cb]) == b1 &&
               __float_as_uint(t[r * IWS + cc]) == b2;
    }
    if (__all_sync(0xffffffffu, cst)) {
      const float* t = sIn + my * IWS + mx;
#pragma unroll
      for (int c = 0; c < kMedBlockW; ++c) {
        const float m = med5(t[c], t[c + 1], t[c + 2], t[c + 3], t[c + 4]);
#pragma unroll
        for (int j = 0; j < kMedBlockH; ++j) med[j][c] = m;
      }
    } else {
      median5_block(sIn + my * IWS + mx, IWS, med);
    }
#pragma unroll
    for (int j = 0; j < kMedBlockH; ++j) {
#pragma unroll
      for (int c = 0; c < kMedBlockW; ++c)
        if (PARTIAL && !(sIn[(my + j + MR) * IWS + mx + c + MR] > kValid)) med[j][c] = 0.0f;
      // 16-byte stores (the block's row is 32-byte aligned): 4x fewer shared wavefronts than scalar stores
#pragma unroll
      for (int c = 0; c < kMedBlockW; c += 4)
        *reinterpret_cast<float4*>(sM + (my + j) * MW + mx + c) =
            make_float4(med[j][c], med[j][c + 1], med[j][c + 2], med[j][c + 3]);
    }
    if (x0 - PR < 0 || y0 - PR < 0 || x0 - PR + MW > W || y0 - PR + MH > H) {  // tile at a frame edge
      __syncthreads();
      for (int i = threadIdx.x; i < MH * MW; i += kThreads) {
        const int py = i / MW, px = i - py * MW;
        const int cy = clampi(y0 - PR + py, H) - y0 + PR, cx = clampi(x0 - PR + px, W) - x0 + PR;
        const float v = sM[cy * MW + cx];  // an in-frame position: never rewritten here
        if (cy != py || cx != px) sM[i] = v;
      }
    }
  } else
  for (int i = threadIdx.x; i < MH * MW; i += kThreads) {
    const int my = i / MW, mx = i - my * MW;
    const int cy = clampi(y0 - PR + my, H) - y0 + HI;  // centre in sIn coordinates
    const int cx = clampi(x0 - PR + mx, W) - x0 + HI;
    const float c = sIn[cy * IWS + cx];
    float v = c;
    if constexpr (MR > 0) {
      v = median_at<MR>(sIn + (cy - MR) * IWS + (cx - MR), IWS);
      if (PARTIAL && !(c > kValid)) v = 0.0f;
    }
    sM[i] = v;
  }
  __syncthreads();

  // stage-7b: Gaussian / bilateral, re-impose, invert back -- two horizontally
  // adjacent outputs per thread in packed fp32x2 (FADD2 / FMUL2 / FFMA2)
  if constexpr (POST == kPostBilateral && PR == 2) {
    bilateral5_sym<PARTIAL, OUT16, MW, false>(sM, out_v, H, W, p, b, x0, y0, over, nvalid);
  } else
  for (int i = threadIdx.x; i < kTX * kTY / 2; i += kThreads) {
    const int oy = i / (kTX / 2), ox = 2 * (i - oy * (kTX / 2));
    const int gy = y0 + oy, gx = x0 + ox;
    if (gy >= H || gx >= W) continue;
    const float* m = sM + oy * MW + ox;  // window top-left of the first output (radius PR)
    // the pair's window rows: columns ox .. ox + 2 PR + 1 as PR + 1 aligned
    // 8-byte loads per row (ox even), taps then come from registers
    float seg[2 * PR + 1][2 * PR + 2];
#pragma unroll
    for (int dy = 0; dy <= 2 * PR; ++dy)
#pragma unroll
      for (int q = 0; q <= PR; ++q) {
        const float2 v = *reinterpret_cast<const float2*>(m + dy * MW + 2 * q);
        seg[dy][2 * q] = v.x;
        seg[dy][2 * q + 1] = v.y;
      }
    const float2 c = make_float2(seg[PR][PR], seg[PR][PR + 1]);
    float2 r = c;
    if constexpr (POST == kPostGauss) {
      // centre-relative: constant neighbourhoods come out exactly constant
      float2 a = make_float2(0.f, 0.f);
#pragma unroll
      for (int dy = 0; dy <= 2 * PR; ++dy)
#pragma unroll
        for (int dx = 0; dx <= 2 * PR; ++dx) {
          const float2 d = __fadd2_rn(make_float2(seg[dy][dx], seg[dy][dx + 1]), make_float2(-c.x, -c.y));
          const float w = p.w2[dy * (2 * PR + 1) + dx];
          a = __ffma2_rn(make_float2(w, w), d, a);
        }
      r = __fadd2_rn(c, a);
    } else if constexpr (POST == kPostBilateral) {
      // the centre tap has d = 0 and weight exactly 1 (ex2(0))
      float2 acc = make_float2(0.f, 0.f), den = make_float2(1.f, 1.f);
#pragma unroll
      for (int dy = 0; dy <= 2 * PR; ++dy)
#pragma unroll
        for (int dx = 0; dx <= 2 * PR; ++dx) {
          if (dy == PR && dx == PR) continue;
          const float2 d = __fadd2_rn(make_float2(seg[dy][dx], seg[dy][dx + 1]), make_float2(-c.x, -c.y));
          const float ks = p.ks[dy * (2 * PR + 1) + dx];
          const float2 e = __ffma2_rn(__fmul2_rn(make_float2(p.kv, p.kv), d), d, make_float2(ks, ks));
          const float2 w = make_float2(ex2_ftz(e.x), ex2_ftz(e.y));  // exponents <= 0
          acc = __ffma2_rn(w, d, acc);
          den = __fadd2_rn(den, w);
        }
      r = make_float2(c.x + __fdividef(acc.x, den.x), c.y + __fdividef(acc.y, den.y));
    }
    finish_pair<PARTIAL, OUT16, POST != kPostNone>(r, c, out_v, b * (int64_t)H * W + (int64_t)gy * W + gx, gx, W, p,
                                                   over, nvalid);
  }
  if (OUT16 && over) atomicOr(status + b, DFC_ST_ENCODE);  // write_depth_png raises (kitti_io.py:60-61)
  if (p.vcount) {
    nvalid = __reduce_add_sync(0xffffffffu, nvalid);
    if ((threadIdx.x & 31) == 0 && nvalid) atomicAdd(p.vcount + 2 * b + 1, nvalid);
  }
}

// With the median: persistent CTAs walk the tiles (frame-major) with two
// input buffers: tile t + grid is staged with cp.async while tile t is
// computed, so the latency-bound staging overlaps the ALU-bound median / blur
// (configs 2 / 4: +4 %).
template <int MR, int POST, int PR, bool PARTIAL, bool OUT16>
__global__ void __launch_bounds__(kThreads, DFC_TAIL_MINB) blur_tail_kernel(const float* __restrict__ in, void* __restrict__ out_v,
                                                             int H, int W, uint32_t* __restrict__ status,
                                                             const __grid_constant__ TailParams p, int tx, int ty,
                                                             int64_t ntiles) {
  using G = TileGeo<MR, PR>;
  extern __shared__ __align__(16) float smem[];
  float* const sIn0 = smem;
  float* const sIn1 = smem + G::IH * G::IWS;
  float* sM = smem + 2 * G::IH * G::IWS;
  int64_t t = blockIdx.x;
  if (t < ntiles) stage_tile<MR, PR>(in, H, W, tx, ty, t, sIn0);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  int cur = 0;
  for (; t < ntiles; t += gridDim.x) {
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) stage_tile<MR, PR>(in, H, W, tx, ty, tn, cur ? sIn0 : sIn1);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // tile t's copies (this thread's)
    __syncthreads();                                          // ... and everyone's
    const unsigned per = (unsigned)(tx * ty), tu = (unsigned)t;
    const unsigned b = tu / per, r = tu - b * per, byi = r / (unsigned)tx, bxi = r - byi * (unsigned)tx;
    tile_process<MR, POST, PR, PARTIAL, OUT16>(cur ? sIn1 : sIn0, sM, out_v, H, W, status, p, (int64_t)b, (int)bxi * G::TX,
                                               (int)byi * G::TY);
    __syncthreads();  // this tile's input buffer and sM are reused
    cur ^= 1;
  }
}

// Without the median: one tile per CTA (plain loads; many resident CTAs hide them).
template <int MR, int POST, int PR, bool PARTIAL, bool OUT16>
__global__ void __launch_bounds__(kThreads, DFC_TAIL_MINB) blur_tail_tile_kernel(const float* __restrict__ in,
                                                                  void* __restrict__ out_v, int H, int W,
                                                                  uint32_t* __restrict__ status,
                                                                  const __grid_constant__ TailParams p) {
  using G = TileGeo<MR, PR>;
  __shared__ __align__(16) float sIn[G::IH * G::IWS];
  __shared__ __align__(16) float sM[kMH * kMW];
  const int64_t b = blockIdx.z;
  const int x0 = blockIdx.x * G::TX, y0 = blockIdx.y * G::TY;
  const float* src = in + b * (int64_t)H * W;
  for (int i = threadIdx.x; i < G::IH * G::IW; i += kThreads) {
    const int iy = i / G::IW, ix = i - iy * G::IW;
    sIn[iy * G::IWS + ix] = __ldg(src + (int64_t)clampi(y0 - G::HI + iy, H) * W + clampi(x0 - G::HI + ix, W));
  }
  __syncthreads();
  tile_process<MR, POST, PR, PARTIAL, OUT16>(sIn, sM, out_v, H, W, status, p, b, x0, y0);
}

template <int MR, int POST, int PR>
cudaError_t launch_t(const float* in, void* out, int64_t B, int H, int W, bool partial, bool out16, uint32_t* status,
                     const TailParams& p, cudaStream_t s) {
  using G = TileGeo<MR, PR>;
  const int tx = (W + G::TX - 1) / G::TX, ty = (H + G::TY - 1) / G::TY;
  if constexpr (!(G::kDB || (POST == kPostBilateral && PR == 2))) {
    // grid.z holds at most 65535 frames: chunk the batch
    const int64_t HW = (int64_t)H * W;
    for (int64_t f0 = 0; f0 < B; f0 += 65535) {
      const int64_t C = std::min<int64_t>(65535, B - f0);
      const dim3 grid(tx, ty, (unsigned)C);
      const float* ic = in + f0 * HW;
      void* oc = static_cast<char*>(out) + f0 * HW * (out16 ? 2 : 4);
      uint32_t* sc = status ? status + f0 : nullptr;
      TailParams pc = p;
      if (pc.vcount) pc.vcount += 2 * f0;
      note_launch();
      if (partial)
        out16 ? blur_tail_tile_kernel<MR, POST, PR, true, true><<<grid, kThreads, 0, s>>>(ic, oc, H, W, sc, pc)
              : blur_tail_tile_kernel<MR, POST, PR, true, false><<<grid, kThreads, 0, s>>>(ic, oc, H, W, sc, pc);
      else
        out16 ? blur_tail_tile_kernel<MR, POST, PR, false, true><<<grid, kThreads, 0, s>>>(ic, oc, H, W, sc, pc)
              : blur_tail_tile_kernel<MR, POST, PR, false, false><<<grid, kThreads, 0, s>>>(ic, oc, H, W, sc, pc);
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  auto k = partial ? (out16 ? blur_tail_kernel<MR, POST, PR, true, true> : blur_tail_kernel<MR, POST, PR, true, false>)
                   : (out16 ? blur_tail_kernel<MR, POST, PR, false, true> : blur_tail_kernel<MR, POST, PR, false, false>);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::kSmem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kThreads, G::kSmem);
  if (e != cudaSuccess) return e;
  // the kernel indexes tiles in 32 bits: chunk the batch below 2^31 tiles per launch
  const int64_t HW = (int64_t)H * W, fmax = std::max<int64_t>(1, ((int64_t)1 << 31) / ((int64_t)tx * ty) - 1);
  for (int64_t f0 = 0; f0 < B; f0 += fmax) {
    const int64_t C = std::min<int64_t>(fmax, B - f0), nt = (int64_t)tx * ty * C;
    TailParams pc = p;
    if (pc.vcount) pc.vcount += 2 * f0;
    const int64_t grid = std::min<int64_t>(nt, (int64_t)std::max(per, 1) * sms);
    note_launch();
    k<<<(unsigned)grid, kThreads, G::kSmem, s>>>(in + f0 * HW, static_cast<char*>(out) + f0 * HW * (out16 ? 2 : 4), H,
                                                 W, status ? status + f0 : nullptr, pc, tx, ty, nt);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

bool blur_tail_supported(const dfc_config& c) {
  if (c.flags & DFC_F_EXACT_BLUR) return false;
  const int bm = c.blur_mode;
  const bool med = bm == DFC_BLUR_MEDIAN || bm == DFC_BLUR_MEDIAN_BILATERAL || bm == DFC_BLUR_MEDIAN_GAUSSIAN;
  const bool gauss = bm == DFC_BLUR_GAUSSIAN || bm == DFC_BLUR_MEDIAN_GAUSSIAN;
  const bool bil = bm == DFC_BLUR_BILATERAL || bm == DFC_BLUR_MEDIAN_BILATERAL;
  if (med && c.median_size != 3 && c.median_size != 5) return false;
  if (gauss && c.gaussian_size != 3 && c.gaussian_size != 5) return false;
  if (bil && c.bilateral_size != 3 && c.bilateral_size != 5) return false;
  return true;
}

// Blur stage + invert back for B frames (in: inverted map; out: direct depth).
cudaError_t launch_blur_tail(const float* in, void* out, int64_t B, int H, int W, const dfc_config& c, bool out_raw,
                             uint32_t* status, unsigned* vcount, cudaStream_t s) {
  const int bm = c.blur_mode;
  const bool med = bm == DFC_BLUR_MEDIAN || bm == DFC_BLUR_MEDIAN_BILATERAL || bm == DFC_BLUR_MEDIAN_GAUSSIAN;
  const bool gauss = bm == DFC_BLUR_GAUSSIAN || bm == DFC_BLUR_MEDIAN_GAUSSIAN;
  const bool bil = bm == DFC_BLUR_BILATERAL || bm == DFC_BLUR_MEDIAN_BILATERAL;
  const bool partial = c.fill_mode == DFC_FILL_PARTIAL;
  TailParams p{};
  p.md = c.max_depth;
  p.vcount = vcount;
  int pr = 0;
  if (gauss) {
    pr = c.gaussian_size / 2;
    const int k = c.gaussian_size;
    double w[5], sum = 0;
    for (int i = -pr; i <= pr; ++i) w[i + pr] = std::exp(-(double)(i * i) / (2.0 * c.gaussian_sigma * c.gaussian_sigma));
    for (int i = 0; i < k; ++i) sum += w[i];
    for (int i = 0; i < k; ++i) w[i] /= sum;
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) p.w2[i * k + j] = (float)(w[i] * w[j]);
  } else if (bil) {
    pr = c.bilateral_size / 2;
    const int k = c.bilateral_size;
    const double l2e = 1.4426950408889634;
    for (int dy = -pr; dy <= pr; ++dy)
      for (int dx = -pr; dx <= pr; ++dx)
        p.ks[(dy + pr) * k + dx + pr] =
            (float)(l2e * -(double)(dy * dy + dx * dx) / (2.0 * c.bilateral_sigma_space * c.bilateral_sigma_space));
    p.kv = (float)(l2e * -1.0 / (2.0 * c.bilateral_sigma_value * c.bilateral_sigma_value));
    p.bsc = (float)std::sqrt(l2e / (2.0 * c.bilateral_sigma_value * c.bilateral_sigma_value));
    p.bisc = (float)(1.0 / std::sqrt(l2e / (2.0 * c.bilateral_sigma_value * c.bilateral_sigma_value)));
  }
  const int mr = med ? c.median_size / 2 : 0;
  const int post = gauss ? kPostGauss : (bil ? kPostBilateral : kPostNone);
#define DFC_TAIL(MR, POST, PR) \
  if (mr == MR && post == POST && pr == PR) return launch_t<MR, POST, PR>(in, out, B, H, W, partial, out_raw, status, p, s);
  DFC_TAIL(0, kPostNone, 0)
  DFC_TAIL(1, kPostNone, 0)
  DFC_TAIL(2, kPostNone, 0)
  DFC_TAIL(0, kPostGauss, 1)
  DFC_TAIL(0, kPostGauss, 2)
  DFC_TAIL(1, kPostGauss, 1)
  DFC_TAIL(1, kPostGauss, 2)
  DFC_TAIL(2, kPostGauss, 1)
  DFC_TAIL(2, kPostGauss, 2)
  DFC_TAIL(0, kPostBilateral, 1)
  DFC_TAIL(0, kPostBilateral, 2)
  DFC_TAIL(1, kPostBilateral, 1)
  DFC_TAIL(1, kPostBilateral, 2)
  DFC_TAIL(2, kPostBilateral, 1)
  DFC_TAIL(2, kPostBilateral, 2)
#undef DFC_TAIL
  return cudaErrorInvalidValue;
}

}  // namespace dfc
