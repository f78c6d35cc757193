// Fused streaming depth-completion kernel for sm_100a (the hot path): the
// kernel templates.  fused_vec{1,2,4}.cu instantiate them per vector width
// (parallel compilation); fused.cu holds the host side.
//
// One persistent CTA works on one (frame, column strip) item at a time; a
// strip is the whole frame for W <= 1248.  Warps own ~104-column slices with
// 12-column lane halos (32 lanes x 4 columns = 128 columns per warp), so all
// horizontal neighbour traffic is warp shuffles and warps meet only at one
// CTA barrier per 4-row block.  Columns outside the frame (one lane at the
// left frame edge, >= 1 lane at the right edge) carry neutral values through
// the min/max stages and replicated values into the blur, which reproduces
// the reference's replicate border exactly.
//
// Phase 1 (FULL mode: extend_to_top needs each column's first valid row r0):
//   top-down over 32-row blocks, validity bit-packed in 64-bit column words.
//   The stage-4 validity equals the binary morphology D7(E5(D5(D_shape(M0))))
//   of the input mask (SURVEY.md App. B probe 13), so r0 needs bit ops only.
//   The scan stops once every owned column has its r0.
// Phase 2: bottom-up streaming in 4-row blocks (going up, a column's r0 row
//   comes before the rows above it, so extend_to_top needs no look-ahead).
//   Producer (registers + shuffles): invert -> cross3 -> cross3 (= 5x5
//   diamond) -> max5 -> min5 (close) -> masked max7 (small fill) -> extend.
//   Stage-5 rows go to a 40-row shared-memory ring; the consumer runs 16 rows
//   behind: 31x31 masked large fill (one warp-wide pass per empty pixel:
//   lanes take the 31 window columns, redux.max combines them; typical
//   frames hold ~50-200 such pixels), 5x5 Gaussian (fp32), invert back,
//   coalesced store.
//   Once the stage-5 rows are above every owned column's r0, stages 1-4 and
//   the input reads stop: those rows are the captured top values.
// Frames that still hold empties after one large-fill iteration are flagged
// for the staged path (capi.cu: dfc_fill_finish).
//
// Reference semantics: depth_core.py:150-156 (invert), morphology.py:39-96
// (dilate / close / masked fill / extend), pipeline.py:154-214 (stage order,
// fill loop, blur, partial re-impose).  Every selection stage is bit-exact by
// construction (min/max over clipped windows == replicate border); the
// Gaussian is fp32 (<= 1e-4 m against the fp64 reference; tested).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>
#include <cmath>
#include <vector>

#include "dfc_common.cuh"
#include "lane_ops.cuh"
#include "tmem.cuh"

namespace dfc {
namespace {

constexpr int kNW = 12;                // warps per CTA
constexpr int kLW = 128;               // columns per warp (32 lanes x 4)
constexpr int kHalo = 12;              // lane-halo columns per side (9 morphology + 2 blur, lane aligned)
constexpr int kRing = 40;              // stage-5 ring rows (39 live)
constexpr int kRingBlocks = kRing / kB;
constexpr int kLag = 16;               // consumer lag behind the stage-5 producer (>= 15)
// Row lags (processing order).  Stage 5 trails the input by 1+1+2+2+3 = 9
// rows (cross3, cross3, max5, min5, max7); with a precomputed stage-2 map
// (PRE: multiscale) by 2+2+3 = 7.  The consumer trails stage 5 by kLag; its
// first block is the one whose rows start in [-3, 0].
template <bool PRE>
struct Lags {
  static constexpr int L2 = PRE ? 0 : 2;  // stage-2 lag
  static constexpr int P = L2 + 7;        // stage-5 lag
  static constexpr int C = P + kLag;      // consumer rows = t0 - C + j
  static constexpr int KFirst = C / kB;
};
constexpr int kMbCount = 32;            // mbarrier arrivals per phase: every lane of the warp
constexpr int kLF = 15;                // large fill radius
constexpr int kStripMax = 1248;        // widest strip handled by one CTA
constexpr uint32_t kNeedsStaged = 0x200u;  // internal status bit (capi.cu)
constexpr uint32_t kRecountOut = 0x400u;   // internal: finalize_kernel recounts the frame's valid outputs
constexpr int kBlurRaw = -1;           // emit the stage-6 (FULL) / stage-4 (PARTIAL) inverted map for blur_tail.cu
constexpr int64_t kRawChunk = 296;     // frames per fused -> blur-tail round (2 per SM) in the raw mode

static_assert(kRing % kB == 0 && kLag % kB == 0, "ring blocks must not wrap inside a block");


// Element types at the boundary.  IO 0: float32 depth in / out; 1: KITTI
// 16-bit raw in (depth = raw / 256, kitti_io.py:53) / float32 out; 2: raw in /
// raw out (rint(depth * 256) clipped, kitti_io.py:62-65).
template <int IO>
struct IoT {
  using In = float;
  using Out = float;
};
template <>
struct IoT<1> {
  using In = uint16_t;
  using Out = float;
};
template <>
struct IoT<2> {
  using In = uint16_t;
  using Out = uint16_t;
};

struct Params {
  const void* in;
  void* out;
  int64_t nframes;
  int dense;  // shared-memory scratch for the dense large fill is available
  int regdense;  // DFC_F_SPARSE: use the register-dense large-fill instantiation
  int32_t* t0g;  // FULL: per-column r0 row (processing order) from r0_kernel, [nframes][W]
  int H, W, strips, SW, nw;
  float md;
  float gw[5];
  float2 gh[6];  // horizontal pass on column pairs: coefficients of e[i] for outputs (c, c+1)
  uint32_t* status;
  int32_t* iters;
  unsigned long long* nfallback;
#ifdef DFC_TIMING
  unsigned long long* tim;  // diagnostics build: per (CTA, warp) cycles [producer, barrier, consumer, phase 1]
#endif
  unsigned* work;
  unsigned* umax;
  unsigned* vcount;  // [nframes][2]: inverted-valid inputs read (non-PRE), valid outputs stored (non-raw)
};

// Stage one lane's 4 columns of an input row into shared memory with cp.async
// (zero-filled where the row or the columns lie outside the frame).
template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(uint32_t sdst, const void* gsrc, bool ok) {
  const int n = ok ? BYTES : 0;
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sdst), "l"(gsrc), "r"(n) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(sdst), "l"(gsrc), "n"(BYTES), "r"(n)
                 : "memory");
}

template <int VEC>
__device__ __forceinline__ void stage_lane(uint32_t sdst, const uint16_t* q, const void* safe, bool rowok, bool full,
                                           unsigned incol) {
  static_assert(VEC == 4, "16-bit input is staged 8 bytes per lane (W % 4 == 0)");
  const bool ok = rowok && full;
  cp_async_zfill<8>(sdst, ok ? (const void*)q : safe, ok);
}

template <int VEC>
__device__ __forceinline__ void stage_lane(uint32_t sdst, const float* q, const void* safe, bool rowok, bool full,
                                           unsigned incol) {
  if constexpr (VEC == 4) {
    const bool ok = rowok && full;
    cp_async_zfill<16>(sdst, ok ? (const void*)q : safe, ok);
  } else if constexpr (VEC == 2) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool ok = rowok && ((incol >> (2 * h)) & 3u) == 3u;
      cp_async_zfill<8>(sdst + 8 * h, ok ? (const void*)(q + 2 * h) : safe, ok);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const bool ok = rowok && (incol >> c & 1);
      cp_async_zfill<4>(sdst + 4 * c, ok ? (const void*)(q + c) : safe, ok);
    }
  }
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ F4 lds4(uint32_t saddr) {
  float4 q;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w) : "r"(saddr)
               : "memory");
  return F4{{q.x, q.y, q.z, q.w}};
}

// raw / 256 is exact in float32 for every 16-bit raw value (kitti_io.py:53)
__device__ __forceinline__ float raw_m(unsigned r) { return (float)r * 0.00390625f; }

__device__ __forceinline__ F4 unpack_raw(unsigned a, unsigned b) {
  return F4{{raw_m(a & 0xFFFFu), raw_m(a >> 16), raw_m(b & 0xFFFFu), raw_m(b >> 16)}};
}

template <typename T>
__device__ __forceinline__ F4 lds4_t(uint32_t saddr) {
  if constexpr (sizeof(T) == 4) {
    return lds4(saddr);
  } else {
    unsigned a, b;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n" : "=r"(a), "=r"(b) : "r"(saddr) : "memory");
    return unpack_raw(a, b);
  }
}

// rint(depth * 256) clipped to [0, 65535] (kitti_io.py:62-65); depth * 256 is
// exact, so round-to-nearest-even here equals numpy's float64 rint
__device__ __forceinline__ unsigned enc_raw(float v) {
  const float r = rintf(v * 256.0f);
  return (unsigned)fminf(fmaxf(r, 0.0f), 65535.0f);
}

template <int VEC, typename T>
__device__ __forceinline__ void store_lane_t(T* q, const F4& a, unsigned colmask, bool& over) {
  if constexpr (sizeof(T) == 4) {
    store_lane<VEC>(q, a, colmask);
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) over |= (colmask >> c & 1u) && a.v[c] >= 256.0f;  // write_depth_png raises
    if (colmask == 0xFu) {
      const uint2 u = make_uint2(enc_raw(a.v[0]) | enc_raw(a.v[1]) << 16, enc_raw(a.v[2]) | enc_raw(a.v[3]) << 16);
      __stcs(reinterpret_cast<uint2*>(q), u);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (colmask >> c & 1u) q[c] = (uint16_t)enc_raw(a.v[c]);
    }
  }
}

// bits 0..3: the four columns hold a valid (> 0.1) value
__device__ __forceinline__ unsigned valid_mask(const F4& a) {
  return (unsigned)(a.v[0] > kValid) | (unsigned)(a.v[1] > kValid) << 1 | (unsigned)(a.v[2] > kValid) << 2 |
         (unsigned)(a.v[3] > kValid) << 3;
}

// store_lane_t plus the min over the stored values (FULL output check, S.omin):
// the full-lane branch takes the min of all four, the partial one per column
template <int VEC, typename T>
__device__ __forceinline__ void store_lane_min(T* q, const F4& a, unsigned colmask, bool& over, float& omin) {
  if (colmask == 0xFu) {
    omin = fmn3(fmn3(omin, a.v[0], a.v[1]), a.v[2], a.v[3]);
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (colmask >> c & 1u) omin = fminf(omin, a.v[c]);
  }
  store_lane_t<VEC>(q, a, colmask, over);
}

// ---------------------------------------------------------------------------
// per-item warp geometry
// ---------------------------------------------------------------------------
// ring row stride: >= the production columns, an odd multiple of 4 floats
// (conflict-free row-per-lane float4 loads in lf_rows)
__host__ __device__ __forceinline__ int ring_width(int pw) { return ((pw + 3) & ~3) | 4; }

struct Geo {
  int o0, o1;  // output columns of the strip
  int p0, p1;  // stage-5 production (ring) columns
  int L;       // first lane column of this warp (-4 at the left frame edge)
  int q0, q1;  // stage-5 columns this warp owns (writes to the ring); empty for spare warps
};

__device__ __forceinline__ int warp_q1(int L, int q0, int p1, int W) {
  if (p1 == W && L + kLW - 4 >= W) return W;  // right frame edge, >= 1 out-of-frame lane
  return min(p1, L + kLW - kHalo);
}

__device__ void item_geometry(int s, const Params& p, int warp, Geo& g) {
  g.o0 = s * p.SW;
  g.o1 = min(p.W, g.o0 + p.SW);
  g.p0 = g.o0 == 0 ? 0 : max(0, (g.o0 - 17) & ~3);
  g.p1 = g.o1 == p.W ? p.W : min(p.W, (g.o1 + 17 + 3) & ~3);
  int q0 = g.p0, L = 0, q1 = 0;
  for (int w = 0; w <= warp; ++w) {
    if (q0 >= g.p1) {  // spare warp: duplicate the last one, own nothing
      q0 = q1 = g.p1;
      break;
    }
    L = q0 == 0 ? -4 : q0 - kHalo;
    q1 = warp_q1(L, q0, g.p1, p.W);
    if (w < warp) q0 = q1;
  }
  g.L = L;
  g.q0 = q0;
  g.q1 = q1;
}

// ---------------------------------------------------------------------------
// Phase 1: first valid stage-4 row per column, bit-packed morphology
// ---------------------------------------------------------------------------
// One lane's 4 columns of successive rows for the r0 scan, read from clamped
// addresses so no row needs a bounds check: columns outside the frame read
// in-frame pixels, which only feed the validation max (harmless) and are
// masked out of the validity bits by the caller's column mask.
template <int VEC, typename T>
struct LaneCols {
  const T* a;  // VEC 4: the lane's clamped first column; VEC 2: pair 0; VEC 1: column 0
  int o1, o2, o3;  // VEC 2: o2 = pair 1; VEC 1: columns 1..3 (offsets from a)
  __device__ __forceinline__ LaneCols(const T* frame, int x0, int W) {
    if constexpr (VEC == 4) {
      a = frame + min(max(x0, 0), W - 4);
      o1 = o2 = o3 = 0;
    } else if constexpr (VEC == 2) {
      const int c0 = min(max(x0, 0), W - 2);
      a = frame + c0;
      o1 = o3 = 0;
      o2 = min(max(x0 + 2, 0), W - 2) - c0;
    } else {
      const int c0 = min(max(x0, 0), W - 1);
      a = frame + c0;
      o1 = min(max(x0 + 1, 0), W - 1) - c0;
      o2 = min(max(x0 + 2, 0), W - 1) - c0;
      o3 = min(max(x0 + 3, 0), W - 1) - c0;
    }
  }
  // row at element offset off (= y * W)
  __device__ __forceinline__ F4 row(int64_t off) const {
    const T* q = a + off;
    if constexpr (sizeof(T) == 2) {
      static_assert(VEC == 4, "16-bit input needs W % 4 == 0");
      const uint2 u = __ldg(reinterpret_cast<const uint2*>(q));
      return unpack_raw(u.x, u.y);
    } else if constexpr (VEC == 4) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(q));
      return F4{{t.x, t.y, t.z, t.w}};
    } else if constexpr (VEC == 2) {
      const float2 u = __ldg(reinterpret_cast<const float2*>(q));
      const float2 w = __ldg(reinterpret_cast<const float2*>(q + o2));
      return F4{{u.x, u.y, w.x, w.y}};
    } else {
      return F4{{__ldg(q), __ldg(q + o1), __ldg(q + o2), __ldg(q + o3)}};
    }
  }
};

// Inverted-encoding validity of one row's 4 columns as bits 0..3.  Frames
// whose inputs are negative, non-finite or >= md are flagged by the
// validation max and raise, so here 0 <= v < md and md - v > 0: the inverted
// value md - v is valid iff min(v, md - v) > 0.1 (depth_core.py:150-156).
template <bool PRE>
__device__ __forceinline__ void row_bits(const F4& v, float md, int i, uint32_t w[4], unsigned& umax) {
  if constexpr (PRE) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (v.v[c] > kValid) w[c] |= 1u << i;
  } else {
    umax = max(max(umax, __float_as_uint(v.v[0])), __float_as_uint(v.v[1]));
    umax = max(max(umax, __float_as_uint(v.v[2])), __float_as_uint(v.v[3]));
    const float2 d01 = __ffma2_rn(make_float2(v.v[0], v.v[1]), make_float2(-1.f, -1.f), make_float2(md, md));
    const float2 d23 = __ffma2_rn(make_float2(v.v[2], v.v[3]), make_float2(-1.f, -1.f), make_float2(md, md));
    const float d[4] = {d01.x, d01.y, d23.x, d23.y};
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (fminf(v.v[c], d[c]) > kValid) w[c] |= 1u << i;
  }
}

// bit i of w[c] (i < N = 16 or 32): (inverted) validity of row y0 + i (0
// outside the frame); PRE: the frame is the stage-2 map in the inverted encoding already
template <int VEC, bool PRE, int N, typename T>
__device__ __forceinline__ void load_bits(const LaneCols<VEC, T>& lc, int H, int W, int y0, float md, uint32_t w[4],
                                          unsigned& umax) {
  static_assert(N == 16 || N == 32, "16-row groups");
#pragma unroll
  for (int c = 0; c < 4; ++c) w[c] = 0;
  if (y0 >= H) return;
  if (y0 >= 0 && y0 + N <= H) {
#pragma unroll
    for (int h = 0; h < N / 16; ++h) {
      F4 v[16];
      const int64_t off = (int64_t)(y0 + 16 * h) * W;
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = lc.row(off + (int64_t)i * W);
#pragma unroll
      for (int i = 0; i < 16; ++i) row_bits<PRE>(v[i], md, 16 * h + i, w, umax);
    }
  } else {
    const uint32_t rows = (uint32_t)(((1ull << (min(H - y0, N))) - 1) & ~((1ull << min(max(-y0, 0), N)) - 1));
#pragma unroll 4
    for (int i = 0; i < N; ++i) {
      const int y = min(max(y0 + i, 0), H - 1);
      row_bits<PRE>(lc.row((int64_t)y * W), md, i, w, umax);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) w[c] &= rows;
  }
}

__device__ __forceinline__ uint64_t vdil(uint64_t x, int r) {
  uint64_t o = x;
  for (int i = 1; i <= r; ++i) o |= (x << i) | (x >> i);
  return o;
}

__device__ __forceinline__ uint64_t vero(uint64_t x, int r) {
  uint64_t o = x;
  for (int i = 1; i <= r; ++i) o &= (x << i) & (x >> i);
  return o;
}

template <int R, bool AND>
__device__ __forceinline__ void hcomb(const uint64_t in[4], uint64_t out[4]) {
  uint64_t e[4 + 2 * R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    e[R - 1 - i] = __shfl_up_sync(kFull, in[3 - i], 1);
    e[R + 4 + i] = __shfl_down_sync(kFull, in[i], 1);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) e[R + i] = in[i];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint64_t a = e[c];
#pragma unroll
    for (int d = 1; d <= 2 * R; ++d) a = AND ? (a & e[c + d]) : (a | e[c + d]);
    out[c] = a;
  }
}

template <int VEC, bool PRE, typename T>
__device__ __forceinline__ void phase1(const T* frame, const Params& p, int x0, bool needed, unsigned incol,
                                       int T0[4], unsigned& umax, int s0 = 0) {
  // blocks start at row s0; rows above s0 hold no (inverted-)valid pixel
  const int H = p.H, W = p.W;
  uint32_t prv[4] = {0, 0, 0, 0}, cur[4], nxt[4];
  const LaneCols<VEC, T> lc(frame, x0, W);
  // the window of block b is rows [s0+32b-16, s0+32b+48): nxt holds only the
  // 16 rows below the block (a block usually finds every r0; the rest of the
  // next block is read only when it is needed)
  load_bits<VEC, PRE, 32>(lc, H, W, s0, p.md, cur, umax);
  load_bits<VEC, PRE, 16>(lc, H, W, s0 + 32, p.md, nxt, umax);
  int r0[4] = {-1, -1, -1, -1};
  uint64_t cm[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) cm[c] = (incol >> c & 1) ? ~0ull : 0ull;
  for (int b = 0; s0 + 32 * b < H; ++b) {
    uint64_t X[4], A[4], Bq[4];
    const int ylo = s0 + 32 * b - 16;  // window bit i <-> row ylo + i
    const int lo = max(0, -ylo), hi = min(64, H - ylo);
    const uint64_t inrow = (hi <= lo) ? 0ull : ((hi - lo == 64) ? ~0ull : (((1ull << (hi - lo)) - 1) << lo));
#pragma unroll
    for (int c = 0; c < 4; ++c)
      X[c] = ((uint64_t)(prv[c] >> 16) | ((uint64_t)cur[c] << 16) | ((uint64_t)nxt[c] << 48)) & cm[c];
    // D_shape = cross3 o cross3 (5x5 diamond); PRE: the stage-2 validity is loaded
#pragma unroll
    for (int it = 0; it < (PRE ? 0 : 2); ++it) {
      hcomb<1, false>(X, A);
#pragma unroll
      for (int c = 0; c < 4; ++c) Bq[c] = (vdil(X[c], 1) | A[c]) & inrow & cm[c];
#pragma unroll
      for (int c = 0; c < 4; ++c) X[c] = Bq[c];
    }
    // D5
#pragma unroll
    for (int c = 0; c < 4; ++c) A[c] = vdil(X[c], 2);
    hcomb<2, false>(A, Bq);
    // E5: outside the frame counts as set (clipped window)
#pragma unroll
    for (int c = 0; c < 4; ++c) A[c] = vero((Bq[c] & inrow & cm[c]) | ~(inrow & cm[c]), 2);
    hcomb<2, true>(A, Bq);
    // D7
#pragma unroll
    for (int c = 0; c < 4; ++c) A[c] = vdil(Bq[c] & inrow & cm[c], 3);
    hcomb<3, false>(A, Bq);
    bool done = true;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t cand = (uint32_t)((Bq[c] & inrow & cm[c]) >> 16);
      if (r0[c] < 0 && cand) r0[c] = s0 + 32 * b + __ffs(cand) - 1;
      done = done && (r0[c] >= 0 || !(incol >> c & 1));
    }
    if (__all_sync(kFull, done || !needed)) break;
    uint32_t nhi[4];
    load_bits<VEC, PRE, 16>(lc, H, W, s0 + 32 * b + 48, p.md, nhi, umax);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      prv[c] = cur[c];
      cur[c] = nxt[c] | nhi[c] << 16;
    }
    load_bits<VEC, PRE, 16>(lc, H, W, s0 + 32 * (b + 2), p.md, nxt, umax);
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) T0[c] = r0[c] >= 0 ? (H - 1 - r0[c]) : INT_MAX;
}

// ---------------------------------------------------------------------------
// Large masked fill of one empty pixel (x, row), warp-cooperative: lane i
// takes column x - 15 + i (i < 31) and the max over ring rows [row-15,
// row+15] (clamped == clipped for max); columns outside [p0, p1) lie outside
// the frame (the strip's ring covers every needed window) and count as 0.
// Stage-5 values are >= 0, so their float bit patterns order like the values
// and one redux.max combines the lanes.
// ---------------------------------------------------------------------------
template <int PLAG>
__device__ __forceinline__ float lf_one(const float* __restrict__ ring, int ringw, int p0, int p1, int H, int lane,
                                        int x, int row) {
  const int col = x - kLF + lane;
  unsigned m = 0u;
  if (lane < 2 * kLF + 1 && col >= p0 && col < p1) {
    const float* rc = ring + (col - p0);
    const int r0 = max(row - kLF, 0), r1 = min(row + kLF, H - 1);
    int slot = (r0 + PLAG) % kRing;
#pragma unroll 8
    for (int r = r0; r <= r1; ++r) {
      m = max(m, __float_as_uint(rc[slot * ringw]));
      slot = slot + 1 == kRing ? 0 : slot + 1;
    }
  }
  return __uint_as_float(__reduce_max_sync(kFull, m));
}

// The same pixel with the rows across lanes: lane i takes ring row row-15+i
// and the max over its 31 window columns (nine aligned float4 loads, the
// partial chunks masked); redux.max combines the rows.  The ring row stride is
// an odd multiple of 4 floats (ring_width), so the lanes' 16-byte loads of one
// chunk hit distinct banks.  Needs the whole window inside the strip's ring
// columns: x - 15 >= p0 and x + 15 < p1.
template <int PLAG>
__device__ __forceinline__ float lf_rows(const float* __restrict__ ring, int ringw, int p0, int H, int lane, int x,
                                         int row) {
  const int t = row - kLF + lane;
  unsigned m = 0u;
  if (lane < 2 * kLF + 1 && t >= 0 && t < H) {
    const int c0 = x - kLF - p0;  // first window column (ring index)
    const int a = c0 & ~3, o = c0 - a;
    const float* rp = ring + ((t + PLAG) % kRing) * ringw + a;
    // the window is columns a+o .. a+o+30: chunk 0 (a .. a+3) counts from o,
    // column a+31 needs o >= 1, a+32 / a+33 need o >= 2 / 3
    const float4 q0 = *reinterpret_cast<const float4*>(rp);
    const float4 q7 = *reinterpret_cast<const float4*>(rp + 28);
    const float4 q8 = *reinterpret_cast<const float4*>(rp + 32);
    unsigned u = max(max(__float_as_uint(q0.w), __float_as_uint(q7.x)), __float_as_uint(q7.y));
    u = max(u, __float_as_uint(q7.z));
    if (o <= 2) u = max(u, __float_as_uint(q0.z));
    if (o <= 1) u = max(u, __float_as_uint(q0.y));
    if (o == 0) u = max(u, __float_as_uint(q0.x));
    if (o >= 1) u = max(u, __float_as_uint(q7.w));
    if (o >= 2) u = max(u, __float_as_uint(q8.x));
    if (o >= 3) u = max(u, __float_as_uint(q8.y));
#pragma unroll
    for (int i = 1; i < 7; ++i) {  // columns a+4 .. a+27: inside the window for every o
      const float4 q = *reinterpret_cast<const float4*>(rp + 4 * i);
      u = max(max(u, __float_as_uint(q.x)), __float_as_uint(q.y));
      u = max(max(u, __float_as_uint(q.z)), __float_as_uint(q.w));
    }
    m = u;
  }
  return __uint_as_float(__reduce_max_sync(kFull, m));
}

// Dense large fill (many empty pixels in a warp's block): one pass for the
// vertical 31-row maxima of the block's four rows over the warp's columns
// L-11 .. L+140 into V[4][kVC] (34 ring rows per column), then each lane takes
// the horizontal 31-max of its own empty pixels from V.
constexpr int kVC = 152, kVOff = 11, kDenseMin = 12;
constexpr int kRegDenseMin = 6;  // lf_regdense from this many eligible empties per warp block (~6 per-pixel passes)
// large-fill strategies (fused kernel template parameter DENSE): per-pixel
// warp passes only; + the shared-scratch dense pass (wide strips, config 4);
// + the register-dense pass (DFC_F_SPARSE: its code in the loop costs dense
// frames ~2 %, so it is a separate instantiation)
constexpr int kLfSparse = 0, kLfSmemDense = 1, kLfRegDense = 2;

template <int PLAG>
__device__ __noinline__ void lf_vquad(const float* __restrict__ ring, int ringw, int p0, int p1, int H, int L,
                                      int lane, int c0, bool consecutive, float* __restrict__ V) {
  // vertical 31-maxima of rows c0 .. c0+3 (windows [c_j - 15, c_j + 15]); the
  // rows [c0-12, c0+15] are common to all four
  constexpr int kNC = (kVC + 31) / 32;  // columns per lane: sc = lane + 32 i
  if (consecutive && c0 - kLF >= 0 && c0 + kB - 1 + kLF < H) {
    // every window row lies inside the frame: walk the 34 ring rows once (the
    // slot sequence is the same for all columns), each row feeding the lane's
    // five columns -- no per-load clamp or modulo
    float core[kNC], u15[kNC], u14[kNC], u13[kNC], d16[kNC], d17[kNC], d18[kNC];
    bool ok[kNC];
#pragma unroll
    for (int i = 0; i < kNC; ++i) {
      const int sc = lane + 32 * i, col = L - kVOff + sc;
      ok[i] = sc < kVC && col >= p0 && col < p1;
    }
    const float* cb = ring + (L - kVOff + lane - p0);
    int slot = (c0 - kLF + PLAG) % kRing;  // c0 >= 15 here
#pragma unroll
    for (int k = 0; k < 2 * kLF + kB; ++k) {
      const float* rp = cb + slot * ringw;
#pragma unroll
      for (int i = 0; i < kNC; ++i) {
        float v = 0.f;
        if (ok[i]) v = rp[32 * i];
        if (k == 0) u15[i] = v;
        else if (k == 1) u14[i] = v;
        else if (k == 2) u13[i] = v;
        else if (k == 3) core[i] = v;
        else if (k < 2 * kLF + 1) core[i] = fmx(core[i], v);
        else if (k == 2 * kLF + 1) d16[i] = v;
        else if (k == 2 * kLF + 2) d17[i] = v;
        else d18[i] = v;
      }
      slot = slot + 1 == kRing ? 0 : slot + 1;
    }
#pragma unroll
    for (int i = 0; i < kNC; ++i) {
      const int sc = lane + 32 * i;
      if (sc < kVC) {
        V[0 * kVC + sc] = fmx(core[i], fmx3(u15[i], u14[i], u13[i]));
        V[1 * kVC + sc] = fmx3(core[i], fmx(u14[i], u13[i]), d16[i]);
        V[2 * kVC + sc] = fmx3(core[i], u13[i], fmx(d16[i], d17[i]));
        V[3 * kVC + sc] = fmx(core[i], fmx3(d16[i], d17[i], d18[i]));
      }
    }
    __syncwarp();
    return;
  }
#pragma unroll 1
  for (int sc = lane; sc < kVC; sc += 32) {
    const int col = L - kVOff + sc;
    float o[kB] = {0.f, 0.f, 0.f, 0.f};
    if (col >= p0 && col < p1) {
      const float* rc = ring + (col - p0);
      auto ld = [&](int r) {
        const int rr = r < 0 ? 0 : (r >= H ? H - 1 : r);
        return rc[((rr + PLAG) % kRing) * ringw];
      };
      // near the frame ends: each row centre and window clamped separately
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const int cj = min(max(c0 + j, 0), H - 1);
        float m = ld(cj - kLF);
        for (int r = cj - kLF + 1; r <= cj + kLF; ++r) m = fmx(m, ld(r));
        o[j] = m;
      }
    }
#pragma unroll
    for (int j = 0; j < kB; ++j) V[j * kVC + sc] = o[j];
  }
  __syncwarp();
}

// horizontal 31-max of scratch row j around column x = L + 4 lane + c
__device__ __forceinline__ float lf_hpixel(const float* __restrict__ V, int j, int lane, int c) {
  const float* vr = V + j * kVC + 4 * lane + c + kVOff - kLF;
  float m = vr[0];
#pragma unroll 10
  for (int d = 1; d <= 2 * kLF; ++d) m = fmx(m, vr[d]);
  return m;
}

// all four columns of the lane at once: windows [x_c - 15, x_c + 15] share
// [x_0 - 12, x_0 + 15]
__device__ __forceinline__ F4 lf_hquad(const float* __restrict__ V, int j, int lane) {
  const float* vr = V + j * kVC + 4 * lane + kVOff;  // <-> column x_0 = L + 4 lane
  float core = vr[-12];
#pragma unroll 9
  for (int d = -11; d <= 15; ++d) core = fmx(core, vr[d]);
  const float u15 = vr[-15], u14 = vr[-14], u13 = vr[-13], d16 = vr[16], d17 = vr[17], d18 = vr[18];
  return F4{{fmx(core, fmx3(u15, u14, u13)), fmx3(core, fmx(u14, u13), d16), fmx3(core, u13, fmx(d16, d17)),
             fmx(core, fmx3(d16, d17, d18))}};
}

// Register-dense large fill (many empty pixels in a warp's block, no shared
// scratch needed): the vertical 31-row maxima of the block's four rows for the
// lane's own four columns (one walk over the 34 ring rows, two columns per
// 8-byte load), then each row's horizontal 31-max from the lanes l-4 .. l+4 by
// shuffles: lanes l-3 .. l+3 whole (a sliding max over 7 lanes), lane l-4's
// suffix and lane l+4's prefix maxima for the partial ends.  Exact for the
// columns whose window lies inside the warp's 128 columns (x in [L+15, L+112]);
// the caller keeps the others on the per-pixel passes.  Needs every window row
// inside the frame.  Values are >= 0, out-of-strip columns count as 0.
template <int PLAG>
__device__ __forceinline__ void lf_regdense(const float* __restrict__ ring, int ringw, int p0, int p1, int x0,
                                            int c0, F4 (&w)[kB]) {
  float vm[kB][4];
  int slot0 = (c0 - kLF + PLAG) % kRing;  // c0 >= 15 here
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // column pairs (0, 1), (2, 3)
    const int xa = x0 + 2 * h;
    const bool oka = xa >= p0 && xa < p1, okb = xa + 1 >= p0 && xa + 1 < p1;
    const float* cb = ring + (xa - p0);
    float u15[2], u14[2], u13[2], core[2], d16[2], d17[2], d18[2];
    int slot = slot0;
#pragma unroll
    for (int k = 0; k < 2 * kLF + kB; ++k) {
      float2 q = make_float2(0.f, 0.f);
      if (oka && okb) q = *reinterpret_cast<const float2*>(cb + slot * ringw);
      else if (oka) q.x = cb[slot * ringw];
      else if (okb) q.y = cb[slot * ringw + 1];
      const float v[2] = {q.x, q.y};
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (k == 0) u15[i] = v[i];
        else if (k == 1) u14[i] = v[i];
        else if (k == 2) u13[i] = v[i];
        else if (k == 3) core[i] = v[i];
        else if (k < 2 * kLF + 1) core[i] = fmx(core[i], v[i]);
        else if (k == 2 * kLF + 1) d16[i] = v[i];
        else if (k == 2 * kLF + 2) d17[i] = v[i];
        else d18[i] = v[i];
      }
      slot = slot + 1 == kRing ? 0 : slot + 1;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      vm[0][2 * h + i] = fmx(core[i], fmx3(u15[i], u14[i], u13[i]));
      vm[1][2 * h + i] = fmx3(core[i], fmx(u14[i], u13[i]), d16[i]);
      vm[2][2 * h + i] = fmx3(core[i], u13[i], fmx(d16[i], d17[i]));
      vm[3][2 * h + i] = fmx(core[i], fmx3(d16[i], d17[i], d18[i]));
    }
  }
#pragma unroll
  for (int j = 0; j < kB; ++j) {
    const float* g = vm[j];
    const float M = fmx(fmx3(g[0], g[1], g[2]), g[3]);
    const float A = fmx(M, __shfl_down_sync(kFull, M, 1));
    const float Bm = fmx(A, __shfl_down_sync(kFull, A, 2));
    const float C = fmx(Bm, __shfl_down_sync(kFull, Bm, 3));
    const float F = __shfl_up_sync(kFull, C, 3);  // max over lanes l-3 .. l+3
    const float s2 = fmx(g[2], g[3]), s1 = fmx(g[1], s2);
    const float p1_ = fmx(g[0], g[1]), p2_ = fmx(p1_, g[2]);
    const float Ls1 = __shfl_up_sync(kFull, s1, 4), Ls2 = __shfl_up_sync(kFull, s2, 4);
    const float Ls3 = __shfl_up_sync(kFull, g[3], 4);
    const float Rp0 = __shfl_down_sync(kFull, g[0], 4), Rp1 = __shfl_down_sync(kFull, p1_, 4);
    const float Rp2 = __shfl_down_sync(kFull, p2_, 4);
    w[j].v[0] = fmx(F, Ls1);
    w[j].v[1] = fmx3(F, Ls2, Rp0);
    w[j].v[2] = fmx3(F, Ls3, Rp1);
    w[j].v[3] = fmx(F, Rp2);
  }
}

// ---------------------------------------------------------------------------
// Tensor memory as a per-thread store for the rows each stage carries from
// one block to the next (TMEM is otherwise idle here: no MMA).  Each warp owns
// 96 columns of its lane quarter (warps w, w+4, w+8 share quarter w & 3); a
// thread reads / writes its own lane with the 32x32b shapes, one x16 / x8
// load right before a stage and one store right after it.  Off the register
// file, the carried rows no longer stay live across the whole block: 168
// registers with 136 B of spills became 148 registers with none, and the
// per-block rotation moves are gone (config 1: 598k -> 701k frames/s).
// ---------------------------------------------------------------------------
constexpr int kTmCols = 512;   // allocation (power of 2 >= 3 warps x 96 columns)
constexpr int kTmSlice = 96;   // c5 0..23, gc 24..39, c3 40..55, c4 56..71, c1 72..79, c2 80..87
static_assert(((kNW + 3) / 4) * kTmSlice <= kTmCols, "TMEM slices");

// ---------------------------------------------------------------------------
// per-item state and one 4-row iteration (EDGE: rows may leave the frame)
// ---------------------------------------------------------------------------
// Per-warp mbarriers (32 arrivals: every lane releases its own stores) replace the per-block CTA barrier.  A
// warp's ring columns are read only by itself and its two neighbours (lane
// halos +-12, large fill +-17 < the 104 owned columns), so warps synchronise
// with their neighbours only: P_w[g & 3] completes when warp w has stored
// block g's stage-5 rows, C_w[g & 3] when it has finished block g's consumer
// (g counts blocks across items).  Warp w overwrites ring slot g mod 10 (rows
// of block g - 10) after C_{w+-1}[g - 2] (consumers read blocks >= g' - 8 at
// block g'); that also implies P_{w+-1}[g - 4], the newest rows a consumer
// reads outside the large fill.  The large fill waits P_{w+-1}[g].
__device__ __forceinline__ void mb_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t a, uint32_t parity) {
#ifdef DFC_MB_HINT
  // suspend until the phase completes (or the hint, in ns, elapses) instead of
  // re-polling: the spin loop's YIELD / TRYWAIT / BRA took issue slots
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity), "n"(DFC_MB_HINT)
      : "memory");
#else
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
#endif
}

struct State {
  const float* rring;  // consumer read base: ring + clamped lane column
  float* wring;        // producer write base: ring + lane column (owned lanes only)
  float* ring;
  int ringw, x0, lane, L, p0, p1;
  unsigned own, outm, oob;
  bool woob;
  unsigned needm;  // columns the consumer needs (owned +- 2 inside the strip)
  int T0[4];
  float top[4];
  int tmin, tmax;
  int tmaxN;           // max r0 row (processing order) over the columns the consumer needs
  bool skip, fast;
  F4 mprev[2];        // PARTIAL: pre-blur rows for the re-impose mask
  F4 ofast;            // output row above every needed r0 (FULL): all such rows are equal
  uint32_t stg;        // shared-memory staging slot of this lane (row j at +512 j)
  const void* lrow;    // input row of processing row t0 + kB at column x0
  void* orow;          // output row of processing row tc0 - 2 at column x0
  bool enc_over;       // IO 2: an output >= 256 m (not encodable)
  bool full;           // all 4 columns inside the frame
  unsigned incol;
#ifdef DFC_TIMING
  long long tacc[6];   // diagnostics: producer, barrier, consumer, phase 1, consumer LF part, store-only rows
#endif
  unsigned umax;
  float2 cin01, cin23, own01, own23;  // per-column valid-input counts (float, exact < 2^24), owned-column weights
  unsigned nin, nout;  // valid-pixel counters (owned output columns): inputs read, outputs stored (PARTIAL)
  float omin;          // FULL: min stored output (fast rows repeat a stored row); outputs are valid
                       // (nearly) always, so the count is H x owned columns unless omin <= 0.1, when
                       // finalize_kernel recounts the frame
  bool had_empty, still_empty;
  int zrun;            // PARTIAL: consecutive producer blocks with an all-zero inverted input
  uint32_t mbW, mbL, mbR;  // shared addresses of this warp's / the neighbours' P[4], C[4] mbarriers
  bool hasL, hasR;
  int gk;              // block counter across items (mbarrier index and phase)
  int pblk;            // ring block of the producer's rows (k mod ring blocks)
  uint32_t tm;         // tensor-memory address of this thread's carried rows (c5, gc)
  bool edgeL;          // this lane holds column 0
  int compR;           // component of column W - 1 in this lane, else -1
};

template <int VEC, bool FULL, int BLUR, bool PRE, int DENSE, int IO, bool EDGE>
__device__ __forceinline__ void iterate(const Params& p, State& S, int k) {
  using TIn = typename IoT<IO>::In;
  using TOut = typename IoT<IO>::Out;
  using LG = Lags<PRE>;
  const int H = p.H, W = p.W;
  const int t0 = kB * k;
  const int tp = t0 - LG::P;
  constexpr int L2 = LG::L2;
#ifdef DFC_TIMING
  const long long ta = clock64();
#endif
  // ======================= producer =======================
  if (FULL && !S.skip && tp > S.tmax) S.skip = true;
  F4 f[kB];
  if (!S.skip) {
    F4 a[kB];
    cp_async_wait_all();  // this block's rows, staged one block ago
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      a[j] = lds4_t<TIn>(S.stg + j * 512);
      if constexpr (!PRE) {
        // invert (depth_core.py:150-156): md - v for a column pair per FFMA2 (exact: -1 * v + md)
        S.umax = max(max(S.umax, __float_as_uint(a[j].v[0])), __float_as_uint(a[j].v[1]));
        S.umax = max(max(S.umax, __float_as_uint(a[j].v[2])), __float_as_uint(a[j].v[3]));
        const float2 d01 = __ffma2_rn(make_float2(a[j].v[0], a[j].v[1]), make_float2(-1.f, -1.f), make_float2(p.md, p.md));
        const float2 d23 = __ffma2_rn(make_float2(a[j].v[2], a[j].v[3]), make_float2(-1.f, -1.f), make_float2(p.md, p.md));
        // validity as 1.0f / 0.0f (one FSET each, ALU pipe); the select and the
        // RunStats.input_density count (pipeline.py:138-141) then run on the FMA
        // pipe: (md - v) * 1 and (md - v) * 0 are exact (md - v > 0 on frames
        // that do not raise), and the per-lane count weights each column by
        // whether this lane owns it as an output column.  Rows above the skip
        // point are not read here; they hold no input that is still valid once
        // inverted, and finalize_kernel recounts the rare frames that hold
        // inputs within 0.1 of max_depth.
        const float2 q01 = make_float2(a[j].v[0] > kValid ? 1.f : 0.f, a[j].v[1] > kValid ? 1.f : 0.f);
        const float2 q23 = make_float2(a[j].v[2] > kValid ? 1.f : 0.f, a[j].v[3] > kValid ? 1.f : 0.f);
        const float2 m01 = __fmul2_rn(d01, q01), m23 = __fmul2_rn(d23, q23);
        a[j].v[0] = m01.x, a[j].v[1] = m01.y, a[j].v[2] = m23.x, a[j].v[3] = m23.y;
        // one accumulator pair for all four columns (two registers less in the block loop: +1.5 % on
        // config 1); W % 4 == 0: a lane owns all of its columns or none, so one weight pair serves both
        S.cin01 = __ffma2_rn(q01, S.own01, S.cin01);
        S.cin01 = __ffma2_rn(q23, VEC == 4 ? S.own01 : S.own23, S.cin01);
      }
    }

    // stage the next block; stops once its stage-5 rows lie above every r0.
    // The values read above are materialised first: the shared reads are
    // complete before the slot is overwritten.
    if constexpr (PRE) {
#pragma unroll
      for (int j = 0; j < kB; ++j)
        asm volatile("" ::"f"(a[j].v[0]), "f"(a[j].v[1]), "f"(a[j].v[2]), "f"(a[j].v[3]));
    } else {
      asm volatile("" ::"r"(S.umax));
    }
    if (!FULL || (t0 + kB - LG::P <= S.tmax)) {
      const TIn* q = static_cast<const TIn*>(S.lrow);
#pragma unroll
      for (int j = 0; j < kB; ++j, q -= W)
        stage_lane<VEC>(S.stg + j * 512, q, p.in, !EDGE || t0 + kB + j < H, S.full, S.incol);
      cp_async_commit();
    }
    // PARTIAL: once the inverted input has been all zero for 6 blocks (24 rows,
    // more than the stages' 2 x 9-row reach), every stage value the block
    // produces or carries in TMEM is 0, so the stages are skipped (the rows
    // above the first LIDAR scanline: about a third of a KITTI-like frame)
    bool zskip = false;
    if constexpr (!FULL) {
      float mx = 0.f;
#pragma unroll
      for (int j = 0; j < kB; ++j) mx = fmx3(mx, fmx3(a[j].v[0], a[j].v[1], a[j].v[2]), a[j].v[3]);
      S.zrun = __all_sync(kFull, mx == 0.f) ? S.zrun + 1 : 0;  // (NaN == 0 is false)
      zskip = S.zrun > 5;
    }
    if (!zskip) {
    // --- stage 2: cross3 o cross3 = 5x5 diamond (rows t0-2+j); PRE: the staged rows ---
    F4 d2[kB];
    if constexpr (PRE) {
#pragma unroll
      for (int j = 0; j < kB; ++j) d2[j] = a[j];  // rows >= H and out-of-frame columns were staged as 0
    } else {
    F4 d1[kB];
    {
      F4 c1[2];
      tm_wait_st();
      tm_ld_rows(S.tm + 72, c1, 2);
      const F4 in[kB + 2] = {c1[0], c1[1], a[0], a[1], a[2], a[3]};
      tm_st_rows(S.tm + 72, a + 2, 2);
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const Ext<1> e = ext_row<1>(in[j + 1]);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          d1[j].v[c] = fmx3(fmx3(in[j].v[c], in[j + 1].v[c], in[j + 2].v[c]), e.e[c], e.e[c + 2]);
      }
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        if (EDGE && (t0 - 1 + j < 0 || t0 - 1 + j >= H)) set_row(d1[j], 0.f);
      }
    }
    // --- cross3 #2 (rows t0-2+j) ---
    {
      F4 c2[2];
      tm_ld_rows(S.tm + 80, c2, 2);
      const F4 in[kB + 2] = {c2[0], c2[1], d1[0], d1[1], d1[2], d1[3]};
      tm_st_rows(S.tm + 80, d1 + 2, 2);
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const Ext<1> e = ext_row<1>(in[j + 1]);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          d2[j].v[c] = fmx3(fmx3(in[j].v[c], in[j + 1].v[c], in[j + 2].v[c]), e.e[c], e.e[c + 2]);
      }
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        if (EDGE && (t0 - 2 + j < 0 || t0 - 2 + j >= H)) set_row(d2[j], 0.f);
      }
    }
    }
    // --- close: max5 (rows t0-L2-2+j) ---
    F4 m5[kB];
    {
      F4 c3[4];
      tm_ld_rows(S.tm + 40, c3, 4);
      const F4 in[kB + 4] = {c3[0], c3[1], c3[2], c3[3], d2[0], d2[1], d2[2], d2[3]};
      tm_st_rows(S.tm + 40, d2, 4);
      F4 vv[kB];
      vwin2<OpMax>(in, vv);
#pragma unroll
      for (int j = 0; j < kB; ++j) m5[j] = hwin2<OpMax>(ext_row<2>(vv[j]));
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        if constexpr (VEC == 4) {
          // W % 4 == 0: a lane lies wholly inside or outside the frame, so the fix is four selects on one
          // lane predicate instead of a mask test per column (the edge warps pace their CTA: +1 %)
          if (S.woob) {
#pragma unroll
            for (int c = 0; c < 4; ++c) m5[j].v[c] = S.oob ? kFMax : m5[j].v[c];
          }
          if (EDGE && (t0 - L2 - 2 + j < 0 || t0 - L2 - 2 + j >= H)) set_row(m5[j], kFMax);
        } else {
          if (EDGE && (t0 - L2 - 2 + j < 0 || t0 - L2 - 2 + j >= H)) set_row(m5[j], kFMax);
          if (S.woob) fix_oob(m5[j], S.oob, kFMax);
        }
      }
    }
    // --- close: min5 (rows t0-L2-4+j) ---
    F4 cl[kB];
    {
      F4 c4[4];
      tm_ld_rows(S.tm + 56, c4, 4);
      const F4 in[kB + 4] = {c4[0], c4[1], c4[2], c4[3], m5[0], m5[1], m5[2], m5[3]};
      tm_st_rows(S.tm + 56, m5, 4);
      F4 vv[kB];
      vwin2<OpMin>(in, vv);
#pragma unroll
      for (int j = 0; j < kB; ++j) cl[j] = hwin2<OpMin>(ext_row<2>(vv[j]));
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        if (EDGE && (t0 - L2 - 4 + j < 0 || t0 - L2 - 4 + j >= H)) set_row(cl[j], 0.f);
        if constexpr (VEC == 4) {
          if (S.woob) {
#pragma unroll
            for (int c = 0; c < 4; ++c) cl[j].v[c] = S.oob ? 0.f : cl[j].v[c];
          }
        } else if (S.woob) {
          fix_oob(cl[j], S.oob, 0.f);
        }
      }
    }
    // --- small fill: masked max7 (rows t0-L2-7+j = tp+j) ---
    {
      F4 c5[6];
      tm_wait_st();  // the previous block's store of these rows
      tm_ld_rows(S.tm, c5, 6);
      const F4 in[kB + 6] = {c5[0], c5[1], c5[2], c5[3], c5[4], c5[5], cl[0], cl[1], cl[2], cl[3]};
      F4 vv[kB];
      vwin3<OpMax>(in, vv);
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const F4 h7 = hwin3<OpMax>(ext_row<3>(vv[j]));
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float ctr = in[j + 3].v[c];
          f[j].v[c] = ctr > kValid ? ctr : h7.v[c];
        }
      }
      {
        const F4 n5[6] = {c5[4], c5[5], cl[0], cl[1], cl[2], cl[3]};
        tm_st_rows(S.tm, n5, 6);
      }
    }
    // --- extend to top (FULL; only blocks reaching some column's r0) ---
    if (FULL && tp + kB - 1 >= S.tmin) {
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const int t = tp + j;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (t == S.T0[c]) S.top[c] = f[j].v[c];
          if (t > S.T0[c]) f[j].v[c] = S.top[c];
        }
      }
    }
    } else {
#pragma unroll
      for (int j = 0; j < kB; ++j) set_row(f[j], 0.f);
    }
  } else {
#pragma unroll
    for (int j = 0; j < kB; ++j)
#pragma unroll
      for (int c = 0; c < 4; ++c) f[j].v[c] = S.top[c];
  }
  S.lrow = static_cast<const TIn*>(S.lrow) - kB * W;
  // --- ring store: ring slot of row t is (t + P) mod 40, so this block is slots 4*(k mod 10) + j ---
  const int g = S.gk++;
  if (g >= 2) {
    const uint32_t o = 32 + ((g - 2) & 3) * 8, ph = ((g - 2) >> 2) & 1;
#ifdef DFC_TIMING
    const long long tw = clock64();
#endif
    if (S.hasL) mb_wait(S.mbL + o, ph);
    if (S.hasR) mb_wait(S.mbR + o, ph);
#ifdef DFC_TIMING
    S.tacc[1] += clock64() - tw;
#endif
  }
  if (S.own) {
    float* w = S.wring + S.pblk * (kB * S.ringw);
#pragma unroll
    for (int j = 0; j < kB; ++j)
      if (!EDGE || (tp + j >= 0 && tp + j < H))
        *reinterpret_cast<float4*>(w + j * S.ringw) = make_float4(f[j].v[0], f[j].v[1], f[j].v[2], f[j].v[3]);
  }
  const int cblk = S.pblk >= kLag / kB ? S.pblk - kLag / kB : S.pblk + kRingBlocks - kLag / kB;
  S.pblk = S.pblk == kRingBlocks - 1 ? 0 : S.pblk + 1;
  mb_arrive(S.mbW + (g & 3) * 8);  // every lane (count 32): each lane's ring stores are released by its own arrival
#ifdef DFC_TIMING
  const long long tb = clock64();
  struct ConsTimer {
    long long* t;
    long long tc;
    __device__ ~ConsTimer() { t[2] += clock64() - tc; }
  } ct{S.tacc, clock64()};
  S.tacc[0] += tb - ta;
#endif
  // ======================= consumer =======================
  do {
  const int tc0 = t0 - LG::C;
  if (k < LG::KFirst) break;
  TOut* orow = static_cast<TOut*>(S.orow);  // output row of processing row tc0 - 2
  S.orow = orow - kB * W;
  if (FULL && S.fast) {
#ifdef DFC_TIMING
    S.tacc[5] += 1;
#endif
    // every row of the blur windows lies above each needed column's r0: the
    // stage-6 rows are the captured top values and every output row is equal
    // output rows: tc0 - 2 + j with the Gaussian, tc0 + j otherwise (as below)
    constexpr int kOff = BLUR == DFC_BLUR_GAUSSIAN ? 2 : 0;
    if (kOff == 0) orow -= 2 * W;
#pragma unroll
    for (int j = 0; j < kB; ++j, orow -= W) {
      const int t = tc0 - kOff + j;
      if (EDGE && (t < 0 || t >= H)) continue;
      if (S.outm) store_lane_t<VEC>(orow, S.ofast, S.outm, S.enc_over);
    }
    break;
  }
  F4 v6[kB];
  {
    // rows tc0 + j live in slots 4*((k + 6) mod 10) + j when inside the frame
    const float* r = S.rring + cblk * (kB * S.ringw);
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const float* rr = r + j * S.ringw;
      if (EDGE) {
        const int t = min(max(tc0 + j, 0), H - 1);
        rr = S.rring + ((t + LG::P) % kRing) * S.ringw;
      }
      const float4 q = *reinterpret_cast<const float4*>(rr);
      v6[j].v[0] = q.x, v6[j].v[1] = q.y, v6[j].v[2] = q.z, v6[j].v[3] = q.w;
    }
  }
  if (FULL) {
    // any needed empty pixel in this block?
    float mn = kFMax;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float cm = fminf(fminf(v6[0].v[c], v6[1].v[c]), fminf(v6[2].v[c], v6[3].v[c]));
      if (S.needm >> c & 1) mn = fminf(mn, cm);
    }
    if (__any_sync(kFull, !(mn > kValid))) {
      unsigned em = 0;  // bit 4j+c: needed empty pixel
#pragma unroll
      for (int j = 0; j < kB; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) em |= (unsigned)((S.needm >> c & 1) && !(v6[j].v[c] > kValid)) << (4 * j + c);
      S.had_empty |= em != 0;
      unsigned lanes = __ballot_sync(kFull, em != 0);
      // neighbours' rows up to tc0 + 18
      if (S.hasL) mb_wait(S.mbL + (g & 3) * 8, (g >> 2) & 1);
      if (S.hasR) mb_wait(S.mbR + (g & 3) * 8, (g >> 2) & 1);
      if constexpr (DENSE == kLfRegDense) {
        // many empties: the register-dense pass for the columns it covers
        // columns whose 31-wide window lies in the warp's lanes: x in [L + 15, L + 112]
        const unsigned elc = (S.lane >= 4 && S.lane <= 27) ? 0xFu
                             : (S.lane == 3 ? 0x8u : (S.lane == 28 ? 0x1u : 0u));
        const unsigned el = em & (elc * 0x1111u);
        if (tc0 - kLF >= 0 && tc0 + kB - 1 + kLF < H &&
            __reduce_add_sync(kFull, __popc(el)) > kRegDenseMin) {
          F4 wv[kB];
          lf_regdense<LG::P>(S.ring, S.ringw, S.p0, S.p1, S.x0, tc0, wv);
#pragma unroll
          for (int j = 0; j < kB; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (el >> (4 * j + c) & 1u) {
                v6[j].v[c] = wv[j].v[c];
                S.still_empty |= !(wv[j].v[c] > kValid);
              }
          em &= ~el;
          lanes = __ballot_sync(kFull, em != 0);
        }
      }
      if (DENSE == kLfSmemDense && __reduce_add_sync(kFull, __popc(em)) > kDenseMin) {
        float* V = S.ring + kRing * S.ringw + p.nw * (kB * 128) + (threadIdx.x >> 5) * (kB * kVC);
        lf_vquad<LG::P>(S.ring, S.ringw, S.p0, S.p1, H, S.L, S.lane, tc0, !EDGE || (tc0 >= 0 && tc0 + kB - 1 < H),
                        V);
#pragma unroll
        for (int j = 0; j < kB; ++j) {
          const unsigned rowm = (em >> (4 * j)) & 0xFu;
          if (__popc(rowm) >= 2) {  // the lane's four windows together
            const F4 h = lf_hquad(V, j, S.lane);
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (rowm >> c & 1u) {
                v6[j].v[c] = h.v[c];
                S.still_empty |= !(h.v[c] > kValid);
              }
          } else if (rowm) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (rowm >> c & 1u) {
                const float r = lf_hpixel(V, j, S.lane, c);
                v6[j].v[c] = r;
                S.still_empty |= !(r > kValid);
              }
          }
        }
        __syncwarp();
        lanes = 0;
      }
      while (lanes) {
        const int src = __ffs(lanes) - 1;
        lanes &= lanes - 1;
        unsigned pe = __shfl_sync(kFull, em, src);
        do {
          const int b = __ffs(pe) - 1;
          pe &= pe - 1;
          const int row = EDGE ? min(max(tc0 + (b >> 2), 0), H - 1) : tc0 + (b >> 2);
          const int x = S.L + 4 * src + (b & 3);
          const float r = (x - kLF >= S.p0 && x + kLF < S.p1)
                              ? lf_rows<LG::P>(S.ring, S.ringw, S.p0, H, S.lane, x, row)
                              : lf_one<LG::P>(S.ring, S.ringw, S.p0, S.p1, H, S.lane, x, row);
          if (S.lane == src) {
#pragma unroll
            for (int j = 0; j < kB; ++j)
#pragma unroll
              for (int c = 0; c < 4; ++c)
                if (b == 4 * j + c) v6[j].v[c] = r;
            S.still_empty |= !(r > kValid);
          }
        } while (pe);
      }
    }
  }
#ifdef DFC_TIMING
  S.tacc[4] += clock64() - ct.tc;
#endif
  if constexpr (BLUR == DFC_BLUR_GAUSSIAN) {
    F4 h[kB];
    // replicate border: the lanes holding column 0 / W - 1 overwrite the
    // out-of-frame entries of their window with the edge value (only they
    // and, when W - 1 starts a lane, the lane before it produce in-frame
    // outputs from out-of-frame columns; that one reads the sender's patch).
    // One warp-uniform branch for the whole block: interior warps skip it.
    if (S.woob) {
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        if constexpr (VEC == 2) {  // W % 4 == 2: column W - 1 is component 1 of its lane
          if (S.compR >= 0) v6[j].v[2] = v6[j].v[3] = v6[j].v[1];
        } else if constexpr (VEC == 1) {
          if (S.compR >= 0 && S.compR < 3) {
            const float ev = S.compR == 0 ? v6[j].v[0] : (S.compR == 1 ? v6[j].v[1] : v6[j].v[2]);
#pragma unroll
            for (int c = 1; c < 4; ++c)
              if (c > S.compR) v6[j].v[c] = ev;
          }
        }
      }
    }
    Ext<2> ex[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) ex[j] = ext_row<2>(v6[j]);
    if (S.woob) {
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        Ext<2>& e = ex[j];
        if (S.edgeL) e.e[0] = e.e[1] = e.e[2];
        if (S.compR >= 0) {
          if constexpr (VEC == 4) {
            e.e[6] = e.e[7] = e.e[5];
          } else if constexpr (VEC == 2) {
            e.e[6] = e.e[7] = e.e[3];
          } else {
            const float ev = S.compR == 0 ? e.e[2] : (S.compR == 1 ? e.e[3] : (S.compR == 2 ? e.e[4] : e.e[5]));
#pragma unroll
            for (int i = 3; i < 8; ++i)
              if (i > S.compR + 2) e.e[i] = ev;
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const Ext<2>& e = ex[j];
#pragma unroll
      for (int hp = 0; hp < 2; ++hp) {  // packed fp32x2: outputs (2hp, 2hp+1), inputs broadcast
        const float* x = e.e + 2 * hp;
        float2 a = __fmul2_rn(make_float2(x[0], x[0]), p.gh[0]);
#pragma unroll
        for (int i = 1; i < 6; ++i) a = __ffma2_rn(make_float2(x[i], x[i]), p.gh[i], a);
        h[j].v[2 * hp] = a.x;
        h[j].v[2 * hp + 1] = a.y;
      }
    }
    F4 gcv[4];
    tm_wait_st();
    tm_ld_rows(S.tm + 24, gcv, 4);
    if (EDGE && k == LG::KFirst) {  // rows above row 0 replicate it (tc0 in [-3, 0]: h[0] is row 0)
#pragma unroll
      for (int i = 0; i < 4; ++i) gcv[i] = h[0];
    }
    const F4 in[kB + 4] = {gcv[0], gcv[1], gcv[2], gcv[3], h[0], h[1], h[2], h[3]};
    tm_st_rows(S.tm + 24, h, 4);
    F4 mk[kB];
    if (!FULL) {  // pre-blur validity of output rows tc0-2+j (pipeline.py:212-214)
      mk[0] = S.mprev[0], mk[1] = S.mprev[1], mk[2] = v6[0], mk[3] = v6[1];
      S.mprev[0] = v6[2], S.mprev[1] = v6[3];
    }
    F4 o;
#pragma unroll
    for (int j = 0; j < kB; ++j, orow -= W) {
      const int t = tc0 + j - 2;  // output row (processing order)
      if (EDGE && (t < 0 || t >= H)) continue;
#pragma unroll
      for (int hp = 0; hp < 2; ++hp) {  // packed fp32x2 over the column pair (2hp, 2hp+1)
        const int c = 2 * hp;
        float2 a = __fmul2_rn(make_float2(in[j].v[c], in[j].v[c + 1]), make_float2(p.gw[0], p.gw[0]));
#pragma unroll
        for (int i = 1; i < 5; ++i)
          a = __ffma2_rn(make_float2(in[j + i].v[c], in[j + i].v[c + 1]), make_float2(p.gw[i], p.gw[i]), a);
        const float2 r = __ffma2_rn(a, make_float2(-1.f, -1.f), make_float2(p.md, p.md));  // md - a, exact negation
        // invert back (depth_core.py:150-156): (md - a) * 1.0f / 0.0f; md - a > 0 (a < md)
        const float2 ov = __fmul2_rn(r, make_float2(a.x > kValid ? 1.f : 0.f, a.y > kValid ? 1.f : 0.f));
        o.v[c] = ov.x;
        o.v[c + 1] = ov.y;
        if (!FULL && !(mk[j].v[c] > kValid)) o.v[c] = 0.0f;
        if (!FULL && !(mk[j].v[c + 1] > kValid)) o.v[c + 1] = 0.0f;
      }
      if (FULL) {
        if (S.outm) store_lane_min<VEC>(orow, o, S.outm, S.enc_over, S.omin);
      } else {
        if (S.outm) store_lane_t<VEC>(orow, o, S.outm, S.enc_over);
        S.nout += __popc(valid_mask(o) & S.outm);
      }
    }
    // rows tc0-4 .. tc0+3 above every needed r0: output row tc0+1 repeats from here on
    if (FULL && !EDGE && tc0 - 4 > S.tmaxN) {
      S.fast = true;
      S.ofast = o;
    }
  } else {
    orow -= 2 * W;  // no blur: output rows are tc0 + j
    F4 o;
#pragma unroll
    for (int j = 0; j < kB; ++j, orow -= W) {
      const int t = tc0 + j;
      if (EDGE && (t < 0 || t >= H)) continue;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        o.v[c] = BLUR == kBlurRaw ? v6[j].v[c] : (v6[j].v[c] > kValid ? p.md - v6[j].v[c] : 0.0f);
      if (FULL && BLUR != kBlurRaw) {
        if (S.outm) store_lane_min<VEC>(orow, o, S.outm, S.enc_over, S.omin);
      } else {
        if (S.outm) store_lane_t<VEC>(orow, o, S.outm, S.enc_over);
        if (BLUR != kBlurRaw) S.nout += __popc(valid_mask(o) & S.outm);
      }
    }
    if (FULL && !EDGE && tc0 > S.tmaxN) {
      S.fast = true;
      S.ofast = o;
    }
  }
  } while (0);
  mb_arrive(S.mbW + 32 + (g & 3) * 8);
}

// ---------------------------------------------------------------------------
// the fused kernel
// ---------------------------------------------------------------------------
template <int VEC, bool FULL, int BLUR, bool PRE, int DENSE, int IO>
__global__ void __launch_bounds__(kNW * 32, 1) fused_kernel(const __grid_constant__ Params p) {
  using TIn = typename IoT<IO>::In;
  using TOut = typename IoT<IO>::Out;
  using LG = Lags<PRE>;
  extern __shared__ __align__(16) float smem[];
  __shared__ unsigned s_item;
  __shared__ __align__(8) unsigned long long s_mb[kNW * 8];  // per warp: P[4], C[4]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(s_mb);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < kNW * 8; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mb0 + 8 * i), "r"(kMbCount) : "memory");
  }
  __shared__ uint32_t s_tm;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tm)),
                 "n"(kTmCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmbase = s_tm;
  int gk = 0;  // blocks done across items (mbarrier phases); first use is after the item barrier below
  const int H = p.H, W = p.W;
  const int64_t HW = (int64_t)H * W;
  const unsigned total = (unsigned)(p.nframes * p.strips);

  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(p.work, 1u);
    __syncthreads();
    const unsigned item = s_item;
    __syncthreads();
    if (item >= total) break;
    const int64_t frame = item / p.strips;
    Geo g;
    item_geometry((int)(item % p.strips), p, warp, g);
    State S;
    S.ringw = ring_width(g.p1 - g.p0);
    S.ring = smem;
    const TIn* src = static_cast<const TIn*>(p.in) + frame * HW;
    TOut* dst = static_cast<TOut*>(p.out) + frame * HW;
    S.x0 = g.L + 4 * lane;
    S.lane = lane;
    S.L = g.L;
    S.p0 = g.p0;
    S.p1 = g.p1;
    S.wring = S.ring + (S.x0 - g.p0);
    S.rring = S.ring + (min(max(S.x0, g.p0), g.p0 + S.ringw - 4) - g.p0);
    unsigned incol = 0, needm = 0;
    S.own = S.outm = S.oob = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int x = S.x0 + c;
      incol |= (unsigned)(x >= 0 && x < W) << c;
      S.oob |= (unsigned)(x < 0 || x >= W) << c;
      S.own |= (unsigned)(x >= g.q0 && x < g.q1) << c;
      S.outm |= (unsigned)(x >= max(g.q0, g.o0) && x < min(g.q1, g.o1)) << c;
      const bool need = x >= max(max(g.q0 - 2, g.o0 - 2), max(g.p0, 0)) && x < min(min(g.q1 + 2, g.o1 + 2), g.p1);
      needm |= (unsigned)need << c;
    }
    S.incol = incol;
    S.needm = needm;

    S.full = incol == 0xFu;
    S.woob = __any_sync(kFull, S.oob != 0);
    S.edgeL = S.x0 == 0;                                           // lane holding column 0
    S.compR = (S.x0 <= W - 1 && W - 1 <= S.x0 + 3) ? W - 1 - S.x0 : -1;  // component of column W - 1
    S.umax = 0;
    S.nin = S.nout = 0;
    S.cin01 = S.cin23 = make_float2(0.f, 0.f);
    S.own01 = make_float2((float)(S.outm & 1u), (float)(S.outm >> 1 & 1u));
    S.own23 = make_float2((float)(S.outm >> 2 & 1u), (float)(S.outm >> 3 & 1u));
    S.omin = kFMax;
    S.had_empty = S.still_empty = false;
    S.skip = S.fast = S.enc_over = false;
    S.zrun = 0;
    S.mbW = mb0 + warp * 64;
    S.mbL = mb0 + (warp - 1) * 64;
    S.mbR = mb0 + (warp + 1) * 64;
    S.hasL = warp > 0;
    S.hasR = warp + 1 < p.nw;
    S.gk = gk;
    S.pblk = 0;
    S.tmaxN = INT_MAX;
    set_row(S.ofast, 0.f);

    // ---------------- phase 1 ----------------
#ifdef DFC_TIMING
    const long long tph = clock64();
    S.tacc[0] = S.tacc[1] = S.tacc[2] = S.tacc[3] = S.tacc[4] = S.tacc[5] = 0;
#endif
#pragma unroll
    for (int c = 0; c < 4; ++c) S.T0[c] = INT_MAX, S.top[c] = 0.f;
    S.tmax = S.tmin = INT_MAX;
    if (FULL) {
      // phase 1 ran in r0_kernel for the whole round (latency-bound scans overlap there)
      const int32_t* tr = p.t0g + frame * W + S.x0;
#pragma unroll
      for (int c = 0; c < 4; ++c) S.T0[c] = (incol >> c & 1) ? __ldg(tr + c) : INT_MAX;
      int mx = INT_MIN, mn = INT_MAX, mxn = INT_MIN;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (S.own >> c & 1) {
          mx = max(mx, S.T0[c]);
          mn = min(mn, S.T0[c]);
        }
        if (needm >> c & 1) mxn = max(mxn, S.T0[c]);
      }
      S.tmax = __reduce_max_sync(kFull, mx);
      S.tmin = __reduce_min_sync(kFull, mn);
      S.tmaxN = __reduce_max_sync(kFull, mxn);
    }

#ifdef DFC_TIMING
    S.tacc[3] = 0;
    (void)tph;
#endif
    // ---------------- phase 2 ----------------
#pragma unroll
    for (int i = 0; i < 2; ++i) set_row(S.mprev[i], 0.f);
    S.tm = tmbase + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * kTmSlice);
    {
      F4 z[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) set_row(z[i], 0.f);
      tm_wait_st();
      tm_st_rows(S.tm, z, 6);
      tm_st_rows(S.tm + 24, z, 4);
      tm_st_rows(S.tm + 40, z, 4);
      tm_st_rows(S.tm + 72, z, 2);
      tm_st_rows(S.tm + 80, z, 2);
#pragma unroll
      for (int i = 0; i < 4; ++i) set_row(z[i], kFMax);
      tm_st_rows(S.tm + 56, z, 4);
    }
    S.stg = (uint32_t)__cvta_generic_to_shared(smem + kRing * S.ringw) + warp * (kB * 512) + lane * 16;
    cp_async_wait_all();  // no copy of the previous item may still land in the slot
#pragma unroll
    for (int j = 0; j < kB; ++j)
      stage_lane<VEC>(S.stg + j * 512, src + (int64_t)(H - 1 - j) * W + S.x0, p.in, j < H, S.full, incol);
    cp_async_commit();
    S.lrow = src + (int64_t)(H - 1 - kB) * W + S.x0;
    S.orow = dst + (int64_t)(H - 1 - (kB * LG::KFirst - LG::C - 2)) * W + S.x0;

    // iterations with every row inside the frame run the lean body
    const int K = (H + LG::C + 2) / kB + 1;
    const int kLo = (LG::C + 2 + kB - 1) / kB;  // tc0 - 2 >= 0 and tp >= 0
    const int kHi = (H - 2 * kB) / kB;           // t0 + 7 <= H - 1 and tc0 + 3 <= H - 1
    int k = 0;
    for (; k < min(kLo, K); ++k) iterate<VEC, FULL, BLUR, PRE, DENSE, IO, true>(p, S, k);
    for (; k <= kHi; ++k) iterate<VEC, FULL, BLUR, PRE, DENSE, IO, false>(p, S, k);
    for (; k < K; ++k) iterate<VEC, FULL, BLUR, PRE, DENSE, IO, true>(p, S, k);

#ifdef DFC_TIMING
    {
      const long long tz = clock64();
      __syncthreads();  // item-end imbalance (diagnostics build only)
      S.tacc[3] = clock64() - tz;
    }
    if (lane == 0)
      for (int i = 0; i < 6; ++i) p.tim[(blockIdx.x * kNW + warp) * 6 + i] += S.tacc[i];
#endif
    gk = S.gk;
    // ---------------- per-frame flags ----------------
    const unsigned um = __reduce_max_sync(kFull, S.umax);
    S.nin = (unsigned)(S.cin01.x + S.cin01.y + S.cin23.x + S.cin23.y);
    const unsigned nin = __reduce_add_sync(kFull, S.nin);
    const unsigned nout = FULL ? __reduce_add_sync(kFull, (unsigned)__popc(S.outm)) * (unsigned)H
                               : __reduce_add_sync(kFull, S.nout);
    const bool recount = FULL && BLUR != kBlurRaw && !(__uint_as_float(__reduce_min_sync(kFull,
                                                                      __float_as_uint(S.omin))) > kValid);
    const bool he = __any_sync(kFull, S.had_empty);
    const bool se = __any_sync(kFull, S.still_empty);
    const bool eo = IO == 2 && __any_sync(kFull, S.enc_over);
    if (lane == 0) {
      if (!PRE) atomicMax(p.umax + frame, um);  // PRE: multiscale.cu records it
      if (!PRE && nin) atomicAdd(p.vcount + 2 * frame, nin);  // PRE: multiscale.cu counts the inputs
      if (BLUR != kBlurRaw && nout) atomicAdd(p.vcount + 2 * frame + 1, nout);  // raw: the blur tail counts
      if (recount) atomicOr(p.status + frame, kRecountOut);
      if (eo) atomicOr(p.status + frame, DFC_ST_ENCODE);
      if (FULL && he && p.iters) atomicOr(p.iters + frame, 1);
      if (FULL && se) {
        atomicOr(p.status + frame, kNeedsStaged);
        atomicAdd(p.nfallback, 1ull);
      }
    }
    __syncthreads();  // ring reuse by the next item
  }
  tm_wait_st();
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmbase), "n"(kTmCols) : "memory");
}

// Phase 1 of every (item, warp slot) of a round as independent warps (the
// fused kernel's geometry): each warp finds its owned columns' r0 rows and
// records the largest input bit pattern of the rows it scanned (the top rows,
// which phase 2 does not read).  One 32-row block costs a global-load round
// trip; many warps per SM hide it, which the fused kernel's 12 could not.
// First row (from the top, a multiple of 16) of the 16-row group holding the
// warp's first valid pixel (H when none); tracks umax over the rows it reads.
// Stage-4 validity reaches at most 7 rows above it (D_diamond 2 + D5 2 + D7 3),
// so the exact scan can start 8 rows higher with all-empty rows before.
template <int VEC, bool PRE, typename T>
__device__ __forceinline__ int first_valid_group(const T* frame, int H, int W, int x0, unsigned& umax) {
  // clamped columns / rows may add in-frame pixels of the warp's strip to the
  // test: the group found can only be earlier, which is safe for the scan start
  const LaneCols<VEC, T> lc(frame, x0, W);
  int y = 0;
  for (; y < H; y += 16) {
    F4 v[16];
    if (y + 16 <= H) {
      const int64_t off = (int64_t)y * W;
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = lc.row(off + (int64_t)i * W);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = lc.row((int64_t)min(y + i, H - 1) * W);
    }
    float mx = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if constexpr (!PRE) {
        umax = max(max(umax, __float_as_uint(v[i].v[0])), __float_as_uint(v[i].v[1]));
        umax = max(max(umax, __float_as_uint(v[i].v[2])), __float_as_uint(v[i].v[3]));
      }
      mx = fmx3(mx, fmx3(v[i].v[0], v[i].v[1], v[i].v[2]), v[i].v[3]);
    }
    if (__any_sync(kFull, mx > kValid)) break;
  }
  return y;
}

template <int VEC, bool PRE, int IO>
__global__ void __launch_bounds__(128, 4) r0_kernel(const __grid_constant__ Params p) {
  using TIn = typename IoT<IO>::In;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (gw >= p.nframes * p.strips * p.nw) return;  // whole warp
  const int64_t item = gw / p.nw;
  const int64_t frame = item / p.strips;
  Geo g;
  item_geometry((int)(item % p.strips), p, (int)(gw % p.nw), g);
  const int x0 = g.L + 4 * lane;
  unsigned incol = 0, own = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int x = x0 + c;
    incol |= (unsigned)(x >= 0 && x < p.W) << c;
    own |= (unsigned)(x >= g.q0 && x < g.q1) << c;
  }
  const TIn* src = static_cast<const TIn*>(p.in) + frame * (int64_t)p.H * p.W;
  int T0[4];
  unsigned umax = 0;
  const int s0 = first_valid_group<VEC, PRE>(src, p.H, p.W, x0, umax) - 8;
  phase1<VEC, PRE>(src, p, x0, own != 0, incol, T0, umax, s0);
  int32_t* dst = p.t0g + frame * p.W + x0;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (own >> c & 1) dst[c] = T0[c];
  if (!PRE) {
    umax = __reduce_max_sync(kFull, umax);
    if (lane == 0) atomicMax(p.umax + frame, umax);
  }
}

template <int VEC, bool FULL, int BLUR, bool PRE, int DENSE = kLfSparse, int IO = 0>
cudaError_t launch_t(const Params& p, size_t smem, int grid, cudaStream_t s) {
  if constexpr (FULL) {
    const int64_t warps = p.nframes * p.strips * p.nw;
    note_launch();
    r0_kernel<VEC, PRE, IO><<<(unsigned)((warps + 3) / 4), 128, 0, s>>>(p);
  }
  auto k = fused_kernel<VEC, FULL, BLUR, PRE, DENSE, IO>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  note_launch();
  k<<<grid, p.nw * 32, smem, s>>>(p);
  return cudaGetLastError();
}

template <int VEC, bool FULL>
cudaError_t dispatch_blur(int blur, bool pre, const Params& p, size_t smem, int grid, cudaStream_t s) {
  if (pre) {
    if (blur == DFC_BLUR_GAUSSIAN) return launch_t<VEC, FULL, DFC_BLUR_GAUSSIAN, true>(p, smem, grid, s);
    if (blur == DFC_BLUR_NONE) return launch_t<VEC, FULL, DFC_BLUR_NONE, true>(p, smem, grid, s);
    return launch_t<VEC, FULL, kBlurRaw, true>(p, smem, grid, s);
  }
  if (blur == DFC_BLUR_GAUSSIAN) return launch_t<VEC, FULL, DFC_BLUR_GAUSSIAN, false>(p, smem, grid, s);
  if (blur == DFC_BLUR_NONE) return launch_t<VEC, FULL, DFC_BLUR_NONE, false>(p, smem, grid, s);
  return launch_t<VEC, FULL, kBlurRaw, false>(p, smem, grid, s);
}

// DENSE (shared-memory scratch for the dense large fill): FULL mode, wide strips, W % 4 == 0
template <int BLUR>
cudaError_t dispatch_dense(bool pre, const Params& p, size_t smem, int grid, cudaStream_t s) {
  return pre ? launch_t<4, true, BLUR, true, kLfSmemDense>(p, smem, grid, s)
             : launch_t<4, true, BLUR, false, kLfSmemDense>(p, smem, grid, s);
}

// DFC_F_SPARSE (FULL mode, narrow strips): the register-dense large fill
template <int BLUR>
cudaError_t dispatch_regdense(bool pre, const Params& p, size_t smem, int grid, cudaStream_t s) {
  return pre ? launch_t<4, true, BLUR, true, kLfRegDense>(p, smem, grid, s)
             : launch_t<4, true, BLUR, false, kLfRegDense>(p, smem, grid, s);
}

}  // namespace
}  // namespace dfc
