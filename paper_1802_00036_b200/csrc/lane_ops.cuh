// Lane-level building blocks of the streaming kernels (fused.cu, multiscale.cu):
// each lane holds 4 adjacent columns of a row (F4); horizontal neighbours come
// from warp shuffles, vertical windows from rows carried in registers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dfc {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr float kFMax = 3.402823466e38f;
constexpr int kB = 4;  // rows per streaming block

struct F4 {
  float v[4];
};

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float fmx(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ float fmx3(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }
__device__ __forceinline__ float fmn3(float a, float b, float c) { return fminf(fminf(a, b), c); }

struct OpMax {
  static __device__ __forceinline__ float f(float a, float b) { return fmaxf(a, b); }
  static __device__ __forceinline__ float f3(float a, float b, float c) { return fmx3(a, b, c); }
};
struct OpMin {
  static __device__ __forceinline__ float f(float a, float b) { return fminf(a, b); }
  static __device__ __forceinline__ float f3(float a, float b, float c) { return fmn3(a, b, c); }
};

// Row extended by R columns each side: e[i] <-> column x0 - R + i.  Lanes 0
// and 31 read their own registers for the missing neighbour; both are halo
// or out-of-frame lanes whose results are never used.
template <int R>
struct Ext {
  float e[4 + 2 * R];
};

template <int R>
__device__ __forceinline__ Ext<R> ext_row(const F4& a) {
  Ext<R> o;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    o.e[R - 1 - i] = __shfl_up_sync(kFull, a.v[3 - i], 1);
    o.e[R + 4 + i] = __shfl_down_sync(kFull, a.v[i], 1);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) o.e[R + i] = a.v[i];
  return o;
}

template <class Op>
__device__ __forceinline__ F4 hwin2(const Ext<2>& x) {
  F4 o;
  const float p = Op::f3(x.e[2], x.e[3], x.e[4]);
  o.v[0] = Op::f3(p, x.e[0], x.e[1]);
  o.v[1] = Op::f3(p, x.e[1], x.e[5]);
  o.v[2] = Op::f3(p, x.e[5], x.e[6]);
  o.v[3] = Op::f3(Op::f3(x.e[3], x.e[4], x.e[5]), x.e[6], x.e[7]);
  return o;
}

template <class Op>
__device__ __forceinline__ F4 hwin3(const Ext<3>& x) {
  F4 o;
  const float q = Op::f(Op::f3(x.e[3], x.e[4], x.e[5]), x.e[6]);
  const float b = Op::f(x.e[1], x.e[2]);
  const float c2 = Op::f(x.e[7], x.e[8]);
  o.v[0] = Op::f3(q, b, x.e[0]);
  o.v[1] = Op::f3(q, b, x.e[7]);
  o.v[2] = Op::f3(q, x.e[2], c2);
  o.v[3] = Op::f3(q, c2, x.e[9]);
  return o;
}

template <class Op>
__device__ __forceinline__ void vwin2(const F4* in, F4* out) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
#pragma unroll
    for (int j = 0; j < kB; j += 2) {
      const float m = Op::f3(in[j + 1].v[c], in[j + 2].v[c], in[j + 3].v[c]);
      out[j].v[c] = Op::f3(m, in[j].v[c], in[j + 4].v[c]);
      out[j + 1].v[c] = Op::f3(m, in[j + 4].v[c], in[j + 5].v[c]);
    }
  }
}

template <class Op>
__device__ __forceinline__ void vwin3(const F4* in, F4* out) {
  static_assert(kB == 4, "vwin3 assumes 4-row blocks");
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float q = Op::f(Op::f3(in[3].v[c], in[4].v[c], in[5].v[c]), in[6].v[c]);
    const float b = Op::f(in[1].v[c], in[2].v[c]);
    const float c2 = Op::f(in[7].v[c], in[8].v[c]);
    out[0].v[c] = Op::f3(q, b, in[0].v[c]);
    out[1].v[c] = Op::f3(q, b, in[7].v[c]);
    out[2].v[c] = Op::f3(q, in[2].v[c], c2);
    out[3].v[c] = Op::f3(q, c2, in[9].v[c]);
  }
}

__device__ __forceinline__ void set_row(F4& a, float v) {
#pragma unroll
  for (int c = 0; c < 4; ++c) a.v[c] = v;
}

__device__ __forceinline__ void fix_oob(F4& a, unsigned oob, float v) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (oob & (1u << c)) a.v[c] = v;
}

// ---------------------------------------------------------------------------
// global memory access for one lane's 4 columns of a row
// ---------------------------------------------------------------------------
template <int VEC, bool STREAM>
__device__ __forceinline__ F4 load4(const float* row, int x0, int W) {
  F4 r;
  if (x0 >= 0 && x0 + 3 < W) {
    if constexpr (VEC == 4) {
      const float4* a = reinterpret_cast<const float4*>(row + x0);
      const float4 t = STREAM ? __ldcs(a) : __ldg(a);
      r.v[0] = t.x, r.v[1] = t.y, r.v[2] = t.z, r.v[3] = t.w;
    } else if constexpr (VEC == 2) {
      const float2* a = reinterpret_cast<const float2*>(row + x0);
      const float2 u = STREAM ? __ldcs(a) : __ldg(a);
      const float2 w = STREAM ? __ldcs(a + 1) : __ldg(a + 1);
      r.v[0] = u.x, r.v[1] = u.y, r.v[2] = w.x, r.v[3] = w.y;
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) r.v[c] = STREAM ? __ldcs(row + x0 + c) : __ldg(row + x0 + c);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) r.v[c] = (x0 + c >= 0 && x0 + c < W) ? __ldg(row + x0 + c) : 0.0f;
  }
  return r;
}

template <int VEC>
__device__ __forceinline__ void store4(float* row, int x0, const F4& a, unsigned colmask) {
  if (colmask == 0xFu) {
    if constexpr (VEC == 4) {
      __stcs(reinterpret_cast<float4*>(row + x0), make_float4(a.v[0], a.v[1], a.v[2], a.v[3]));
      return;
    } else if constexpr (VEC == 2) {
      __stcs(reinterpret_cast<float2*>(row + x0), make_float2(a.v[0], a.v[1]));
      __stcs(reinterpret_cast<float2*>(row + x0 + 2), make_float2(a.v[2], a.v[3]));
      return;
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (colmask & (1u << c)) __stcs(row + x0 + c, a.v[c]);
}

// q points at the lane's first column of a row
template <int VEC>
__device__ __forceinline__ void store_lane(float* q, const F4& a, unsigned colmask) {
  if (colmask == 0xFu) {
    if constexpr (VEC == 4) {
      __stcs(reinterpret_cast<float4*>(q), make_float4(a.v[0], a.v[1], a.v[2], a.v[3]));
      return;
    } else if constexpr (VEC == 2) {
      __stcs(reinterpret_cast<float2*>(q), make_float2(a.v[0], a.v[1]));
      __stcs(reinterpret_cast<float2*>(q + 2), make_float2(a.v[2], a.v[3]));
      return;
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (colmask & (1u << c)) __stcs(q + c, a.v[c]);
}

}  // namespace
}  // namespace dfc
