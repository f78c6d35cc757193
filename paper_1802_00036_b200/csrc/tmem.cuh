// Tensor-memory helpers: per-thread 32x32b loads / stores of carried rows.
// The streaming kernels (fused_impl.cuh, multiscale.cu) keep the rows each
// stage carries from one 4-row block to the next in TMEM instead of
// registers: TMEM is otherwise idle here (no MMA), and off the register file
// the carries no longer stay live across the whole block.  A thread reaches
// its own TMEM lane (lane quarter = warp % 4); rows are 4 consecutive columns.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lane_ops.cuh"

namespace dfc {
namespace {

__device__ __forceinline__ void tm_alloc(uint32_t smem_slot, int cols) {
  // one warp; the base address lands in shared memory
  if (cols == 128)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_slot) : "memory");
  else
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_slot) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tm_dealloc(uint32_t base, int cols) {
  if (cols == 128)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(base) : "memory");
  else
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(base) : "memory");
}

__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

template <int N>
__device__ __forceinline__ void tm_ld(uint32_t a, float* v);
template <>
__device__ __forceinline__ void tm_ld<16>(uint32_t a, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(a)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tm_ld<8>(uint32_t a, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(a)
               : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void tm_st(uint32_t a, const float* v);
template <>
__device__ __forceinline__ void tm_st<16>(uint32_t a, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(a),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}
template <>
__device__ __forceinline__ void tm_st<8>(uint32_t a, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(a),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
}
// c5 (6 rows x 4 columns) at columns 0..23, gc (4 rows x 4) at 24..39 of the warp's slice
__device__ __forceinline__ void tm_ld_rows(uint32_t a, F4* rows, int n) {
  float v[24];
  if (n == 6) {
    tm_ld<16>(a, v);
    tm_ld<8>(a + 16, v + 16);
  } else if (n == 4) {
    tm_ld<16>(a, v);
  } else {
    tm_ld<8>(a, v);
  }
  tm_wait_ld();
#pragma unroll
  for (int i = 0; i < 6; ++i)
    if (i < n) rows[i] = F4{{v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]}};
}
__device__ __forceinline__ void tm_st_rows(uint32_t a, const F4* rows, int n) {
  float v[24];
#pragma unroll
  for (int i = 0; i < 6; ++i)
    if (i < n)
#pragma unroll
      for (int c = 0; c < 4; ++c) v[4 * i + c] = rows[i].v[c];
  if (n == 6) {
    tm_st<16>(a, v);
    tm_st<8>(a + 16, v + 16);
  } else if (n == 4) {
    tm_st<16>(a, v);
  } else {
    tm_st<8>(a, v);
  }
}

}  // namespace
}  // namespace dfc
