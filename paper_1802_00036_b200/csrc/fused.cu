// Fused streaming depth-completion kernel (csrc/fused_impl.cuh): host side --
// layout, workspace, chunked rounds (multiscale stage 2 -> fused -> blur tail)
// and the per-frame status finalize kernel.
#include "fused_impl.cuh"

namespace dfc {

cudaError_t fused_dispatch_vec4(bool full, int blur, bool pre, bool dense, const void* params, size_t smem, int grid,
                                cudaStream_t s);
cudaError_t fused_dispatch_vec2(bool full, int blur, bool pre, bool dense, const void* params, size_t smem, int grid,
                                cudaStream_t s);
cudaError_t fused_dispatch_vec1(bool full, int blur, bool pre, bool dense, const void* params, size_t smem, int grid,
                                cudaStream_t s);
cudaError_t fused_dispatch_raw16(int io, bool full, int blur, const void* params, size_t smem, int grid, cudaStream_t s);

namespace {

// Per-frame status from the input's largest bit pattern; frames whose max is
// suspicious (negative sign, non-finite, >= max_depth) are rescanned.
// vcount[2b] holds the inverted-valid inputs the fused kernel read (every
// pixel once); an input can be valid (> 0.1) but inverted-invalid only when
// md - v <= 0.1, i.e. only if the frame's max already is (md - v is monotone),
// so only such frames (count_in) are recounted here with the plain v > 0.1
// (pipeline.py:138-141), the raw input as raw > 25 (raw / 256 > 0.1).
// Frames whose fused output may hold an empty pixel (kRecountOut, FULL mode)
// get their valid outputs recounted from the stored output.
__device__ void recount_outputs(const void* out_v, int64_t HW, int64_t b, bool out_raw, unsigned* vcount) {
  __shared__ unsigned sc;
  if (threadIdx.x == 0) sc = 0;
  __syncthreads();
  unsigned n = 0;
  if (out_raw) {
    const uint16_t* o = static_cast<const uint16_t*>(out_v) + b * HW;
    for (int64_t i = threadIdx.x; i < HW; i += blockDim.x) n += o[i] > 25u;  // raw / 256 > 0.1
  } else {
    const float* o = static_cast<const float*>(out_v) + b * HW;
    for (int64_t i = threadIdx.x; i < HW; i += blockDim.x) n += o[i] > kValid;
  }
  n = __reduce_add_sync(kFull, n);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(&sc, n);
  __syncthreads();
  if (threadIdx.x == 0) vcount[2 * b + 1] = sc;
}

__global__ void finalize_kernel(const void* __restrict__ in_v, const void* __restrict__ out_v, int64_t HW,
                                const unsigned* __restrict__ umax, uint32_t* status, float md, bool in_raw,
                                bool out_raw, unsigned* vcount, bool count_in) {
  const int64_t b = blockIdx.x;
  if (status[b] & kRecountOut) {  // uniform: every thread reads it before anyone clears it
    recount_outputs(out_v, HW, b, out_raw, vcount);
    if (threadIdx.x == 0) atomicAnd(status + b, ~kRecountOut);
  }
  const unsigned u = umax[b];
  const float uf = __uint_as_float(u);
  const bool rare = count_in && uf > kValid && uf < md && !(__fadd_rn(md, -uf) > kValid);
  if (in_raw) {  // raw / 256 is finite and >= 0: the max decides RANGE and DEGENERATE alone
    if (threadIdx.x == 0 && u >= __float_as_uint(md)) atomicOr(status + b, DFC_ST_RANGE);
    if (threadIdx.x == 0 && u <= __float_as_uint(kValid)) atomicOr(status + b, DFC_ST_DEGENERATE);
    if (!rare) return;
  } else if (u < __float_as_uint(md) && !rare) {
    if (u <= __float_as_uint(kValid) && threadIdx.x == 0) atomicOr(status + b, DFC_ST_DEGENERATE);
    return;
  }
  __shared__ unsigned sb, sv, sn;
  if (threadIdx.x == 0) sb = 0, sv = 0, sn = 0;
  __syncthreads();
  if (in_raw) {  // rare only: recount (raw / 256 > 0.1 <=> raw > 25)
    const uint16_t* src = static_cast<const uint16_t*>(in_v) + b * HW;
    unsigned n = 0;
    for (int64_t i = threadIdx.x; i < HW; i += blockDim.x) n += src[i] > 25u;
    n = __reduce_add_sync(kFull, n);
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(&sn, n);
    __syncthreads();
    if (threadIdx.x == 0) vcount[2 * b] = sn;
    return;
  }
  const float* in = static_cast<const float*>(in_v);
  const float* src = in + b * HW;
  uint32_t bits = 0;
  unsigned n = 0;
  for (int64_t i = threadIdx.x; i < HW; i += blockDim.x) {
    const float v = src[i];
    if (!isfinite(v))
      bits |= DFC_ST_NONFINITE;
    else if (v < 0.0f)
      bits |= DFC_ST_NEGATIVE;
    else if (v >= md)
      bits |= DFC_ST_RANGE;
    n += v > kValid;
  }
  bits = __reduce_or_sync(kFull, bits);
  n = __reduce_add_sync(kFull, n);
  if ((threadIdx.x & 31) == 0) {
    atomicOr(&sb, bits);
    if (n) atomicOr(&sv, 1u), atomicAdd(&sn, n);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t st = sb;
    if (!sv) st |= DFC_ST_DEGENERATE;
    if (st) atomicOr(status + b, st);
    if (count_in) vcount[2 * b] = sn;
  }
}

constexpr size_t kSmemMax = 232448;  // 227 KB opt-in dynamic shared memory per CTA

struct Layout {
  int strips, SW, nw, per_sm;  // per_sm: resident CTAs per SM (1)
  bool dense;
  size_t smem;
};

int host_warps(int o0, int o1, int W) {
  const int p0 = o0 == 0 ? 0 : std::max(0, (o0 - 17) & ~3);
  const int p1 = o1 == W ? W : std::min(W, (o1 + 17 + 3) & ~3);
  int q0 = p0, nw = 0;
  while (q0 < p1) {
    const int L = q0 == 0 ? -4 : q0 - kHalo;
    const int q1 = (p1 == W && L + kLW - 4 >= W) ? W : std::min(p1, L + kLW - kHalo);
    q0 = q1;
    ++nw;
  }
  return nw;
}

Layout layout_for(int W, int strips) {
  Layout L;
  L.strips = strips;
  L.SW = strips == 1 ? W : (((W + strips - 1) / strips) + 3) & ~3;
  L.strips = (W + L.SW - 1) / L.SW;
  L.nw = 0;
  int pwmax = 0;
  for (int s = 0; s < L.strips; ++s) {
    const int o0 = s * L.SW, o1 = std::min(W, o0 + L.SW);
    L.nw = std::max(L.nw, host_warps(o0, o1, W));
    const int p0 = o0 == 0 ? 0 : std::max(0, (o0 - 17) & ~3);
    const int p1 = o1 == W ? W : std::min(W, (o1 + 17 + 3) & ~3);
    pwmax = std::max(pwmax, p1 - p0);
  }
  const int ringw = ring_width(pwmax);
  L.smem = (size_t)kRing * ringw * 4 + (size_t)L.nw * kB * 512;
  // dense large-fill scratch when it fits next to the ring (wide strips; a
  // whole 1216-wide frame's ring leaves no room -- its empties are sparse)
  L.dense = L.smem + (size_t)L.nw * kB * kVC * 4 <= kSmemMax;
  if (L.dense) L.smem += (size_t)L.nw * kB * kVC * 4;
  L.per_sm = 1;
  return L;
}

// One CTA per strip of <= 1248 columns (a whole 1216- or 1242-wide frame).
// Splitting such frames into two 6-warp CTAs per SM measured slower (the
// strip halos and phase 1 are paid twice).
Layout layout(int W) { return layout_for(W, W <= kStripMax ? 1 : (W + 1023) / 1024); }

cudaError_t dispatch(int vec, bool full, int blur, bool pre, int io, const Params& p, size_t smem, int grid,
                     cudaStream_t s) {
  if (io) return fused_dispatch_raw16(io, full, blur, &p, smem, grid, s);  // vec 4, no PRE (fused_supports_raw16)
  const bool dense = p.dense && vec == 4 && full;
  if (vec == 4) return fused_dispatch_vec4(full, blur, pre, dense, &p, smem, grid, s);
  if (vec == 2) return fused_dispatch_vec2(full, blur, pre, false, &p, smem, grid, s);
  return fused_dispatch_vec1(full, blur, pre, false, &p, smem, grid, s);
}

}  // namespace

bool fused_supported(const dfc_config& c, int H, int W) {
  if (c.custom_n > 0 || (c.flags & DFC_F_EXACT_BLUR)) return false;
  if (c.multiscale ? !multiscale_stage2_supported(c)
                   : (c.dilation_shape != DFC_SHAPE_DIAMOND || c.dilation_size != 5))
    return false;
  if (c.closure_size != 5 || c.small_fill_size != 7 || c.large_fill_size != 31) return false;
  // Gaussian-5 and no blur run inside the kernel; every other blur goes
  // through the raw mode and the blur-tail kernel
  const bool direct = c.blur_mode == DFC_BLUR_NONE || (c.blur_mode == DFC_BLUR_GAUSSIAN && c.gaussian_size == 5);
  if (!direct && !blur_tail_supported(c)) return false;
  if (H < 16 || W < 16) return false;
  const Layout L = layout(W);
  return L.nw <= kNW && L.smem <= kSmemMax;
}

bool raw_mode(const dfc_config& c) {
  return !(c.blur_mode == DFC_BLUR_NONE || (c.blur_mode == DFC_BLUR_GAUSSIAN && c.gaussian_size == 5));
}

size_t raw_offset(int64_t B) { return ((16 + (size_t)B * 4) + 255) & ~(size_t)255; }

// Frames per round when intermediate maps go through the workspace (the
// stage-6 map of the raw mode, the stage-2 map of multiscale): every kernel of
// a round (stage 2 -> fused -> blur tail) ramps up and drains once per round, so
// rounds are as long as an 8 GiB budget of maps allows, between 2 and 32 CTA
// waves of a 148-SM B200 (measured on 1024-frame batches against 2-wave
// rounds: config 2 +8 %, config 4 +2 %, config 0 +1.3 %; the maps do not fit L2
// either way).  DFC_RAW_CHUNK sets the items per round for A/B runs.
int64_t round_frames(const dfc_config& c, int64_t B, int H, int W) {
  if (!raw_mode(c) && !c.multiscale) return B;
  const int64_t strips = layout(W).strips;
  const int64_t forced = getenv("DFC_RAW_CHUNK") ? atoll(getenv("DFC_RAW_CHUNK")) : 0;  // read per call: tests set it
  const int64_t lo = (kRawChunk + strips - 1) / strips, hi = (16 * kRawChunk + strips - 1) / strips;
  const int64_t fit = (int64_t)(((size_t)8 << 30) / ((size_t)2 * H * W * 4));
  const int64_t ch = forced ? (forced + strips - 1) / strips : std::max(lo, std::min(hi, fit));
  return B < ch ? B : ch;
}

size_t t0_bytes(const dfc_config& c, int64_t B, int H, int W) {
  return c.fill_mode == DFC_FILL_FULL ? (((size_t)round_frames(c, B, H, W) * W * 4 + 255) & ~(size_t)255) : 0;
}

size_t fused_workspace_bytes(const dfc_config& c, int64_t B, int H, int W) {
  // [0] u64 frames needing the staged path, [8] u32 work counter, [16..) u32 umax[B],
  // then one round of stage-6 maps (raw mode), of stage-2 maps (multiscale) and
  // of per-column r0 rows (FULL)
  const size_t map = (size_t)round_frames(c, B, H, W) * H * W * 4;
  const size_t a = (map + 255) & ~(size_t)255;
  return raw_offset(B) + (raw_mode(c) ? a : 0) + (c.multiscale ? a : 0) + t0_bytes(c, B, H, W) + 256;
}

bool fused_supports_raw16(const dfc_config& c, int H, int W) {
  return fused_supported(c, H, W) && W % 4 == 0 && !c.multiscale;
}

// io 0: float32 in / out; 1: 16-bit KITTI raw in, float32 out; 2: raw in / raw out
cudaError_t launch_fused(const void* in_v, void* out_v, int64_t B, int H, int W, const dfc_config& c,
                         uint32_t* status, int32_t* iters, unsigned* vcount, void* ws, size_t ws_bytes,
                         cudaStream_t s, int io) {
  const float* in = static_cast<const float*>(in_v);  // io 0; raw pointers below go through in_v / out_v
  float* out = static_cast<float*>(out_v);
  const size_t isz = io ? 2 : 4, osz = io == 2 ? 2 : 4;
  if (ws_bytes < fused_workspace_bytes(c, B, H, W)) return cudaErrorInvalidValue;
  Params p;
  p.in = in;
  p.out = out;
  p.nframes = B;
  p.H = H;
  p.W = W;
  const Layout L = layout(W);
  p.strips = L.strips;
  p.SW = L.SW;
  p.nw = L.nw;
  p.dense = L.dense;
  p.regdense = (c.flags & DFC_F_SPARSE) ? 1 : 0;
  p.md = c.max_depth;
  {
    // only the in-kernel Gaussian (size 5) uses these taps; every other blur
    // mode (any gaussian_size up to 63) leaves them zero
    double w[5] = {0, 0, 0, 0, 0}, sum = 0;
    if (c.blur_mode == DFC_BLUR_GAUSSIAN && c.gaussian_size == 5) {
      for (int i = -2; i <= 2; ++i)
        w[i + 2] = std::exp(-(double)(i * i) / (2.0 * c.gaussian_sigma * c.gaussian_sigma));
      for (int i = 0; i < 5; ++i) sum += w[i];
    }
    for (int i = 0; i < 5; ++i) p.gw[i] = sum > 0 ? (float)(w[i] / sum) : 0.f;
    for (int i = 0; i < 6; ++i)
      p.gh[i] = make_float2(i < 5 ? p.gw[i] : 0.f, i > 0 ? p.gw[i - 1] : 0.f);
  }
  p.status = status;
  p.iters = iters;
  char* w8 = static_cast<char*>(ws);
  p.nfallback = reinterpret_cast<unsigned long long*>(w8);
#ifdef DFC_TIMING
  p.tim = reinterpret_cast<unsigned long long*>(getenv("DFC_TIM_PTR") ? strtoull(getenv("DFC_TIM_PTR"), nullptr, 0) : 0);
#endif
  p.work = reinterpret_cast<unsigned*>(w8 + 8);
  p.umax = reinterpret_cast<unsigned*>(w8 + 16);
  cudaError_t e = cudaMemsetAsync(ws, 0, 16 + (size_t)B * 4, s);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(vcount, 0, (size_t)B * 8, s)) != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int vec = (W % 4 == 0) ? 4 : ((W % 2 == 0) ? 2 : 1);
  const bool full = c.fill_mode == DFC_FILL_FULL;
  const bool raw = raw_mode(c);
  const int blur = raw ? kBlurRaw : c.blur_mode;
  const int64_t HW = (int64_t)H * W;
  const bool pre = c.multiscale != 0;
  const int64_t chunk = round_frames(c, B, H, W);
  const size_t map = (((size_t)chunk * HW * 4) + 255) & ~(size_t)255;
  float* tmp = raw ? reinterpret_cast<float*>(w8 + raw_offset(B)) : nullptr;
  float* s2 = pre ? reinterpret_cast<float*>(w8 + raw_offset(B) + (raw ? map : 0)) : nullptr;
  p.t0g = full ? reinterpret_cast<int32_t*>(w8 + raw_offset(B) + (raw ? map : 0) + (pre ? map : 0)) : nullptr;
  unsigned* umax0 = p.umax;
  std::vector<int32_t> offs[3];
  const int32_t* op[3];
  int on[3];
  if (pre) {
    const int shp[3] = {c.near_shape, c.med_shape, c.far_shape};
    const int siz[3] = {c.near_size, c.med_size, c.far_size};
    for (int k = 0; k < 3; ++k) {
      bool full;
      offs[k] = kernel_offsets(shp[k], siz[k], &full);
      op[k] = offs[k].data();
      on[k] = (int)offs[k].size() / 2;
    }
  }
  for (int64_t f0 = 0; f0 < B; f0 += chunk) {
    const int64_t C = B - f0 < chunk ? B - f0 : chunk;
    // the stage-2 kernel's item queue is the word after the fused kernel's (zeroed with it above)
    if (pre && f0 > 0 && (e = cudaMemsetAsync(p.work + 1, 0, 4, s)) != cudaSuccess) return e;
    if (pre && (e = launch_multiscale_stage2(in + f0 * HW, s2, C, H, W, c, op, on, umax0 + f0, vcount + 2 * f0,
                                             p.work + 1, s)) != cudaSuccess)
      return e;
    char* out_c = static_cast<char*>(out_v) + f0 * HW * osz;
    p.in = pre ? (const void*)s2 : (const void*)(static_cast<const char*>(in_v) + f0 * HW * isz);
    p.out = raw ? (void*)tmp : (void*)out_c;
    p.nframes = C;
    p.status = status + f0;
    p.iters = iters ? iters + f0 : nullptr;
    p.umax = umax0 + f0;
    p.vcount = vcount + 2 * f0;
    if (f0 > 0 && (e = cudaMemsetAsync(p.work, 0, 4, s)) != cudaSuccess) return e;
    const int64_t items = C * L.strips;
    const int64_t slots = (int64_t)sms * L.per_sm;
    const int grid = (int)(items < slots ? items : slots);
    // raw mode: the fused kernel writes float32 stage-6 maps; the blur tail encodes
    e = dispatch(vec, full, blur, pre, raw && io == 2 ? 1 : io, p, L.smem, grid, s);
    if (e != cudaSuccess) return e;
    if (raw && (e = launch_blur_tail(tmp, out_c, C, H, W, c, io == 2, status + f0, vcount + 2 * f0, s)) !=
                   cudaSuccess)
      return e;
  }
  note_launch();
  finalize_kernel<<<(unsigned)B, 256, 0, s>>>(in_v, out_v, HW, umax0, status, c.max_depth, io != 0, io == 2, vcount,
                                              !pre);
  return cudaGetLastError();
}

}  // namespace dfc
