// extern "C" entry points of libdfc.so (include/dfc.h), argument checking,
// and the staged (one op per launch) pipeline used when the fused kernel does
// not cover a configuration and for frames that need more than one
// large-fill iteration.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "dfc_common.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define DFC_CK(expr)                                                                          \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) return fail(DFC_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

bool odd3(int v) { return v >= 3 && (v % 2) == 1; }

int check_shape(int64_t B, int32_t H, int32_t W) {
  if (B < 0) return fail(DFC_E_INVALID, "batch size must be >= 0");
  if (H < 1 || W < 1) return fail(DFC_E_INVALID, "depth map dimensions must be >= 1, got " +
                                                      std::to_string(W) + "x" + std::to_string(H));
  if ((int64_t)H * W > (int64_t)1 << 31)
    return fail(DFC_E_INVALID, "depth map dimensions " + std::to_string(W) + "x" + std::to_string(H) +
                                   " exceed supported size");
  return DFC_OK;
}

// PipelineConfig.__post_init__ (pipeline.py:71-89)
int check_config(const dfc_config& c) {
  const struct {
    const char* name;
    int v;
  } sizes[] = {{"dilation_size", c.dilation_size},     {"closure_size", c.closure_size},
               {"small_fill_size", c.small_fill_size}, {"large_fill_size", c.large_fill_size},
               {"median_size", c.median_size},         {"gaussian_size", c.gaussian_size},
               {"bilateral_size", c.bilateral_size}};
  for (auto& s : sizes)
    if (!odd3(s.v))
      return fail(DFC_E_INVALID, std::string(s.name) + " must be an odd integer >= 3, got " + std::to_string(s.v));
  if (c.large_fill_max_iters < 1) return fail(DFC_E_INVALID, "large_fill_max_iters must be >= 1");
  if (!(c.gaussian_sigma > 0)) return fail(DFC_E_INVALID, "gaussian_sigma must be positive");
  if (!(c.bilateral_sigma_value > 0) || !(c.bilateral_sigma_space > 0))
    return fail(DFC_E_INVALID, "bilateral sigmas must be positive");
  if (c.dilation_shape < 0 || c.dilation_shape > 3) return fail(DFC_E_INVALID, "unknown kernel shape");
  if (c.blur_mode < 0 || c.blur_mode > 5) return fail(DFC_E_INVALID, "unknown blur mode");
  if (c.fill_mode < 0 || c.fill_mode > 1) return fail(DFC_E_INVALID, "unknown fill mode");
  if (!std::isfinite(c.max_depth) || !(c.max_depth > 0.1f)) return fail(DFC_E_INVALID, "max_depth must be > 0.1");
  if (c.gaussian_size > 63) return fail(DFC_E_UNSUPPORTED, "gaussian_size > 63 not supported");
  if (c.custom_n < 0 || (c.custom_n > 0 && !c.custom_offsets)) return fail(DFC_E_INVALID, "bad custom kernel");
  if (c.custom_n > 4096) return fail(DFC_E_UNSUPPORTED, "custom kernel with more than 4096 taps");
  for (int t = 0; t < 2 * c.custom_n; ++t)
    if (c.custom_offsets[t] < -127 || c.custom_offsets[t] > 127)
      return fail(DFC_E_UNSUPPORTED, "custom kernel offset magnitude > 127");
  if (c.multiscale) {
    const int ks[3][2] = {{c.near_shape, c.near_size}, {c.med_shape, c.med_size}, {c.far_shape, c.far_size}};
    for (auto& k : ks) {
      if (k[0] < 0 || k[0] > 3) return fail(DFC_E_INVALID, "unknown kernel shape");
      if (!odd3(k[1])) return fail(DFC_E_INVALID, "bin kernel size must be an odd integer >= 3");
    }
    if (!(c.bin_edge_near < c.bin_edge_far)) return fail(DFC_E_INVALID, "bin edges must be increasing");
  }
  return DFC_OK;
}

// pipeline._fit_to_frame (:241-254) -- also applied to the multiscale bin kernels
dfc_config fit_to_frame(const dfc_config& c, int H, int W) {
  dfc_config o = c;
  const int limit = 2 * (H < W ? H : W) + 1;
  const int fit = limit > 3 ? limit : 3;
  int* fields[] = {&o.dilation_size, &o.closure_size, &o.small_fill_size, &o.large_fill_size,
                   &o.near_size,     &o.med_size,     &o.far_size};
  for (int* f : fields)
    if (*f > limit) *f = fit;
  return o;
}

// ---- staged pipeline -------------------------------------------------------

struct StagedBufs {
  float *a, *b, *c, *d, *e;  // e follows d: (d,e) doubles as a float64 scratch
  int64_t *n_valid, *counts;
  unsigned long long* total;
  void* lf;  // large-fill loop scratch (dfc::large_fill_scratch_bytes)
};

// frames per staged round: about 64 MB of frames (at most 65535: grid.y limits)
int64_t staged_chunk(int64_t B, int H, int W) {
  const int64_t per = (int64_t)H * W * 4;
  int64_t c = ((int64_t)64 << 20) / per;
  if (c < 1) c = 1;
  if (c > 65535) c = 65535;
  return c < B ? c : B;
}

size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

size_t staged_bytes(int64_t chunk, int H, int W) {
  if (chunk <= 0) return 0;
  const size_t f = align256((size_t)chunk * H * W * 4);
  return 5 * f + align256(chunk * 8) * 2 + 256 + align256(dfc::large_fill_scratch_bytes(chunk));
}

// fused-path fallback: frames flagged by the fused kernel are gathered into
// [in][out] maps of one staged chunk, with their indices, statuses and counts
size_t fallback_bytes(int64_t chunk, int H, int W) {
  if (chunk <= 0) return 0;
  return 2 * align256((size_t)chunk * H * W * 4) + align256(chunk * 8) + 2 * align256(chunk * 4) +
         align256(chunk * 8);
}

StagedBufs carve_staged(void* ws, int64_t chunk, int H, int W) {
  char* p = static_cast<char*>(ws);
  const size_t f = align256((size_t)chunk * H * W * 4);
  StagedBufs s;
  s.a = (float*)p;
  s.b = (float*)(p + f);
  s.c = (float*)(p + 2 * f);
  s.d = (float*)(p + 3 * f);
  s.e = (float*)(p + 4 * f);
  s.n_valid = (int64_t*)(p + 5 * f);
  s.counts = (int64_t*)(p + 5 * f + align256(chunk * 8));
  s.total = (unsigned long long*)(p + 5 * f + 2 * align256(chunk * 8));
  s.lf = p + 5 * f + 2 * align256(chunk * 8) + 256;
  return s;
}

cudaError_t dilate_any(const float* in, float* out, float* tmp, int64_t B, int H, int W, int shape, int size,
                       bool is_min, cudaStream_t s) {
  bool full;
  auto offs = dfc::kernel_offsets(shape, size, &full);
  if (full) {
    cudaError_t e = dfc::launch_line_minmax(in, tmp, B, H, W, size / 2, is_min, 1, s);
    if (e != cudaSuccess) return e;
    return dfc::launch_line_minmax(tmp, out, B, H, W, size / 2, is_min, 0, s);
  }
  return dfc::launch_offsets_minmax(in, out, B, H, W, offs.data(), (int)offs.size() / 2, is_min, s);
}

int gaussian_weights(int size, double sigma, double* w) {
  // morphology.gaussian_weights (:128-133)
  const int r = size / 2;
  double sum = 0.0;
  for (int i = -r; i <= r; ++i) {
    w[i + r] = std::exp(-(double)(i * i) / (2.0 * sigma * sigma));
  }
  for (int i = 0; i < size; ++i) sum += w[i];  // np.sum pairwise == sequential for <= 8 terms
  for (int i = 0; i < size; ++i) w[i] /= sum;
  return size;
}

int run_staged(const float* in, float* out, int64_t B, int H, int W, const dfc_config& c, uint32_t* status,
               int32_t* iters, unsigned* vcount, void* ws, size_t ws_bytes, cudaStream_t s) {
  const int64_t chunk = staged_chunk(B, H, W);
  if (!ws || ws_bytes < staged_bytes(chunk, H, W)) return fail(DFC_E_WORKSPACE, "workspace too small (staged)");
  const int64_t HW = (int64_t)H * W;
  const bool full = c.fill_mode == DFC_FILL_FULL;
  const bool exact = (c.flags & DFC_F_EXACT_BLUR) != 0;
  double gw[64];
  gaussian_weights(c.gaussian_size, c.gaussian_sigma, gw);
  for (int64_t f0 = 0; f0 < B; f0 += chunk) {
    const int64_t C = B - f0 < chunk ? B - f0 : chunk;
    StagedBufs q = carve_staged(ws, chunk, H, W);
    const float* x = in + f0 * HW;
    float* y = out + f0 * HW;
    uint32_t* st = status + f0;
    int32_t* it = iters ? iters + f0 : nullptr;
    const int64_t n = C * HW;
    DFC_CK(cudaMemsetAsync(q.n_valid, 0, C * 8, s));
    DFC_CK(dfc::launch_validate(x, HW, C, st, q.n_valid, s));
    DFC_CK(dfc::launch_finalize_status(q.n_valid, st, C, s));
    // 1. invert
    DFC_CK(dfc::launch_invert(x, q.a, HW, C, c.max_depth, st, s));
    // 2. shaped dilation (or depth-binned multiscale dilation)
    if (!c.multiscale && c.custom_n > 0) {
      DFC_CK(dfc::launch_offsets_minmax(q.a, q.b, C, H, W, c.custom_offsets, c.custom_n, false, s));
    } else if (!c.multiscale) {
      DFC_CK(dilate_any(q.a, q.b, q.d, C, H, W, c.dilation_shape, c.dilation_size, false, s));
    } else {
      const float inf = INFINITY;
      const float lo[3] = {-inf, c.bin_edge_near, c.bin_edge_far};
      const float hi[3] = {c.bin_edge_near, c.bin_edge_far, inf};
      const int shp[3] = {c.near_shape, c.med_shape, c.far_shape};
      const int siz[3] = {c.near_size, c.med_size, c.far_size};
      for (int k = 0; k < 3; ++k) {
        DFC_CK(dfc::launch_bin_select(x, q.a, q.c, n, lo[k], hi[k], s));
        DFC_CK(dilate_any(q.c, k == 0 ? q.b : q.e, q.d, C, H, W, shp[k], siz[k], false, s));
        if (k > 0) DFC_CK(dfc::launch_max2(q.b, q.e, q.b, n, s));
      }
    }
    // 3. close (FULL closure_size)
    DFC_CK(dilate_any(q.b, q.c, q.d, C, H, W, DFC_SHAPE_FULL, c.closure_size, false, s));
    DFC_CK(dilate_any(q.c, q.b, q.d, C, H, W, DFC_SHAPE_FULL, c.closure_size, true, s));
    // 4. small masked fill
    DFC_CK(dilate_any(q.b, q.c, q.d, C, H, W, DFC_SHAPE_FULL, c.small_fill_size, false, s));
    DFC_CK(dfc::launch_masked_fill(q.b, q.c, q.a, n, s));
    float* cur = q.a;
    float* spare = q.b;
    if (full) {
      // 5. extend to top
      DFC_CK(dfc::launch_extend_to_top(q.a, q.b, C, H, W, s));
      cur = q.b;
      spare = q.a;
      // 6. large fill, iterated per frame while empties remain: device-gated
      //    tiled iterations, one host check per group of iterations
      if (dfc::large_fill_tiled_supported(c.large_fill_size / 2)) {
        DFC_CK(dfc::launch_large_fill_loop(cur, spare, C, H, W, c.large_fill_size / 2, c.large_fill_max_iters, it,
                                           q.lf, s));
      } else
      for (int k = 0; k < c.large_fill_max_iters; ++k) {
        DFC_CK(cudaMemsetAsync(q.counts, 0, C * 8, s));
        DFC_CK(cudaMemsetAsync(q.total, 0, 8, s));
        DFC_CK(dfc::launch_count_empty(cur, HW, C, q.counts, s));
        DFC_CK(dfc::launch_iter_update(q.counts, it, C, q.total, s));
        unsigned long long total = 0;
        DFC_CK(cudaMemcpyAsync(&total, q.total, 8, cudaMemcpyDeviceToHost, s));
        DFC_CK(cudaStreamSynchronize(s));
        if (total == 0) break;
        DFC_CK(dilate_any(cur, q.c, q.d, C, H, W, DFC_SHAPE_FULL, c.large_fill_size, false, s));
        DFC_CK(dfc::launch_masked_fill(cur, q.c, cur, n, s));
      }
    }
    // 7 + 8. blur stage (pipeline._blur_stage :206-238) and invert back, one tiled kernel
    if (dfc::blur_tail_supported(c)) {
      DFC_CK(dfc::launch_blur_tail(cur, y, C, H, W, c, false, st, nullptr, s));
      if (vcount) DFC_CK(dfc::launch_valid_counts(y, HW, C, q.n_valid, vcount + 2 * f0, s));
      continue;
    }
    // exact float64 blurs: one op per launch
    const int bm = c.blur_mode;
    const bool partial = !full;
    if (bm == DFC_BLUR_MEDIAN || bm == DFC_BLUR_MEDIAN_BILATERAL || bm == DFC_BLUR_MEDIAN_GAUSSIAN) {
      DFC_CK(dfc::launch_median(cur, q.c, C, H, W, c.median_size, s));
      if (partial) DFC_CK(dfc::launch_reimpose(q.c, cur, q.c, n, s));
      std::swap(cur, q.c);
      if (cur == q.c) std::swap(q.c, spare);
    }
    if (bm == DFC_BLUR_GAUSSIAN || bm == DFC_BLUR_MEDIAN_GAUSSIAN) {
      DFC_CK(dfc::launch_gauss_line(cur, q.d, C, H, W, gw, c.gaussian_size, 1, exact, false, exact, s));
      DFC_CK(dfc::launch_gauss_line((const float*)q.d, spare, C, H, W, gw, c.gaussian_size, 0, exact, exact,
                                    false, s));
      if (partial) DFC_CK(dfc::launch_reimpose(spare, cur, spare, n, s));
      std::swap(cur, spare);
    }
    if (bm == DFC_BLUR_BILATERAL || bm == DFC_BLUR_MEDIAN_BILATERAL) {
      DFC_CK(dfc::launch_bilateral(cur, spare, C, H, W, c.bilateral_size, c.bilateral_sigma_value,
                                   c.bilateral_sigma_space, exact, s));
      if (partial) DFC_CK(dfc::launch_reimpose(spare, cur, spare, n, s));
      std::swap(cur, spare);
    }
    // 8. invert back
    DFC_CK(dfc::launch_invert(cur, y, HW, C, c.max_depth, nullptr, s));
    if (vcount) DFC_CK(dfc::launch_valid_counts(y, HW, C, q.n_valid, vcount + 2 * f0, s));
  }
  return DFC_OK;
}

// workspace layout: [fused region][staged region][valid counts [B][2] u32]
struct WsLayout {
  size_t fused, staged, cnt, total;
  int64_t chunk;
  bool use_fused;
};

WsLayout ws_layout(const dfc_config& c, int64_t B, int H, int W) {
  WsLayout L;
  L.use_fused = !(c.flags & DFC_F_FORCE_STAGED) && dfc::fused_supported(c, H, W);
  L.chunk = staged_chunk(B, H, W);
  if (L.use_fused) {
    L.fused = align256(dfc::fused_workspace_bytes(c, B, H, W));
    // flagged frames are gathered and finished a staged chunk at a time
    L.staged = staged_bytes(L.chunk > 0 ? L.chunk : 1, H, W) + fallback_bytes(L.chunk > 0 ? L.chunk : 1, H, W);
  } else {
    L.fused = 0;
    L.staged = staged_bytes(L.chunk > 0 ? L.chunk : 1, H, W);
  }
  L.cnt = align256((size_t)B * 8);
  L.total = L.fused + L.staged + L.cnt;
  return L;
}

}  // namespace

// ===========================================================================
extern "C" {

int dfc_abi_version(void) { return DFC_ABI_VERSION; }

unsigned long long dfc_kernel_launches(void) { return dfc::g_kernel_launches.load(); }

const char* dfc_last_error_string(void) { return g_err.c_str(); }

int dfc_config_init(dfc_config* c) {
  if (!c) return fail(DFC_E_INVALID, "null config");
  std::memset(c, 0, sizeof(*c));
  c->dilation_shape = DFC_SHAPE_DIAMOND;
  c->dilation_size = 5;
  c->closure_size = 5;
  c->small_fill_size = 7;
  c->large_fill_size = 31;
  c->large_fill_max_iters = 100;
  c->blur_mode = DFC_BLUR_MEDIAN_GAUSSIAN;
  c->median_size = 5;
  c->gaussian_size = 5;
  c->bilateral_size = 5;
  c->gaussian_sigma = 1.1;
  c->bilateral_sigma_value = 1.5;
  c->bilateral_sigma_space = 2.0;
  c->fill_mode = DFC_FILL_FULL;
  c->max_depth = 100.0f;
  c->multiscale = 0;
  c->bin_edge_near = 15.0f;
  c->bin_edge_far = 30.0f;
  c->near_shape = DFC_SHAPE_FULL;
  c->near_size = 7;
  c->med_shape = DFC_SHAPE_DIAMOND;
  c->med_size = 7;
  c->far_shape = DFC_SHAPE_DIAMOND;
  c->far_size = 5;
  c->flags = 0;
  return DFC_OK;
}

size_t dfc_workspace_bytes(const dfc_config* cfg, int64_t B, int32_t H, int32_t W) {
  if (!cfg || check_shape(B, H, W) != DFC_OK || check_config(*cfg) != DFC_OK) return 0;
  const dfc_config c = fit_to_frame(*cfg, H, W);
  return ws_layout(c, B, H, W).total;
}

int dfc_fill_batch(const float* in, float* out, int64_t B, int32_t H, int32_t W, const dfc_config* cfg,
                   uint32_t* frame_status, int32_t* large_fill_iters, void* workspace, size_t ws_bytes,
                   void* stream) {
  if (!cfg) return fail(DFC_E_INVALID, "null config");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  rc = check_config(*cfg);
  if (rc) return rc;
  if (B == 0) return DFC_OK;
  if (!in || !out || !frame_status) return fail(DFC_E_INVALID, "null buffer");
  const dfc_config c = fit_to_frame(*cfg, H, W);
  const WsLayout L = ws_layout(c, B, H, W);
  if (!workspace || ws_bytes < L.total)
    return fail(DFC_E_WORKSPACE, "workspace too small: need " + std::to_string(L.total) + " bytes");
  cudaStream_t s = as_stream(stream);
  DFC_CK(cudaMemsetAsync(frame_status, 0, B * 4, s));
  if (large_fill_iters) DFC_CK(cudaMemsetAsync(large_fill_iters, 0, B * 4, s));
  unsigned* vcount = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + L.fused + L.staged);
  if (!L.use_fused) {
    return run_staged(in, out, B, H, W, c, frame_status, large_fill_iters, vcount,
                      static_cast<char*>(workspace) + L.fused, L.staged, s);
  }
  DFC_CK(dfc::launch_fused(in, out, B, H, W, c, frame_status, large_fill_iters, vcount, workspace, L.fused, s));
  if (c.flags & DFC_F_NO_FINISH) return DFC_OK;
  return dfc_fill_finish(in, out, B, H, W, cfg, frame_status, large_fill_iters, workspace, ws_bytes, stream);
}

int dfc_fill_finish(const float* in, float* out, int64_t B, int32_t H, int32_t W, const dfc_config* cfg,
                    uint32_t* frame_status, int32_t* large_fill_iters, void* workspace, size_t ws_bytes,
                    void* stream) {
  if (!cfg) return fail(DFC_E_INVALID, "null config");
  const dfc_config c = fit_to_frame(*cfg, H, W);
  const WsLayout L = ws_layout(c, B, H, W);
  if (!L.use_fused || B == 0) return DFC_OK;
  if (!workspace || ws_bytes < L.total) return fail(DFC_E_WORKSPACE, "workspace too small");
  cudaStream_t s = as_stream(stream);
  // fused.cu keeps a device counter of frames that need the staged path at the
  // start of its workspace region.
  unsigned long long nfb = 0;
  DFC_CK(cudaMemcpyAsync(&nfb, workspace, 8, cudaMemcpyDeviceToHost, s));
  DFC_CK(cudaStreamSynchronize(s));
  if (nfb == 0) return DFC_OK;
  std::vector<uint32_t> st(B);
  DFC_CK(cudaMemcpyAsync(st.data(), frame_status, B * 4, cudaMemcpyDeviceToHost, s));
  DFC_CK(cudaStreamSynchronize(s));
  std::vector<int64_t> idx;
  for (int64_t b = 0; b < B; ++b)
    if (st[b] & 0x200u) idx.push_back(b);  // internal "needs staged" bit set by the fused kernel
  // the flagged frames, a staged chunk at a time: gather -> staged pipeline
  // (device-gated large-fill loop) -> scatter outputs, statuses and counts
  const int64_t HW = (int64_t)H * W;
  const int64_t chunk = L.chunk;
  char* sw = static_cast<char*>(workspace) + L.fused;
  const size_t sb = staged_bytes(chunk, H, W);
  const size_t f = align256((size_t)chunk * HW * 4);
  float* g_in = reinterpret_cast<float*>(sw + sb);
  float* g_out = reinterpret_cast<float*>(sw + sb + f);
  int64_t* g_idx = reinterpret_cast<int64_t*>(sw + sb + 2 * f);
  uint32_t* g_st = reinterpret_cast<uint32_t*>(sw + sb + 2 * f + align256(chunk * 8));
  int32_t* g_it = reinterpret_cast<int32_t*>(sw + sb + 2 * f + align256(chunk * 8) + align256(chunk * 4));
  unsigned* g_vc = reinterpret_cast<unsigned*>(sw + sb + 2 * f + align256(chunk * 8) + 2 * align256(chunk * 4));
  unsigned* vcount = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + L.fused + L.staged);
  for (size_t i0 = 0; i0 < idx.size(); i0 += (size_t)chunk) {
    const int64_t C = std::min<int64_t>(chunk, (int64_t)idx.size() - (int64_t)i0);
    DFC_CK(cudaMemcpyAsync(g_idx, idx.data() + i0, C * 8, cudaMemcpyHostToDevice, s));
    DFC_CK(dfc::launch_gather_frames(in, g_in, HW, g_idx, C, false, s));
    DFC_CK(cudaMemsetAsync(g_st, 0, C * 4, s));
    DFC_CK(cudaMemsetAsync(g_it, 0, C * 4, s));
    int rc = run_staged(g_in, g_out, C, H, W, c, g_st, g_it, g_vc, sw, sb, s);
    if (rc) return rc;
    DFC_CK(dfc::launch_gather_frames(g_out, out, HW, g_idx, C, true, s));
    DFC_CK(dfc::launch_scatter_status(g_st, g_it, g_vc, g_idx, C, frame_status, large_fill_iters, vcount,
                                      DFC_ST_FALLBACK, s));
    DFC_CK(cudaStreamSynchronize(s));  // idx (host) is reused by the next chunk's copy
  }
  return DFC_OK;
}

int dfc_fill_counts(const dfc_config* cfg, int64_t B, int32_t H, int32_t W, const void* workspace, size_t ws_bytes,
                    uint32_t* valid_counts, void* stream) {
  if (!cfg) return fail(DFC_E_INVALID, "null config");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (B == 0) return DFC_OK;
  const dfc_config c = fit_to_frame(*cfg, H, W);
  const WsLayout L = ws_layout(c, B, H, W);
  if (!workspace || ws_bytes < L.total || !valid_counts) return fail(DFC_E_INVALID, "bad workspace or counts buffer");
  DFC_CK(cudaMemcpyAsync(valid_counts, static_cast<const char*>(workspace) + L.fused + L.staged, (size_t)B * 8,
                         cudaMemcpyDeviceToDevice, as_stream(stream)));
  return DFC_OK;
}

size_t dfc_op_workspace_bytes(int64_t B, int32_t H, int32_t W) { return (size_t)B * H * W * 8; }

static int op_prologue(const void* in, const void* out, int64_t B, int32_t H, int32_t W) {
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (B > 0 && (!in || !out)) return fail(DFC_E_INVALID, "null buffer");
  return DFC_OK;
}

static int box_op(const float* in, float* out, int64_t B, int32_t H, int32_t W, int32_t radius, void* ws,
                  size_t wsb, void* stream, bool is_min) {
  int rc = op_prologue(in, out, B, H, W);
  if (rc || B == 0) return rc;
  if (radius < 0) return fail(DFC_E_INVALID, "radius must be >= 0");
  if (!ws || wsb < (size_t)B * H * W * 4) return fail(DFC_E_WORKSPACE, "workspace too small");
  cudaStream_t s = as_stream(stream);
  DFC_CK(dfc::launch_line_minmax(in, (float*)ws, B, H, W, radius, is_min, 1, s));
  DFC_CK(dfc::launch_line_minmax((float*)ws, out, B, H, W, radius, is_min, 0, s));
  return DFC_OK;
}

int dfc_box_max(const float* in, float* out, int64_t B, int32_t H, int32_t W, int32_t radius, void* ws, size_t wsb,
                void* stream) {
  return box_op(in, out, B, H, W, radius, ws, wsb, stream, false);
}

int dfc_box_min(const float* in, float* out, int64_t B, int32_t H, int32_t W, int32_t radius, void* ws, size_t wsb,
                void* stream) {
  return box_op(in, out, B, H, W, radius, ws, wsb, stream, true);
}

static int offs_op(const float* in, float* out, int64_t B, int32_t H, int32_t W, const int32_t* offsets, int32_t n,
                   void* stream, bool is_min) {
  int rc = op_prologue(in, out, B, H, W);
  if (rc || B == 0) return rc;
  if (!offsets || n < 1) return fail(DFC_E_INVALID, "empty offset list");
  if (n > 4096) return fail(DFC_E_UNSUPPORTED, "more than 4096 offsets");
  for (int t = 0; t < 2 * n; ++t)
    if (offsets[t] < -127 || offsets[t] > 127) return fail(DFC_E_UNSUPPORTED, "offset magnitude > 127");
  DFC_CK(dfc::launch_offsets_minmax(in, out, B, H, W, offsets, n, is_min, as_stream(stream)));
  return DFC_OK;
}

int dfc_offsets_max(const float* in, float* out, int64_t B, int32_t H, int32_t W, const int32_t* offsets,
                    int32_t n, void* stream) {
  return offs_op(in, out, B, H, W, offsets, n, stream, false);
}

int dfc_offsets_min(const float* in, float* out, int64_t B, int32_t H, int32_t W, const int32_t* offsets,
                    int32_t n, void* stream) {
  return offs_op(in, out, B, H, W, offsets, n, stream, true);
}

int dfc_median(const float* in, float* out, int64_t B, int32_t H, int32_t W, int32_t size, void* stream) {
  int rc = op_prologue(in, out, B, H, W);
  if (rc || B == 0) return rc;
  if (!odd3(size)) return fail(DFC_E_INVALID, "window size must be odd and >= 3, got " + std::to_string(size));
  DFC_CK(dfc::launch_median(in, out, B, H, W, size, as_stream(stream)));
  return DFC_OK;
}

int dfc_gaussian_separable(const float* in, float* out, int64_t B, int32_t H, int32_t W, const double* weights,
                           int32_t k, int32_t exact, void* ws, size_t wsb, void* stream) {
  int rc = op_prologue(in, out, B, H, W);
  if (rc || B == 0) return rc;
  if (!weights || k < 1 || k > 64) return fail(DFC_E_INVALID, "weights must have 1..64 taps");
  const size_t need = (size_t)B * H * W * (exact ? 8 : 4);
  if (!ws || wsb < need) return fail(DFC_E_WORKSPACE, "workspace too small");
  cudaStream_t s = as_stream(stream);
  DFC_CK(dfc::launch_gauss_line(in, ws, B, H, W, weights, k, 1, exact != 0, false, exact != 0, s));
  DFC_CK(dfc::launch_gauss_line((const float*)ws, out, B, H, W, weights, k, 0, exact != 0, exact != 0, false, s));
  return DFC_OK;
}

int dfc_bilateral(const float* in, float* out, int64_t B, int32_t H, int32_t W, int32_t size, double sigma_value,
                  double sigma_space, int32_t exact, void* stream) {
  int rc = op_prologue(in, out, B, H, W);
  if (rc || B == 0) return rc;
  if (!odd3(size)) return fail(DFC_E_INVALID, "window size must be odd and >= 3, got " + std::to_string(size));
  if (!(sigma_value > 0) || !(sigma_space > 0)) return fail(DFC_E_INVALID, "bilateral sigmas must be positive");
  DFC_CK(dfc::launch_bilateral(in, out, B, H, W, size, sigma_value, sigma_space, exact != 0, as_stream(stream)));
  return DFC_OK;
}

int dfc_invert(const float* in, float* out, int64_t B, int32_t H, int32_t W, float offset, uint32_t* frame_status,
               void* stream) {
  int rc = op_prologue(in, out, B, H, W);
  if (rc || B == 0) return rc;
  DFC_CK(dfc::launch_invert(in, out, (int64_t)H * W, B, offset, frame_status, as_stream(stream)));
  return DFC_OK;
}

int dfc_validate(const float* in, int64_t B, int32_t H, int32_t W, uint32_t* frame_status, int64_t* n_valid,
                 void* stream) {
  int rc = op_prologue(in, frame_status, B, H, W);
  if (rc || B == 0) return rc;
  cudaStream_t s = as_stream(stream);
  if (n_valid) {
    DFC_CK(cudaMemsetAsync(n_valid, 0, B * 8, s));
  }
  DFC_CK(dfc::launch_validate(in, (int64_t)H * W, B, frame_status, n_valid, s));
  if (n_valid) DFC_CK(dfc::launch_finalize_status(n_valid, frame_status, B, s));
  return DFC_OK;
}

int dfc_masked_fill(const float* cur, const float* dilated, float* out, int64_t B, int32_t H, int32_t W,
                    void* stream) {
  int rc = op_prologue(cur, out, B, H, W);
  if (rc || B == 0) return rc;
  if (!dilated) return fail(DFC_E_INVALID, "null buffer");
  DFC_CK(dfc::launch_masked_fill(cur, dilated, out, B * H * (int64_t)W, as_stream(stream)));
  return DFC_OK;
}

int dfc_extend_to_top(const float* in, float* out, int64_t B, int32_t H, int32_t W, void* stream) {
  int rc = op_prologue(in, out, B, H, W);
  if (rc || B == 0) return rc;
  if (in == out) return fail(DFC_E_INVALID, "extend_to_top cannot run in place");
  DFC_CK(dfc::launch_extend_to_top(in, out, B, H, W, as_stream(stream)));
  return DFC_OK;
}

int dfc_count_empty(const float* in, int64_t B, int32_t H, int32_t W, int64_t* counts, void* stream) {
  int rc = op_prologue(in, counts, B, H, W);
  if (rc || B == 0) return rc;
  cudaStream_t s = as_stream(stream);
  DFC_CK(cudaMemsetAsync(counts, 0, B * 8, s));
  DFC_CK(dfc::launch_count_empty(in, (int64_t)H * W, B, counts, s));
  return DFC_OK;
}

int dfc_reimpose(const float* blurred, const float* mask_src, float* out, int64_t B, int32_t H, int32_t W,
                 void* stream) {
  int rc = op_prologue(blurred, out, B, H, W);
  if (rc || B == 0) return rc;
  if (!mask_src) return fail(DFC_E_INVALID, "null buffer");
  DFC_CK(dfc::launch_reimpose(blurred, mask_src, out, B * H * (int64_t)W, as_stream(stream)));
  return DFC_OK;
}

// ---- KITTI 16-bit raw at the boundary ------------------------------------
// Fused path: the fused kernel reads raw rows (and, for Gaussian / no blur,
// writes raw rows); frames needing more large-fill iterations are decoded one
// at a time and finished by the staged path.  Other configurations decode a
// chunk into the workspace, run the float32 pipeline and encode.
static int64_t raw16_chunk(int64_t B) { return B < 64 ? B : 64; }

size_t dfc_workspace_bytes_raw16(const dfc_config* cfg, int64_t B, int32_t H, int32_t W) {
  if (!cfg || check_shape(B, H, W) != DFC_OK || check_config(*cfg) != DFC_OK) return 0;
  const dfc_config c = fit_to_frame(*cfg, H, W);
  const size_t HW4 = align256((size_t)H * W * 4);
  if (!(c.flags & DFC_F_FORCE_STAGED) && dfc::fused_supports_raw16(c, H, W))
    return ws_layout(c, B, H, W).total + 2 * HW4;
  const int64_t ch = raw16_chunk(B > 0 ? B : 1);
  return ws_layout(c, ch, H, W).total + 2 * (size_t)ch * HW4;
}

int dfc_fill_batch_raw16(const uint16_t* raw_in, void* out, int32_t out_raw, int64_t B, int32_t H, int32_t W,
                         const dfc_config* cfg, uint32_t* frame_status, int32_t* large_fill_iters, void* workspace,
                         size_t ws_bytes, void* stream) {
  if (!cfg) return fail(DFC_E_INVALID, "null config");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  rc = check_config(*cfg);
  if (rc) return rc;
  if (B == 0) return DFC_OK;
  if (!raw_in || !out || !frame_status) return fail(DFC_E_INVALID, "null buffer");
  const dfc_config c = fit_to_frame(*cfg, H, W);
  const size_t need = dfc_workspace_bytes_raw16(cfg, B, H, W);
  if (!workspace || ws_bytes < need)
    return fail(DFC_E_WORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes");
  cudaStream_t s = as_stream(stream);
  const int64_t HW = (int64_t)H * W;
  const size_t HW4 = align256((size_t)HW * 4);
  char* ws = static_cast<char*>(workspace);
  dfc_config cf = c;
  cf.flags &= ~(uint32_t)DFC_F_NO_FINISH;
  if (!(c.flags & DFC_F_FORCE_STAGED) && dfc::fused_supports_raw16(c, H, W)) {
    const WsLayout L = ws_layout(c, B, H, W);
    float* fin = reinterpret_cast<float*>(ws + L.total);
    float* fout = reinterpret_cast<float*>(ws + L.total + HW4);
    DFC_CK(cudaMemsetAsync(frame_status, 0, B * 4, s));
    if (large_fill_iters) DFC_CK(cudaMemsetAsync(large_fill_iters, 0, B * 4, s));
    unsigned* vcount = reinterpret_cast<unsigned*>(ws + L.fused + L.staged);
    DFC_CK(dfc::launch_fused(raw_in, out, B, H, W, c, frame_status, large_fill_iters, vcount, ws, L.fused, s,
                             out_raw ? 2 : 1));
    if (c.flags & DFC_F_NO_FINISH) return DFC_OK;  // the caller re-runs frames with status bit 0x200
    unsigned long long nfb = 0;
    DFC_CK(cudaMemcpyAsync(&nfb, ws, 8, cudaMemcpyDeviceToHost, s));
    DFC_CK(cudaStreamSynchronize(s));
    if (nfb == 0) return DFC_OK;
    std::vector<uint32_t> st(B);
    DFC_CK(cudaMemcpyAsync(st.data(), frame_status, B * 4, cudaMemcpyDeviceToHost, s));
    DFC_CK(cudaStreamSynchronize(s));
    for (int64_t b = 0; b < B; ++b) {
      if (!(st[b] & 0x200u)) continue;  // the fused kernel's "needs staged" bit
      DFC_CK(cudaMemsetAsync(frame_status + b, 0, 4, s));
      if (large_fill_iters) DFC_CK(cudaMemsetAsync(large_fill_iters + b, 0, 4, s));
      DFC_CK(dfc::launch_decode_raw16(raw_in + b * HW, fin, HW, s));
      float* dst = out_raw ? fout : static_cast<float*>(out) + b * HW;
      rc = run_staged(fin, dst, 1, H, W, c, frame_status + b, large_fill_iters ? large_fill_iters + b : nullptr,
                      vcount + 2 * b, ws + L.fused, L.staged, s);
      if (rc) return rc;
      if (out_raw) DFC_CK(dfc::launch_encode_raw16(fout, static_cast<uint16_t*>(out) + b * HW, HW, HW, frame_status + b, s));
      DFC_CK(dfc::launch_or_status(frame_status + b, DFC_ST_FALLBACK, s));
    }
    return DFC_OK;
  }
  const int64_t ch = raw16_chunk(B);
  const size_t inner = ws_layout(c, ch, H, W).total;
  float* fin = reinterpret_cast<float*>(ws + inner);
  float* fout = reinterpret_cast<float*>(ws + inner + (size_t)ch * HW4);
  for (int64_t f0 = 0; f0 < B; f0 += ch) {
    const int64_t C = B - f0 < ch ? B - f0 : ch;
    DFC_CK(dfc::launch_decode_raw16(raw_in + f0 * HW, fin, C * HW, s));
    float* dst = out_raw ? fout : static_cast<float*>(out) + f0 * HW;
    rc = dfc_fill_batch(fin, dst, C, H, W, &cf, frame_status + f0, large_fill_iters ? large_fill_iters + f0 : nullptr,
                        ws, inner, stream);
    if (rc) return rc;
    if (out_raw)
      DFC_CK(dfc::launch_encode_raw16(fout, static_cast<uint16_t*>(out) + f0 * HW, HW, C * HW, frame_status + f0, s));
  }
  return DFC_OK;
}

int dfc_decode_raw16(const uint16_t* raw, float* depth, int64_t n, void* stream) {
  if (n < 0) return fail(DFC_E_INVALID, "negative size");
  if (n == 0) return DFC_OK;
  if (!raw || !depth) return fail(DFC_E_INVALID, "null buffer");
  DFC_CK(dfc::launch_decode_raw16(raw, depth, n, as_stream(stream)));
  return DFC_OK;
}

int dfc_encode_raw16(const float* depth, uint16_t* raw, int64_t B, int64_t n_per_frame, uint32_t* frame_status,
                     void* stream) {
  if (B < 0 || n_per_frame < 0) return fail(DFC_E_INVALID, "negative size");
  if (B == 0 || n_per_frame == 0) return DFC_OK;
  if (!depth || !raw) return fail(DFC_E_INVALID, "null buffer");
  DFC_CK(dfc::launch_encode_raw16(depth, raw, n_per_frame, B * n_per_frame, frame_status, as_stream(stream)));
  return DFC_OK;
}

int dfc_error_sums(const float* pred, const float* gt, int64_t B, int32_t H, int32_t W, double* sums, int64_t* counts,
                   void* stream) {
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (B == 0) return DFC_OK;
  if (!pred || !gt || !sums || !counts) return fail(DFC_E_INVALID, "null buffer");
  DFC_CK(dfc::launch_error_sums(pred, gt, B, (int64_t)H * W, sums, counts, as_stream(stream)));
  return DFC_OK;
}

int dfc_error_map(const float* pred, const float* gt, float* out, int64_t B, int32_t H, int32_t W, void* stream) {
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (B == 0) return DFC_OK;
  if (!pred || !gt || !out) return fail(DFC_E_INVALID, "null buffer");
  DFC_CK(dfc::launch_error_map(pred, gt, out, B * H * (int64_t)W, as_stream(stream)));
  return DFC_OK;
}

int dfc_colormap(const float* values, uint8_t* rgb, int64_t n, double range_min, double range_max, void* stream) {
  if (!(range_max > range_min))
    return fail(DFC_E_INVALID, "degenerate range [" + std::to_string(range_min) + ", " + std::to_string(range_max) + "]");
  if (n < 0) return fail(DFC_E_INVALID, "negative size");
  if (n == 0) return DFC_OK;
  if (!values || !rgb) return fail(DFC_E_INVALID, "null buffer");
  DFC_CK(dfc::launch_colormap(values, rgb, n, range_min, range_max, as_stream(stream)));
  return DFC_OK;
}

}  // extern "C"
