/*
 * dfc.h -- C ABI of the B200 depth-completion library (libdfc.so).
 *
 * Drop-in boundary for the reference package `depthfill` (arXiv 1802.00036
 * reference, /root/reference/pkg/src/depthfill).  Plain pointers and sizes
 * only; no C++ or torch types.  All device pointers are CUDA device memory
 * (e.g. torch.Tensor.data_ptr()); `stream` is a cudaStream_t passed as void*
 * (NULL = legacy default stream).  Frames are row-major float32 [B][H][W],
 * contiguous (frame stride H*W).
 *
 * Conventions
 *   - every function returns DFC_OK (0) or a negative DFC_E_* code;
 *     dfc_last_error_string() returns the message for the calling thread;
 *   - calls are stream-ordered and asynchronous unless documented otherwise;
 *   - the caller owns every buffer; the library keeps no mutable global state
 *     besides the per-thread error string and immutable constant tables.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/depthfill):
 *   dfc_box_max/min           _native_ops.pyx:31-155, _numpy_ops.py:17-29
 *   dfc_offsets_max/min       _native_ops.pyx:158-195, _numpy_ops.py:32-49
 *   dfc_median                _native_ops.pyx:198-296 (+ _native.py:23-26), _numpy_ops.py:52-58
 *   dfc_gaussian_separable    _native_ops.pyx:299-337, _numpy_ops.py:61-73
 *   dfc_bilateral             _native_ops.pyx:340-369, _numpy_ops.py:76-95
 *   dfc_invert                depth_core.py:132-156 (invert / invert_back / _flip)
 *   dfc_validate              depth_core.py:58-75 + pipeline.py:136-140
 *   dfc_masked_fill           morphology.py:70-78 (the np.where part)
 *   dfc_extend_to_top         morphology.py:81-96
 *   dfc_count_empty           pipeline.py:181 (any(v <= 0.1) per frame)
 *   dfc_reimpose              pipeline.py:212-214
 *   dfc_fill_batch            pipeline.py:118-203 (complete / complete_with_stats),
 *                             batched; covers fill_in_fast and fill_in_multiscale
 *   dfc_fill_batch_raw16      kitti_io.py:36-66 read_depth_png / write_depth_png value
 *                             conversion fused at the boundary of dfc_fill_batch
 *   dfc_decode_raw16          kitti_io.py:53 (raw.astype(f32) / f32(256))
 *   dfc_encode_raw16          kitti_io.py:60-65 (rint(f64(d) * 256) clipped, < 256 m check)
 *   dfc_error_sums            metrics.py:119-137 (_error_sums, per frame; MetricsAccumulator sums them)
 *   dfc_error_map             metrics.py:101-108 (error_map)
 *   dfc_colormap              kitti_io.py:69-85 (write_colormap_png pixel values; PNG encoding stays on the host)
 */
#ifndef DFC_H_
#define DFC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFC_ABI_VERSION 1

/* return codes */
#define DFC_OK 0
#define DFC_E_INVALID (-1)     /* bad argument (maps to ValueError) */
#define DFC_E_CUDA (-2)        /* CUDA runtime error */
#define DFC_E_WORKSPACE (-3)   /* workspace missing or too small */
#define DFC_E_UNSUPPORTED (-4) /* configuration not supported */

/* per-frame status bits written by dfc_validate / dfc_fill_batch */
#define DFC_ST_NONFINITE 0x1u   /* ValueError "depth values must be finite"   (depth_core.py:68-69) */
#define DFC_ST_NEGATIVE 0x2u    /* ValueError "depth values must be non-negative" (depth_core.py:70-71) */
#define DFC_ST_DEGENERATE 0x4u  /* DegenerateInputError (pipeline.py:138-140) */
#define DFC_ST_RANGE 0x8u       /* DepthRangeError (depth_core.py:152-155) */
#define DFC_ST_ENCODE 0x10u     /* ValueError "depth values must be < 256 m to be encodable" (kitti_io.py:60-61) */
#define DFC_ST_FALLBACK 0x100u  /* informational: frame was finished by the staged path */

/* kernel shapes (kernels.py:15-19) */
#define DFC_SHAPE_FULL 0
#define DFC_SHAPE_CIRCLE 1
#define DFC_SHAPE_CROSS 2
#define DFC_SHAPE_DIAMOND 3

/* blur modes (pipeline.py:30-36) */
#define DFC_BLUR_NONE 0
#define DFC_BLUR_BILATERAL 1
#define DFC_BLUR_MEDIAN 2
#define DFC_BLUR_MEDIAN_BILATERAL 3
#define DFC_BLUR_GAUSSIAN 4
#define DFC_BLUR_MEDIAN_GAUSSIAN 5

/* fill modes (pipeline.py:39-41) */
#define DFC_FILL_FULL 0
#define DFC_FILL_PARTIAL 1

/* dfc_config.flags */
#define DFC_F_FORCE_STAGED 0x1u /* never use the fused kernel */
#define DFC_F_EXACT_BLUR 0x2u   /* fp64 blurs in the reference's operation order */
#define DFC_F_NO_FINISH 0x4u    /* dfc_fill_batch does not synchronize; call dfc_fill_finish */
#define DFC_F_SPARSE 0x8u       /* performance hint, results unchanged: frames with many empty pixels after the
                                   small fill (about <= 2 % valid inputs) -- the fused kernel's register-dense
                                   large fill (without it, dense frames run ~2 % faster) */

/* PipelineConfig (pipeline.py:50-89) + inversion offset + multiscale bins. */
typedef struct dfc_config {
  int32_t dilation_shape; /* DFC_SHAPE_* */
  int32_t dilation_size;
  int32_t closure_size;
  int32_t small_fill_size;
  int32_t large_fill_size;
  int32_t large_fill_max_iters;
  int32_t blur_mode; /* DFC_BLUR_* */
  int32_t median_size;
  int32_t gaussian_size;
  int32_t bilateral_size;
  double gaussian_sigma;
  double bilateral_sigma_value;
  double bilateral_sigma_space;
  int32_t fill_mode; /* DFC_FILL_* */
  float max_depth;   /* depth_core.INVERSION_OFFSET; BASELINE "max_depth" */
  /* fill_in_multiscale: depth-binned stage-2 dilation */
  int32_t multiscale;                 /* 0 = fill_in_fast, 1 = binned */
  float bin_edge_near, bin_edge_far;  /* near: d<=near, medium: near<d<=far, far: d>far */
  int32_t near_shape, near_size;
  int32_t med_shape, med_size;
  int32_t far_shape, far_size;
  uint32_t flags; /* DFC_F_* */
  /* optional arbitrary stage-2 footprint ("custom kernel"): n (dy,dx) int32
   * pairs in host memory; when n > 0 it replaces dilation_shape/size. */
  int32_t custom_n;
  const int32_t* custom_offsets;
} dfc_config;

/* ---- library ------------------------------------------------------------ */
int dfc_abi_version(void);
const char* dfc_last_error_string(void);
/* Number of kernels this library has launched in the process (diagnostics). */
unsigned long long dfc_kernel_launches(void);
/* Fill *cfg with the reference defaults (pipeline.py:52-69, max_depth 100). */
int dfc_config_init(dfc_config* cfg);

/* ---- fused pipeline (pipeline.complete over a batch) --------------------- */
/* Workspace bytes dfc_fill_batch needs for this config and shape. */
size_t dfc_workspace_bytes(const dfc_config* cfg, int64_t B, int32_t H, int32_t W);
/* Complete B frames.  frame_status[B] (device, uint32) receives DFC_ST_* bits;
 * large_fill_iters[B] (device, int32, may be NULL) the per-frame iteration
 * count of RunStats.large_fill_iterations.  Frames with error bits set have
 * unspecified output.  Unless DFC_F_NO_FINISH is set, the call synchronizes
 * `stream` once to run the staged fallback for the (rare) frames that need
 * more than one large-fill iteration. */
int dfc_fill_batch(const float* in, float* out, int64_t B, int32_t H, int32_t W, const dfc_config* cfg,
                   uint32_t* frame_status, int32_t* large_fill_iters, void* workspace, size_t ws_bytes,
                   void* stream);
/* Second half of dfc_fill_batch when DFC_F_NO_FINISH was given (synchronizes). */
int dfc_fill_finish(const float* in, float* out, int64_t B, int32_t H, int32_t W, const dfc_config* cfg,
                    uint32_t* frame_status, int32_t* large_fill_iters, void* workspace, size_t ws_bytes,
                    void* stream);
/* RunStats' density counters (pipeline.py:138-141, 192-202) of the last
 * dfc_fill_batch (+ dfc_fill_finish) run with this workspace, config and shape:
 * valid_counts[B][2] (device, uint32) = pixels > 0.1 in the input and in the
 * output of each frame.  They are counted inside the fused read / store
 * passes (density = count / (H * W)); enqueued on `stream` (no sync). */
int dfc_fill_counts(const dfc_config* cfg, int64_t B, int32_t H, int32_t W, const void* workspace, size_t ws_bytes,
                    uint32_t* valid_counts, void* stream);

/* ---- operator surface (_native_ops / _numpy_ops), batched --------------- */
/* Workspace for the separable ops (box max/min, gaussian): B*H*W*8 bytes. */
size_t dfc_op_workspace_bytes(int64_t B, int32_t H, int32_t W);
int dfc_box_max(const float* in, float* out, int64_t B, int32_t H, int32_t W, int32_t radius, void* workspace,
                size_t ws_bytes, void* stream);
int dfc_box_min(const float* in, float* out, int64_t B, int32_t H, int32_t W, int32_t radius, void* workspace,
                size_t ws_bytes, void* stream);
/* offsets: host pointer to n (dy,dx) int32 pairs */
int dfc_offsets_max(const float* in, float* out, int64_t B, int32_t H, int32_t W, const int32_t* offsets,
                    int32_t n, void* stream);
int dfc_offsets_min(const float* in, float* out, int64_t B, int32_t H, int32_t W, const int32_t* offsets,
                    int32_t n, void* stream);
int dfc_median(const float* in, float* out, int64_t B, int32_t H, int32_t W, int32_t size, void* stream);
/* weights: host pointer to k float64 taps; exact != 0 selects fp64 in the reference order */
int dfc_gaussian_separable(const float* in, float* out, int64_t B, int32_t H, int32_t W, const double* weights,
                           int32_t k, int32_t exact, void* workspace, size_t ws_bytes, void* stream);
int dfc_bilateral(const float* in, float* out, int64_t B, int32_t H, int32_t W, int32_t size, double sigma_value,
                  double sigma_space, int32_t exact, void* stream);

/* ---- stage kernels -------------------------------------------------------- */
/* _flip: out = v > 0.1f ? offset - v : 0; status |= DFC_ST_RANGE if any v >= offset */
int dfc_invert(const float* in, float* out, int64_t B, int32_t H, int32_t W, float offset, uint32_t* frame_status,
               void* stream);
/* finite / non-negative / degenerate checks; n_valid[B] (int64, may be NULL) */
int dfc_validate(const float* in, int64_t B, int32_t H, int32_t W, uint32_t* frame_status, int64_t* n_valid,
                 void* stream);
/* out = cur > 0.1f ? cur : dilated */
int dfc_masked_fill(const float* cur, const float* dilated, float* out, int64_t B, int32_t H, int32_t W,
                    void* stream);
int dfc_extend_to_top(const float* in, float* out, int64_t B, int32_t H, int32_t W, void* stream);
/* counts[B] (int64) = number of pixels with v <= 0.1f */
int dfc_count_empty(const float* in, int64_t B, int32_t H, int32_t W, int64_t* counts, void* stream);
/* out = mask_src > 0.1f ? blurred : 0 */
int dfc_reimpose(const float* blurred, const float* mask_src, float* out, int64_t B, int32_t H, int32_t W,
                 void* stream);

/* ---- KITTI 16-bit depth PNG values at the boundary ----
 * raw_in: [B][H][W] uint16, depth = raw / 256 m, raw 0 = empty.
 * out: float32 depth (out_raw == 0) or uint16 raw (out_raw != 0, rint(depth * 256)
 * clipped to [0, 65535]; frames with an output >= 256 m get DFC_ST_ENCODE).
 * Same config, status and iteration semantics as dfc_fill_batch.  Frames that
 * need more than one large-fill iteration are finished inside the call unless
 * DFC_F_NO_FINISH is set: then (fused path only) they keep status bit 0x200 and
 * the caller re-runs them, e.g. with DFC_F_FORCE_STAGED. */
size_t dfc_workspace_bytes_raw16(const dfc_config* cfg, int64_t B, int32_t H, int32_t W);
int dfc_fill_batch_raw16(const uint16_t* raw_in, void* out, int32_t out_raw, int64_t B, int32_t H, int32_t W,
                         const dfc_config* cfg, uint32_t* frame_status, int32_t* large_fill_iters, void* workspace,
                         size_t ws_bytes, void* stream);
/* depth = raw / 256 (exact), n elements */
int dfc_decode_raw16(const uint16_t* raw, float* depth, int64_t n, void* stream);
/* raw = rint(depth * 256) clipped; frame_status[b] |= DFC_ST_ENCODE if any depth >= 256 (may be NULL) */
int dfc_encode_raw16(const float* depth, uint16_t* raw, int64_t B, int64_t n_per_frame, uint32_t* frame_status,
                     void* stream);

/* ---- error metrics vs ground truth ----
 * Over pixels where pred and gt are both > 0.1f: sums[b][0..3] (device, float64) =
 * sum err^2, sum |err|, sum (1/d - 1/g)^2, sum |1/d - 1/g| (err = d - g, meters);
 * counts[b][0] = such pixels, counts[b][1] = gt-valid pixels left empty by pred. */
int dfc_error_sums(const float* pred, const float* gt, int64_t B, int32_t H, int32_t W, double* sums, int64_t* counts,
                   void* stream);
/* out = |f64(pred) - f64(gt)| (float32) where both are valid, else 0 */
int dfc_error_map(const float* pred, const float* gt, float* out, int64_t B, int32_t H, int32_t W, void* stream);
/* rgb[n][3] (uint8) = the blue -> cyan -> green -> yellow -> red ramp of clip((v - lo) / (hi - lo), 0, 1),
 * black where v == 0; DFC_E_INVALID unless hi > lo */
int dfc_colormap(const float* values, uint8_t* rgb, int64_t n, double range_min, double range_max, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DFC_H_ */
