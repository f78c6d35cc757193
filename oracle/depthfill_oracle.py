"""CPU oracle for the depth-completion hot path -- TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy restatement of the reference package
``depthfill`` (``/root/reference/pkg/src/depthfill``).  It exists so that the
tests, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg have a
checker that runs on a box without ``/root/reference``.  The product path
(``paper_1802_00036_b200``) never imports it.

Pinning: every function here is checked bit-for-bit against outputs of the
reference itself (``tests/golden/make_golden.py`` imports the reference with
its numpy backend and stores the results under ``tests/golden/``), see
``tests/test_oracle_golden.py``.

Semantics notes:
* validity is the float32 compare ``v > float32(0.1)`` (numpy-2 weak scalars),
* inversion is ``where(valid, float32(offset) - v, 0)`` in float32,
* max/min filters use replicate borders, which for these (orthogonally convex)
  kernels equals the clipped window,
* the Gaussian and bilateral blurs accumulate in float64 in the reference's
  numpy order and round to float32 once.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from enum import Enum

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

# depth_core.py:20,25
VALIDITY_THRESHOLD = np.float32(0.1)
INVERSION_OFFSET = 100.0


class EncodingError(ValueError):
    """depth_core.py:38-39"""


class DepthRangeError(ValueError):
    """depth_core.py:42-43"""


class DegenerateInputError(ValueError):
    """pipeline.py:44-45"""


# ----------------------------------------------------------------------------
# depth_core
# ----------------------------------------------------------------------------

def validate(values: np.ndarray) -> np.ndarray:
    """DepthMap.__post_init__ checks (depth_core.py:58-75), same order."""
    arr = np.asarray(values)
    if arr.ndim != 2:
        raise ValueError(f"depth map must be 2-D, got shape {arr.shape}")
    h, w = arr.shape
    if h < 1 or w < 1:
        raise ValueError(f"depth map dimensions must be >= 1, got {w}x{h}")
    arr = np.ascontiguousarray(arr, dtype=np.float32)
    if not np.isfinite(arr).all():
        raise ValueError("depth values must be finite")
    if (arr < 0).any():
        raise ValueError("depth values must be non-negative")
    return arr


def valid_mask(values: np.ndarray) -> np.ndarray:
    """depth_core.py:151,161 -- float32 compare against 0.1f."""
    return values > VALIDITY_THRESHOLD


def flip(values: np.ndarray, offset: float = INVERSION_OFFSET) -> np.ndarray:
    """depth_core._flip (depth_core.py:150-156); used by invert and invert_back."""
    off = np.float32(offset)
    valid = values > VALIDITY_THRESHOLD
    if (values >= off).any():
        raise DepthRangeError(f"values must be < {offset} to be invertible")
    return np.where(valid, off - values, np.float32(0.0)).astype(np.float32)


# ----------------------------------------------------------------------------
# kernels.py
# ----------------------------------------------------------------------------

class KernelShape(Enum):
    """kernels.py:15-19"""

    FULL = "full"
    CIRCLE = "circle"
    CROSS = "cross"
    DIAMOND = "diamond"


def make_kernel(shape: KernelShape, size: int) -> np.ndarray:
    """kernels.py:45-71 -- boolean k x k footprint."""
    size = int(size)
    if size < 3 or size % 2 == 0:
        raise ValueError(f"kernel size must be odd and >= 3, got {size}")
    r = size // 2
    d = np.arange(-r, r + 1)
    dx, dy = np.meshgrid(d, d)
    shape = KernelShape(shape)
    if shape is KernelShape.FULL:
        return np.ones((size, size), dtype=bool)
    if shape is KernelShape.DIAMOND:
        return np.abs(dx) + np.abs(dy) <= r
    if shape is KernelShape.CROSS:
        return (dx == 0) | (dy == 0)
    return 4 * (dx * dx + dy * dy) <= size * size


def kernel_offsets(bits: np.ndarray) -> np.ndarray:
    """kernels.py:74-78 -- (n,2) int32 (dy,dx) in row-major scan order."""
    r = bits.shape[0] // 2
    return np.ascontiguousarray(np.argwhere(bits).astype(np.int32) - r)


# ----------------------------------------------------------------------------
# operator surface (_numpy_ops.py / _native_ops.pyx)
# ----------------------------------------------------------------------------

def box_max(values: np.ndarray, radius: int) -> np.ndarray:
    """_numpy_ops.box_max (:17-24): separable (2r+1) max, replicate border."""
    k = 2 * radius + 1
    p = np.pad(values, ((0, 0), (radius, radius)), mode="edge")
    out = sliding_window_view(p, k, axis=1).max(axis=-1)
    p = np.pad(out, ((radius, radius), (0, 0)), mode="edge")
    out = sliding_window_view(p, k, axis=0).max(axis=-1)
    return np.ascontiguousarray(out, dtype=np.float32)


def box_min(values: np.ndarray, radius: int) -> np.ndarray:
    """_numpy_ops.box_min (:27-29)."""
    return -box_max(-values, radius)


def offsets_max(values: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """_numpy_ops.offsets_max (:32-45): max over (dy,dx) offsets, replicate."""
    h, w = values.shape
    ry = int(np.abs(offsets[:, 0]).max())
    rx = int(np.abs(offsets[:, 1]).max())
    p = np.pad(values, ((ry, ry), (rx, rx)), mode="edge")
    out = None
    for dy, dx in offsets:
        win = p[ry + dy: ry + dy + h, rx + dx: rx + dx + w]
        out = win.copy() if out is None else np.maximum(out, win)
    return np.ascontiguousarray(out, dtype=np.float32)


def offsets_min(values: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """_numpy_ops.offsets_min (:48-49)."""
    return -offsets_max(-values, offsets)


def median_filter(values: np.ndarray, size: int) -> np.ndarray:
    """_numpy_ops.median_filter (:52-58): exact median of size*size replicate
    samples (odd count, so the median is an element of the window)."""
    h, w = values.shape
    r = size // 2
    p = np.pad(values, r, mode="edge")
    win = sliding_window_view(p, (size, size)).reshape(h, w, size * size)
    mid = (size * size) // 2
    return np.ascontiguousarray(np.partition(win, mid, axis=-1)[..., mid], dtype=np.float32)


def gaussian_weights(size: int, sigma: float) -> np.ndarray:
    """morphology.gaussian_weights (:128-133), float64."""
    r = size // 2
    i = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-(i * i) / (2.0 * sigma * sigma))
    return w / w.sum()


def gaussian_separable(values: np.ndarray, weights: np.ndarray) -> np.ndarray:
    """_numpy_ops.gaussian_separable (:61-73): float64, horizontal then
    vertical, taps in index order, separate multiply and add."""
    h, w = values.shape
    r = len(weights) // 2
    p = np.pad(values.astype(np.float64), ((0, 0), (r, r)), mode="edge")
    tmp = np.zeros((h, w), dtype=np.float64)
    for t, wt in enumerate(weights):
        tmp += wt * p[:, t: t + w]
    p = np.pad(tmp, ((r, r), (0, 0)), mode="edge")
    out = np.zeros((h, w), dtype=np.float64)
    for t, wt in enumerate(weights):
        out += wt * p[t: t + h, :]
    return out.astype(np.float32)


def bilateral_filter(values: np.ndarray, size: int, sigma_value: float,
                     sigma_space: float) -> np.ndarray:
    """_numpy_ops.bilateral_filter (:76-95): float64, one exp per tap of the
    summed exponent, taps in (dy, dx) row-major order."""
    h, w = values.shape
    r = size // 2
    v64 = values.astype(np.float64)
    p = np.pad(v64, r, mode="edge")
    inv2_value = -0.5 / (sigma_value * sigma_value)
    inv2_space = -0.5 / (sigma_space * sigma_space)
    num = np.zeros((h, w), dtype=np.float64)
    den = np.zeros((h, w), dtype=np.float64)
    for dy in range(-r, r + 1):
        for dx in range(-r, r + 1):
            win = p[r + dy: r + dy + h, r + dx: r + dx + w]
            diff = win - v64
            wgt = np.exp((dy * dy + dx * dx) * inv2_space + diff * diff * inv2_value)
            num += wgt * win
            den += wgt
    return (num / den).astype(np.float32)


class NumpyOps:
    """The 7-function backend surface (_numpy_ops.py:1-7)."""

    NAME = "oracle"
    box_max = staticmethod(box_max)
    box_min = staticmethod(box_min)
    offsets_max = staticmethod(offsets_max)
    offsets_min = staticmethod(offsets_min)
    median_filter = staticmethod(median_filter)
    gaussian_separable = staticmethod(gaussian_separable)
    bilateral_filter = staticmethod(bilateral_filter)


# ----------------------------------------------------------------------------
# morphology.py
# ----------------------------------------------------------------------------

def _check_kernel(size: int, values: np.ndarray) -> None:
    """morphology._check_kernel (:30-36)."""
    h, w = values.shape
    limit = 2 * min(w, h) + 1
    if size > limit:
        raise ValueError(f"kernel size {size} too large for {w}x{h} map (limit {limit})")


def dilate(values, bits, ops=NumpyOps):
    """morphology.dilate (:39-51): full kernels take the box path."""
    _check_kernel(bits.shape[0], values)
    if bits.all():
        return ops.box_max(values, bits.shape[0] // 2)
    return ops.offsets_max(values, kernel_offsets(bits))


def erode(values, bits, ops=NumpyOps):
    """morphology.erode (:54-62)."""
    _check_kernel(bits.shape[0], values)
    if bits.all():
        return ops.box_min(values, bits.shape[0] // 2)
    return ops.offsets_min(values, kernel_offsets(bits))


def close(values, bits, ops=NumpyOps):
    """morphology.close (:65-67)."""
    return erode(dilate(values, bits, ops), bits, ops)


def masked_fill_dilate(values, bits, ops=NumpyOps):
    """morphology.masked_fill_dilate (:70-78)."""
    d = dilate(values, bits, ops)
    return np.where(values > VALIDITY_THRESHOLD, values, d).astype(np.float32)


def extend_to_top(values):
    """morphology.extend_to_top (:81-96)."""
    h, w = values.shape
    valid = values > VALIDITY_THRESHOLD
    first = valid.argmax(axis=0)
    has = valid.any(axis=0)
    top = values[first, np.arange(w)]
    rows = np.arange(h)[:, None]
    fill = (rows < first[None, :]) & has[None, :]
    return np.where(fill, top[None, :], values).astype(np.float32)


# ----------------------------------------------------------------------------
# pipeline.py
# ----------------------------------------------------------------------------

class BlurMode(Enum):
    """pipeline.py:30-36"""

    NONE = "none"
    BILATERAL = "bilateral"
    MEDIAN = "median"
    MEDIAN_BILATERAL = "median_bilateral"
    GAUSSIAN = "gaussian"
    MEDIAN_GAUSSIAN = "median_gaussian"


class FillMode(Enum):
    """pipeline.py:39-41"""

    FULL = "full"
    PARTIAL = "partial"


@dataclass(frozen=True)
class OracleConfig:
    """PipelineConfig field set and defaults (pipeline.py:50-69), plus the
    inversion offset (depth_core.INVERSION_OFFSET, BASELINE ``max_depth``) and
    the multiscale dilation description (BASELINE config 2/4; see
    ``multiscale_dilate``)."""

    dilation_shape: KernelShape = KernelShape.DIAMOND
    dilation_size: int = 5
    closure_size: int = 5
    small_fill_size: int = 7
    large_fill_size: int = 31
    large_fill_max_iters: int = 100
    blur_mode: BlurMode = BlurMode.MEDIAN_GAUSSIAN
    median_size: int = 5
    gaussian_size: int = 5
    gaussian_sigma: float = 1.1
    bilateral_size: int = 5
    bilateral_sigma_value: float = 1.5
    bilateral_sigma_space: float = 2.0
    fill_mode: FillMode = FillMode.FULL
    max_depth: float = INVERSION_OFFSET
    # multiscale: None (fill_in_fast) or ((edge_near, edge_far),
    # (near_shape, near_size), (med_shape, med_size), (far_shape, far_size))
    multiscale: tuple | None = None


def fit_to_frame(cfg: OracleConfig, h: int, w: int) -> OracleConfig:
    """pipeline._fit_to_frame (:241-254)."""
    limit = 2 * min(w, h) + 1
    ch = {}
    for name in ("dilation_size", "closure_size", "small_fill_size", "large_fill_size"):
        if getattr(cfg, name) > limit:
            ch[name] = max(limit, 3)
    if cfg.multiscale is not None:
        edges, *ks = cfg.multiscale
        ks = tuple((s, min(z, max(limit, 3)) if z > limit else z) for s, z in ks)
        ch["multiscale"] = (edges, *ks)
    return replace(cfg, **ch) if ch else cfg


def multiscale_dilate(direct: np.ndarray, inverted: np.ndarray, cfg: OracleConfig,
                      ops=NumpyOps) -> np.ndarray:
    """Depth-binned stage-2 dilation for ``fill_in_multiscale``.

    NOT IN THE REFERENCE: composed only from pinned
    reference primitives (morphology.dilate per bin).  Builder decision,
    recorded in DESIGN.md:
      bin(p) = near   if 0.1 < d(p) <= edge_near
               medium if edge_near < d(p) <= edge_far
               far    if d(p) > edge_far
    with d the direct input depth; each bin's inverted values (others zeroed)
    are dilated with that bin's kernel and the three results are merged with
    a pointwise max (inverted encoding: nearer wins, exactly as stage 2 does).
    With three identical kernels this equals the fill_in_fast stage 2.
    """
    (e_near, e_far), (sn, zn), (sm, zm), (sf, zf) = cfg.multiscale
    e_near = np.float32(e_near)
    e_far = np.float32(e_far)
    near = direct <= e_near
    med = (direct > e_near) & (direct <= e_far)
    far = direct > e_far
    out = None
    for sel, shape, size in ((near, sn, zn), (med, sm, zm), (far, sf, zf)):
        part = np.where(sel, inverted, np.float32(0.0)).astype(np.float32)
        d = dilate(part, make_kernel(shape, size), ops)
        out = d if out is None else np.maximum(out, d)
    return out


def blur_stage(v: np.ndarray, cfg: OracleConfig, ops=NumpyOps) -> np.ndarray:
    """pipeline._blur_stage (:206-238)."""
    partial = cfg.fill_mode is FillMode.PARTIAL
    mode = cfg.blur_mode

    def reimpose(b, m):
        return np.where(m, b, np.float32(0.0)).astype(np.float32)

    if mode in (BlurMode.MEDIAN, BlurMode.MEDIAN_BILATERAL, BlurMode.MEDIAN_GAUSSIAN):
        m = v > VALIDITY_THRESHOLD
        v = ops.median_filter(v, cfg.median_size)
        if partial:
            v = reimpose(v, m)
    if mode in (BlurMode.GAUSSIAN, BlurMode.MEDIAN_GAUSSIAN):
        m = v > VALIDITY_THRESHOLD
        v = ops.gaussian_separable(v, gaussian_weights(cfg.gaussian_size, cfg.gaussian_sigma))
        if partial:
            v = reimpose(v, m)
    if mode in (BlurMode.BILATERAL, BlurMode.MEDIAN_BILATERAL):
        m = v > VALIDITY_THRESHOLD
        v = ops.bilateral_filter(v, cfg.bilateral_size, float(cfg.bilateral_sigma_value),
                                 float(cfg.bilateral_sigma_space))
        if partial:
            v = reimpose(v, m)
    return v


def complete_with_stats(values: np.ndarray, cfg: OracleConfig | None = None, ops=NumpyOps,
                        return_stages: bool = False):
    """pipeline.complete_with_stats (:124-203) restated on arrays.

    Returns (dense, info) where info holds input/output density and the
    large-fill iteration count (RunStats fields, pipeline.py:104-115); with
    ``return_stages`` also every intermediate stage map.
    """
    cfg = cfg or OracleConfig()
    values = validate(values)
    n_valid = int(np.count_nonzero(values > VALIDITY_THRESHOLD))
    if n_valid == 0:
        raise DegenerateInputError("input depth map has no valid pixels")
    h, w = values.shape
    cfg = fit_to_frame(cfg, h, w)
    full = cfg.fill_mode is FillMode.FULL
    stages = {}

    cur = flip(values, cfg.max_depth)
    stages["invert"] = cur
    if cfg.multiscale is None:
        cur = dilate(cur, make_kernel(cfg.dilation_shape, cfg.dilation_size), ops)
    else:
        cur = multiscale_dilate(values, cur, cfg, ops)
    stages["dilate"] = cur
    cur = close(cur, make_kernel(KernelShape.FULL, cfg.closure_size), ops)
    stages["close"] = cur
    cur = masked_fill_dilate(cur, make_kernel(KernelShape.FULL, cfg.small_fill_size), ops)
    stages["small_fill"] = cur
    if full:
        cur = extend_to_top(cur)
    stages["extend_top"] = cur
    iters = 0
    if full:
        big = make_kernel(KernelShape.FULL, cfg.large_fill_size)
        while iters < cfg.large_fill_max_iters:
            if not (cur <= VALIDITY_THRESHOLD).any():
                break
            cur = masked_fill_dilate(cur, big, ops)
            iters += 1
    stages["large_fill"] = cur
    cur = blur_stage(cur, cfg, ops)
    stages["blur"] = cur
    dense = flip(cur, cfg.max_depth)
    stages["invert_back"] = dense
    info = {
        "input_density": n_valid / values.size,
        "output_density": float(np.count_nonzero(dense > VALIDITY_THRESHOLD)) / dense.size,
        "large_fill_iterations": iters,
    }
    if return_stages:
        info["stages"] = stages
    return dense, info


def complete(values: np.ndarray, cfg: OracleConfig | None = None, ops=NumpyOps) -> np.ndarray:
    """pipeline.complete (:118-121)."""
    return complete_with_stats(values, cfg, ops)[0]


# Default multiscale description (builder decision).
DEFAULT_MULTISCALE = (
    (15.0, 30.0),
    (KernelShape.FULL, 7),      # near   0.1 - 15 m : objects large in the image
    (KernelShape.DIAMOND, 7),   # medium 15 - 30 m
    (KernelShape.DIAMOND, 5),   # far    > 30 m     : the fill_in_fast kernel
)
