"""Pipeline API mirroring the reference's ``depthfill.pipeline`` on the GPU.

Mirrors pipeline.py:30-203 -- ``BlurMode``, ``FillMode``, ``PipelineConfig``
(same fields, defaults and validation), ``STAGE_NAMES``, ``RunStats``,
``complete`` and ``complete_with_stats`` -- and adds ``complete_batch`` for
[B, H, W] batches.  ``complete``/``complete_batch`` run the fused sm_100a
pipeline through ``dfc_fill_batch``; ``complete_with_stats`` runs the stages
one launch at a time with CUDA events around each, the GPU analogue of the
reference's per-stage ``perf_counter`` timing (pipeline.py:145-152).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace
from enum import Enum

import numpy as np
import torch

from . import _lib, domain, ops
from .domain import (DegenerateInputError, DepthEncoding, DepthMap, DepthRangeError, EncodingError,
                     KernelShape, kernel_offsets, make_kernel)


class BlurMode(Enum):
    NONE = "none"
    BILATERAL = "bilateral"
    MEDIAN = "median"
    MEDIAN_BILATERAL = "median_bilateral"
    GAUSSIAN = "gaussian"
    MEDIAN_GAUSSIAN = "median_gaussian"


class FillMode(Enum):
    FULL = "full"
    PARTIAL = "partial"


_SIZE_FIELDS = ("dilation_size", "closure_size", "small_fill_size", "large_fill_size", "median_size",
                "gaussian_size", "bilateral_size")


@dataclass(frozen=True)
class PipelineConfig:
    """pipeline.PipelineConfig (pipeline.py:50-89), plus two optional extras:
    ``max_depth`` (None = domain.INVERSION_OFFSET, read at call time like the
    reference's _flip) and ``exact_blur`` (fp64 blurs in the reference's
    operation order instead of the fp32 fast path)."""

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
    max_depth: float | None = None
    exact_blur: bool = False

    def __post_init__(self):
        for name in _SIZE_FIELDS:
            v = getattr(self, name)
            if not isinstance(v, int) or v < 3 or v % 2 == 0:
                raise ValueError(f"{name} must be an odd integer >= 3, got {v!r}")
        if self.large_fill_max_iters < 1:
            raise ValueError("large_fill_max_iters must be >= 1")
        if self.gaussian_sigma <= 0:
            raise ValueError("gaussian_sigma must be positive")
        if self.bilateral_sigma_value <= 0 or self.bilateral_sigma_space <= 0:
            raise ValueError("bilateral sigmas must be positive")


@dataclass(frozen=True)
class MultiscaleConfig:
    """Depth-binned stage-2 dilation for ``fill_in_multiscale``.

    near: 0.1 < d <= edges[0]; medium: edges[0] < d <= edges[1]; far: d > edges[1]
    (d = direct input depth).  Each bin is dilated with its own kernel and the
    three results are merged by pointwise max (inverted encoding: nearer wins).
    """

    bin_edges: tuple[float, float] = (15.0, 30.0)
    near: tuple[KernelShape, int] = (KernelShape.FULL, 7)
    medium: tuple[KernelShape, int] = (KernelShape.DIAMOND, 7)
    far: tuple[KernelShape, int] = (KernelShape.DIAMOND, 5)

    def __post_init__(self):
        lo, hi = self.bin_edges
        if not lo < hi:
            raise ValueError("bin edges must be increasing")
        for name in ("near", "medium", "far"):
            shape, size = getattr(self, name)
            make_kernel(KernelShape(shape), size)  # validates


STAGE_NAMES = ("invert", "dilate", "close", "small_fill", "extend_top", "large_fill", "blur", "invert_back")


@dataclass(frozen=True)
class RunStats:
    """pipeline.RunStats (pipeline.py:104-115); stage times are CUDA-event ms."""

    stage_ms: tuple[tuple[str, float], ...]
    total_ms: float
    input_density: float
    output_density: float
    large_fill_iterations: int = 0

    def stage(self, name: str) -> float:
        return dict(self.stage_ms)[name]


def _max_depth(config: PipelineConfig) -> float:
    return float(domain.INVERSION_OFFSET if config.max_depth is None else config.max_depth)


def fit_to_frame(config: PipelineConfig, height: int, width: int) -> PipelineConfig:
    """pipeline._fit_to_frame (pipeline.py:241-254)."""
    limit = 2 * min(width, height) + 1
    ch = {n: max(limit, 3) for n in ("dilation_size", "closure_size", "small_fill_size", "large_fill_size")
          if getattr(config, n) > limit}
    return replace(config, **ch) if ch else config


def to_dfc_config(config: PipelineConfig, multiscale: MultiscaleConfig | None = None,
                  custom_offsets: np.ndarray | None = None, force_staged: bool = False) -> _lib.DfcConfig:
    """Marshal a PipelineConfig into the POD ``dfc_config`` of include/dfc.h."""
    c = _lib.DfcConfig()
    _lib.load().dfc_config_init(ctypes.byref(c))
    c.dilation_shape = _lib.SHAPE_CODES[KernelShape(config.dilation_shape).value]
    for name in _SIZE_FIELDS + ("large_fill_max_iters",):
        setattr(c, name, int(getattr(config, name)))
    c.blur_mode = _lib.BLUR_CODES[BlurMode(config.blur_mode).value]
    c.fill_mode = _lib.FILL_CODES[FillMode(config.fill_mode).value]
    c.gaussian_sigma = float(config.gaussian_sigma)
    c.bilateral_sigma_value = float(config.bilateral_sigma_value)
    c.bilateral_sigma_space = float(config.bilateral_sigma_space)
    c.max_depth = _max_depth(config)
    flags = 0
    if config.exact_blur:
        flags |= _lib.F_EXACT_BLUR
    if force_staged:
        flags |= _lib.F_FORCE_STAGED
    c.flags = flags
    if multiscale is not None:
        c.multiscale = 1
        c.bin_edge_near, c.bin_edge_far = (float(e) for e in multiscale.bin_edges)
        for pre, (shape, size) in (("near", multiscale.near), ("med", multiscale.medium), ("far", multiscale.far)):
            setattr(c, f"{pre}_shape", _lib.SHAPE_CODES[KernelShape(shape).value])
            setattr(c, f"{pre}_size", int(size))
    if custom_offsets is not None:
        o = np.ascontiguousarray(np.asarray(custom_offsets, dtype=np.int32).reshape(-1, 2))
        arr = (ctypes.c_int32 * o.size)(*o.ravel().tolist())
        c.custom_n = o.shape[0]
        c.custom_offsets = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int32))
        c._keepalive = arr  # noqa: SLF001 -- keep the host array alive with the struct
    return c


def raise_for_status(status: np.ndarray, max_depth: float) -> None:
    """Map per-frame DFC_ST_* bits to the reference's exceptions, first bad frame first."""
    bad = np.nonzero(status & 0xFF)[0]
    if bad.size == 0:
        return
    b = int(bad[0])
    s = int(status[b])
    where = f" (frame {b})" if status.size > 1 else ""
    if s & _lib.ST_NONFINITE:
        raise ValueError("depth values must be finite" + where)
    if s & _lib.ST_NEGATIVE:
        raise ValueError("depth values must be non-negative" + where)
    if s & _lib.ST_DEGENERATE:
        raise DegenerateInputError("input depth map has no valid pixels" + where)
    if s & _lib.ST_RANGE:
        raise DepthRangeError(f"values must be < {max_depth} to be invertible" + where)
    if s & _lib.ST_ENCODE:  # kitti_io.write_depth_png (kitti_io.py:60-61)
        raise ValueError("depth values must be < 256 m to be encodable" + where)


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1802_00036_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


# Input density below which the previous batch on a device selects the fused
# kernel's register-dense large fill for the next one (DFC_F_SPARSE; dense
# frames run ~2 % faster without it, 1 %-density frames 2.4x faster with it).
SPARSE_DENSITY = 0.025
_last_sparse: dict[int, bool] = {}


def complete_batch(frames, config: PipelineConfig | None = None, multiscale: MultiscaleConfig | None = None,
                   custom_offsets=None, raise_on_error: bool = True, force_staged: bool = False,
                   sparse_hint: bool | None = None) -> ops.FillResult:
    """Complete a [B, H, W] batch (torch CUDA tensor, or host array copied in).

    ``sparse_hint`` (performance only, results are identical): True / False
    selects / skips the register-dense large fill for frames with many empty
    pixels; None (default) follows the input density the previous call
    measured on this device."""
    config = config or PipelineConfig()
    if isinstance(frames, np.ndarray):
        frames = np.ascontiguousarray(frames, dtype=np.float32)
        if not frames.flags.writeable:
            frames = frames.copy()
        frames = torch.from_numpy(frames)
    if frames.device.type != "cuda":
        frames = frames.to(_device(), non_blocking=True)
    if frames.dim() == 2:
        frames = frames.unsqueeze(0)
    cfg = to_dfc_config(config, multiscale, custom_offsets, force_staged)
    dev = frames.device.index or 0
    if sparse_hint if sparse_hint is not None else _last_sparse.get(dev, False):
        cfg.flags |= _lib.F_SPARSE
    res = ops.fill_batch(frames, cfg)
    if raise_on_error:
        raise_for_status(res.status.cpu().numpy(), _max_depth(config))
    if res.valid_counts is not None and res.dense.numel():
        n_in = float(res.valid_counts[:, 0].sum().item())
        _last_sparse[dev] = n_in / res.dense.numel() < SPARSE_DENSITY
    return res


def complete(sparse, config: PipelineConfig | None = None) -> DepthMap:
    """Densify a sparse direct-encoded depth map (pipeline.complete, :118-121)."""
    config = config or PipelineConfig()
    sparse = DepthMap.coerce(sparse)
    if sparse.encoding is not DepthEncoding.DIRECT:
        raise EncodingError("pipeline input must be direct-encoded")
    res = complete_batch(sparse.values[None], config)
    return DepthMap._wrap(res.dense[0].cpu().numpy(), DepthEncoding.DIRECT)


# ---------------------------------------------------------------------------
# staged execution with per-stage CUDA-event timing
# ---------------------------------------------------------------------------

def _dilate(t: torch.Tensor, shape: KernelShape, size: int) -> torch.Tensor:
    k = make_kernel(shape, size)
    return ops.box_max(t, size // 2) if k.is_full else ops.offsets_max(t, kernel_offsets(k))


def _gaussian_weights(size: int, sigma: float) -> np.ndarray:
    half = size // 2
    i = np.arange(-half, half + 1, dtype=np.float64)
    w = np.exp(-(i * i) / (2.0 * sigma * sigma))
    return w / w.sum()


def _blur(v: torch.Tensor, config: PipelineConfig) -> torch.Tensor:
    """pipeline._blur_stage (pipeline.py:206-238)."""
    partial = FillMode(config.fill_mode) is FillMode.PARTIAL
    mode = BlurMode(config.blur_mode)
    if mode in (BlurMode.MEDIAN, BlurMode.MEDIAN_BILATERAL, BlurMode.MEDIAN_GAUSSIAN):
        b = ops.median(v, config.median_size)
        v = ops.reimpose(b, v) if partial else b
    if mode in (BlurMode.GAUSSIAN, BlurMode.MEDIAN_GAUSSIAN):
        b = ops.gaussian_separable(v, _gaussian_weights(config.gaussian_size, config.gaussian_sigma),
                                   config.exact_blur)
        v = ops.reimpose(b, v) if partial else b
    if mode in (BlurMode.BILATERAL, BlurMode.MEDIAN_BILATERAL):
        b = ops.bilateral(v, config.bilateral_size, config.bilateral_sigma_value, config.bilateral_sigma_space,
                          config.exact_blur)
        v = ops.reimpose(b, v) if partial else b
    return v


def complete_with_stats(sparse, config: PipelineConfig | None = None) -> tuple[DepthMap, RunStats]:
    """pipeline.complete_with_stats (:124-203): eight stages, each timed."""
    config = config or PipelineConfig()
    sparse = DepthMap.coerce(sparse)
    if sparse.encoding is not DepthEncoding.DIRECT:
        raise EncodingError("pipeline input must be direct-encoded")
    dev = _device()
    x = torch.from_numpy(np.array(sparse.values, dtype=np.float32, copy=True)).to(dev)
    # input density: the device validity reduction (pipeline.py:138-141)
    n_valid = int(ops.validate(x)[1].cpu()[0])
    if n_valid == 0:
        raise DegenerateInputError("input depth map has no valid pixels")
    config = fit_to_frame(config, sparse.height, sparse.width)
    full = FillMode(config.fill_mode) is FillMode.FULL
    off = _max_depth(config)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(STAGE_NAMES) + 1)]
    ev[0].record()
    cur, st = ops.invert(x, off)
    ev[1].record()
    if int(st.cpu()[0]) & _lib.ST_RANGE:
        raise DepthRangeError(f"values must be < {off} to be invertible")
    cur = _dilate(cur, KernelShape(config.dilation_shape), config.dilation_size)
    ev[2].record()
    cur = ops.box_min(ops.box_max(cur, config.closure_size // 2), config.closure_size // 2)
    ev[3].record()
    cur = ops.masked_fill(cur, ops.box_max(cur, config.small_fill_size // 2))
    ev[4].record()
    if full:
        cur = ops.extend_to_top(cur)
    ev[5].record()
    iters = 0
    if full:
        while iters < config.large_fill_max_iters:
            if int(ops.count_empty(cur).cpu()[0]) == 0:
                break
            cur = ops.masked_fill(cur, ops.box_max(cur, config.large_fill_size // 2))
            iters += 1
    ev[6].record()
    cur = _blur(cur, config)
    ev[7].record()
    dense, _ = ops.invert(cur, off)
    ev[8].record()
    torch.cuda.synchronize()
    times = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(STAGE_NAMES))]
    if not full:
        times[4] = times[5] = 0.0
    # output density: the device count of pixels > 0.1 (pipeline.py:192-202)
    n_out = dense.numel() - int(ops.count_empty(dense)[0].cpu())
    out = dense.cpu().numpy()
    stats = RunStats(
        stage_ms=tuple(zip(STAGE_NAMES, times)),
        total_ms=ev[0].elapsed_time(ev[-1]),
        input_density=n_valid / sparse.values.size,
        output_density=n_out / out.size,
        large_fill_iterations=iters,
    )
    return DepthMap._wrap(out, DepthEncoding.DIRECT), stats


# ---------------------------------------------------------------------------
# host-buffer batch API: pinned host in -> GPU -> pinned host out, pipelined
# ---------------------------------------------------------------------------

class HostPipeline:
    """Complete frames that live in (pinned) host memory.

    The batch is cut into chunks; chunk k's host->device copy, pipeline launch
    and device->host copy are issued on stream k % n_streams, so copies in both
    directions overlap with computation of neighbouring chunks.  Fused-kernel
    statuses are collected for the whole batch and checked once at the end;
    frames that the fused kernel flagged for the multi-iteration fallback are
    re-run through the staged path from the host input.
    """

    def __init__(self, config: PipelineConfig | None = None, multiscale: MultiscaleConfig | None = None,
                 chunk: int = 64, n_streams: int = 3, device=None):
        self.config = config or PipelineConfig()
        self.multiscale = multiscale
        self.chunk = int(chunk)
        self.device = torch.device(device) if device is not None else _device()
        self.streams = [torch.cuda.Stream(self.device) for _ in range(n_streams)]
        self.cfg = to_dfc_config(self.config, multiscale)
        self.cfg.flags |= _lib.F_NO_FINISH
        self._bufs = None

    def _alloc(self, H, W):
        if self._bufs is not None and self._bufs[0] == (H, W):
            return self._bufs[1]
        bufs = []
        for _ in self.streams:
            bufs.append((torch.empty((self.chunk, H, W), dtype=torch.float32, device=self.device),
                         torch.empty((self.chunk, H, W), dtype=torch.float32, device=self.device),
                         ops.Workspace()))
        self._bufs = ((H, W), bufs)
        return bufs

    def run(self, host_in: torch.Tensor, host_out: torch.Tensor | None = None,
            raise_on_error: bool = True) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
        """host_in: [B,H,W] float32 CPU tensor (pinned for full overlap).
        Returns (host_out, status[B] int32 CPU, iterations[B] int32 CPU)."""
        if host_in.dim() == 2:
            host_in = host_in.unsqueeze(0)
        B, H, W = host_in.shape
        if host_out is None:
            host_out = torch.empty((B, H, W), dtype=torch.float32, pin_memory=True)
        bufs = self._alloc(H, W)
        status = torch.empty(B, dtype=torch.int32, device=self.device)
        iters = torch.empty(B, dtype=torch.int32, device=self.device)
        cur = torch.cuda.current_stream(self.device)
        for s in self.streams:
            s.wait_stream(cur)
        for k, a in enumerate(range(0, B, self.chunk)):
            b = min(B, a + self.chunk)
            s = self.streams[k % len(self.streams)]
            d_in, d_out, ws = bufs[k % len(self.streams)]
            with torch.cuda.stream(s):
                d_in[: b - a].copy_(host_in[a:b], non_blocking=True)
                ops.fill_batch(d_in[: b - a], self.cfg, out=d_out[: b - a], workspace=ws, status=status[a:b],
                               iterations=iters[a:b])
                host_out[a:b].copy_(d_out[: b - a], non_blocking=True)
        for s in self.streams:
            cur.wait_stream(s)
        st = status.cpu()
        it = iters.cpu()
        need = torch.nonzero(st & 0x200).flatten().tolist()
        if need:  # rare: frames needing more than one large-fill iteration
            res = complete_batch(host_in[need], self.config, self.multiscale, raise_on_error=False,
                                 force_staged=True)
            host_out[need] = res.dense.cpu()
            st[need] = res.status.cpu() | _lib.ST_FALLBACK
            it[need] = res.iterations.cpu()
        if raise_on_error:
            raise_for_status(st.numpy(), _max_depth(self.config))
        return host_out, st, it
