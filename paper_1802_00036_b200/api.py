"""BASELINE-named entry points: ``fill_in_fast`` and ``fill_in_multiscale``.

These names are absent from the reference package (SURVEY.md finding 2); the
argument mapping onto the reference's ``complete(DepthMap, PipelineConfig)``
is SURVEY.md 8(b):

  max_depth      -> depth_core.INVERSION_OFFSET (depth_core.py:25,152,156)
  custom_kernel  -> dilation_shape + dilation_size (pipeline.py:52-53,159);
                    a Kernel / (shape, size) / square bool array
  extrapolate    -> fill_mode FULL (True) or PARTIAL (False) (pipeline.py:39-41)
  blur_type      -> blur_mode by enum value (pipeline.py:30-36)

Inputs may be one [H, W] map or a [B, H, W] batch, as a numpy array (copied to
the GPU and back) or a CUDA tensor (kept on the device).  The result has the
same kind and shape as the input.
"""

from __future__ import annotations

import numpy as np
import torch

from .completion import BlurMode, FillMode, MultiscaleConfig, PipelineConfig, complete_batch
from .domain import Kernel, KernelShape, kernel_offsets, make_kernel

DIAMOND_KERNEL_5 = make_kernel(KernelShape.DIAMOND, 5)


def _kernel_args(custom_kernel):
    """-> (shape, size, custom_offsets or None)."""
    if custom_kernel is None:
        return KernelShape.DIAMOND, 5, None
    if isinstance(custom_kernel, tuple) and len(custom_kernel) == 2:
        shape, size = custom_kernel
        return KernelShape(shape), int(size), None
    k = custom_kernel if isinstance(custom_kernel, Kernel) else Kernel(np.asarray(custom_kernel, dtype=bool))
    named = k.named()
    if named is not None:
        return named[0], named[1], None
    return KernelShape.DIAMOND, k.size, kernel_offsets(k)


def _run(depth_map, config, multiscale=None, custom_offsets=None):
    is_np = not isinstance(depth_map, torch.Tensor)
    x = np.asarray(depth_map, dtype=np.float32) if is_np else depth_map
    single = x.ndim == 2
    if x.ndim not in (2, 3):
        raise ValueError(f"depth map must be 2-D or a [B,H,W] batch, got shape {tuple(x.shape)}")
    if custom_offsets is not None:
        limit = 2 * min(x.shape[-2], x.shape[-1]) + 1
        if config.dilation_size > limit:
            raise ValueError(f"kernel size {config.dilation_size} too large for {x.shape[-1]}x{x.shape[-2]} map "
                             f"(limit {limit})")
    res = complete_batch(x[None] if single else x, config, multiscale, custom_offsets)
    out = res.dense[0] if single else res.dense
    if is_np:
        return out.cpu().numpy()
    return out


def fill_in_fast(depth_map, max_depth: float = 100.0, custom_kernel=DIAMOND_KERNEL_5, extrapolate: bool = False,
                 blur_type: str = "bilateral", exact_blur: bool = False):
    """Depth completion with a single stage-2 kernel (the paper's algorithm)."""
    shape, size, offs = _kernel_args(custom_kernel)
    cfg = PipelineConfig(dilation_shape=shape, dilation_size=size, blur_mode=BlurMode(blur_type),
                         fill_mode=FillMode.FULL if extrapolate else FillMode.PARTIAL,
                         max_depth=float(max_depth), exact_blur=exact_blur)
    return _run(depth_map, cfg, custom_offsets=offs)


def fill_in_multiscale(depth_map, max_depth: float = 100.0, near_kernel=(KernelShape.FULL, 7),
                       medium_kernel=(KernelShape.DIAMOND, 7), far_kernel=(KernelShape.DIAMOND, 5),
                       bin_edges=(15.0, 30.0), extrapolate: bool = True, blur_type: str = "bilateral",
                       median_blur: bool = True, exact_blur: bool = False):
    """Depth completion with depth-binned stage-2 dilation (BASELINE config 2/4).

    ``blur_type`` 'bilateral' or 'gaussian' (or 'none'); ``median_blur`` adds the
    5x5 median before it ('bilateral' + median = BlurMode.MEDIAN_BILATERAL).
    """
    def kern(k):
        if isinstance(k, Kernel):
            named = k.named()
            if named is None:
                raise ValueError("multiscale bin kernels must be one of the Fig. 3 shapes")
            return named
        return KernelShape(k[0]), int(k[1])

    ms = MultiscaleConfig(bin_edges=tuple(float(e) for e in bin_edges), near=kern(near_kernel),
                          medium=kern(medium_kernel), far=kern(far_kernel))
    bt = BlurMode(blur_type)
    if median_blur:
        bt = {BlurMode.BILATERAL: BlurMode.MEDIAN_BILATERAL, BlurMode.GAUSSIAN: BlurMode.MEDIAN_GAUSSIAN,
              BlurMode.NONE: BlurMode.MEDIAN}.get(bt, bt)
    cfg = PipelineConfig(blur_mode=bt, fill_mode=FillMode.FULL if extrapolate else FillMode.PARTIAL,
                         max_depth=float(max_depth), exact_blur=exact_blur)
    return _run(depth_map, cfg, multiscale=ms)
