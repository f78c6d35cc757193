"""KITTI 16-bit depth values at the boundary.

The reference reads and writes KITTI depth PNGs with `kitti_io.read_depth_png`
(depth = raw / 256, kitti_io.py:36-54) and `write_depth_png` (raw =
rint(depth * 256) clipped to 16 bits, values >= 256 m rejected,
kitti_io.py:57-66).  PNG (de)compression stays on the host; these functions
take the decoded uint16 raw arrays and fuse the value conversion into the
pipeline's read and write passes, so a frame moves 2 B/px in and 2 B/px out
instead of 4 + 4.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib, ops
from .completion import PipelineConfig, _device, _max_depth, raise_for_status, to_dfc_config

DEPTH_SCALE = 256.0
MAX_DEPTH_M = 65535 / DEPTH_SCALE


def _raw_tensor(raw) -> torch.Tensor:
    if isinstance(raw, np.ndarray):
        if raw.dtype != np.uint16:
            if raw.size and (raw.min() < 0 or raw.max() > 65535):
                raise ValueError("sample values exceed 16-bit range")  # kitti_io.py:49-51
            raw = raw.astype(np.uint16)
        raw = torch.from_numpy(np.ascontiguousarray(raw))
    if raw.device.type != "cuda":
        raw = raw.to(_device())
    return raw


def decode(raw) -> torch.Tensor:
    """uint16 raw -> float32 depth in meters (read_depth_png's conversion)."""
    return ops.decode_raw16(_raw_tensor(raw))


def encode(depth) -> torch.Tensor:
    """float32 depth -> uint16 raw (write_depth_png's conversion); raises ValueError for >= 256 m."""
    d = depth if isinstance(depth, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(depth, np.float32))
    if d.device.type != "cuda":
        d = d.to(_device())
    raw, status = ops.encode_raw16(d)
    raise_for_status(status.cpu().numpy(), 0.0)
    return raw


def complete_raw16_batch(raw, config: PipelineConfig | None = None, out_raw: bool = True, multiscale=None,
                         raise_on_error: bool = True, force_staged: bool = False) -> ops.FillResult:
    """complete() on a [B, H, W] batch of KITTI raw frames; uint16 raw (or float32 depth) out."""
    config = config or PipelineConfig()
    cfg = to_dfc_config(config, multiscale, None, force_staged)
    res = ops.fill_batch_raw16(_raw_tensor(raw), cfg, out_raw=out_raw)
    if raise_on_error:
        raise_for_status(res.status.cpu().numpy(), _max_depth(config))
    return res


def colormap(values, range_min: float, range_max: float) -> torch.Tensor:
    """write_colormap_png's pixels (kitti_io.py:69-85) on the GPU: uint8 [..., 3] on the
    blue -> red ramp of clip((v - lo) / (hi - lo), 0, 1), black where v == 0."""
    if range_max <= range_min:
        raise ValueError(f"degenerate range [{range_min}, {range_max}]")
    v = values if isinstance(values, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(values, np.float32))
    if v.device.type != "cuda":
        v = v.to(_device())
    v = v.contiguous()
    rgb = torch.empty(tuple(v.shape) + (3,), dtype=torch.uint8, device=v.device)
    _lib.check(_lib.load().dfc_colormap(ops._ptr(v), ops._ptr(rgb), v.numel(), float(range_min), float(range_max),
                                        ops._stream()))
    return rgb

