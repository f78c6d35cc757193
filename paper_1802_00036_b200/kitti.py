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
    if v.dtype != torch.float32:  # dfc_colormap reads float32
        v = v.to(torch.float32)
    v = v.contiguous()
    rgb = torch.empty(tuple(v.shape) + (3,), dtype=torch.uint8, device=v.device)
    _lib.check(_lib.load().dfc_colormap(ops._ptr(v), ops._ptr(rgb), v.numel(), float(range_min), float(range_max),
                                        ops._stream()))
    return rgb


class RawPipeline:
    """KITTI raw frames in pinned host memory -> GPU -> raw frames in pinned host
    memory, like completion.HostPipeline: chunk k's copies and launch go to stream
    k % n_streams so both copy directions overlap computation; 2 B/px each way.
    Frames the fused kernel flags for more large-fill iterations are re-run
    through the staged path at the end."""

    def __init__(self, config: PipelineConfig | None = None, chunk: int = 64, n_streams: int = 3, device=None):
        self.config = config or PipelineConfig()
        self.chunk = int(chunk)
        self.device = torch.device(device) if device is not None else _device()
        self.streams = [torch.cuda.Stream(self.device) for _ in range(n_streams)]
        self.cfg = to_dfc_config(self.config)
        self.cfg.flags |= _lib.F_NO_FINISH
        self._bufs = None

    def _alloc(self, H, W):
        if self._bufs is None or self._bufs[0] != (H, W):
            self._bufs = ((H, W), [(torch.empty((self.chunk, H, W), dtype=torch.uint16, device=self.device),
                                    torch.empty((self.chunk, H, W), dtype=torch.uint16, device=self.device),
                                    ops.Workspace()) for _ in self.streams])
        return self._bufs[1]

    def run(self, host_in: torch.Tensor, host_out: torch.Tensor | None = None, raise_on_error: bool = True):
        """host_in: [B, H, W] uint16 CPU tensor (pinned for full overlap); returns (host_out, status, iterations)."""
        B, H, W = host_in.shape
        if host_out is None:
            host_out = torch.empty((B, H, W), dtype=torch.uint16, pin_memory=True)
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
                ops.fill_batch_raw16(d_in[: b - a], self.cfg, out_raw=True, workspace=ws, out=d_out[: b - a],
                                     status=status[a:b], iterations=iters[a:b])
                host_out[a:b].copy_(d_out[: b - a], non_blocking=True)
        for s in self.streams:
            cur.wait_stream(s)
        st = status.cpu()
        it = iters.cpu()
        need = torch.nonzero(st & 0x200).flatten().tolist()
        if need:  # rare: frames needing more than one large-fill iteration
            raw_need = host_in.view(torch.int16)[need].view(torch.uint16)  # (no uint16 gather / scatter in torch)
            res = complete_raw16_batch(raw_need, self.config, out_raw=True, raise_on_error=False, force_staged=True)
            host_out.view(torch.int16)[need] = res.dense.cpu().view(torch.int16)
            st[need] = res.status.cpu() | _lib.ST_FALLBACK
            it[need] = res.iterations.cpu()
        if raise_on_error:
            raise_for_status(st.numpy(), _max_depth(self.config))
        return host_out, st, it

