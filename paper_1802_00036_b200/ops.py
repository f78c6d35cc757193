"""Device-tensor wrappers over the C ABI (torch tensors only at this boundary).

Every function takes CUDA float32 tensors shaped [B, H, W] (or [H, W]) and
returns fresh tensors, launching on torch's current stream.  Nothing here
computes on the CPU: a missing libdfc.so or CUDA device raises.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _as_batch(t: torch.Tensor) -> tuple[torch.Tensor, bool]:
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if t.device.type != "cuda":
        raise ValueError("libdfc ops need CUDA tensors")
    if t.dtype != torch.float32:
        raise ValueError("depth maps must be float32")
    squeeze = t.dim() == 2
    if squeeze:
        t = t.unsqueeze(0)
    if t.dim() != 3:
        raise ValueError(f"expected [B,H,W] or [H,W], got {tuple(t.shape)}")
    return t.contiguous(), squeeze


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _out(t, squeeze):
    return t.squeeze(0) if squeeze else t


def _op_ws(B, H, W, device) -> torch.Tensor:
    n = _lib.load().dfc_op_workspace_bytes(B, H, W)
    return torch.empty(max(int(n), 1), dtype=torch.uint8, device=device)


def box_max(t: torch.Tensor, radius: int) -> torch.Tensor:
    x, sq = _as_batch(t)
    B, H, W = x.shape
    out = torch.empty_like(x)
    ws = _op_ws(B, H, W, x.device)
    check(_lib.load().dfc_box_max(_ptr(x), _ptr(out), B, H, W, int(radius), _ptr(ws), ws.numel(), _stream()))
    return _out(out, sq)


def box_min(t: torch.Tensor, radius: int) -> torch.Tensor:
    x, sq = _as_batch(t)
    B, H, W = x.shape
    out = torch.empty_like(x)
    ws = _op_ws(B, H, W, x.device)
    check(_lib.load().dfc_box_min(_ptr(x), _ptr(out), B, H, W, int(radius), _ptr(ws), ws.numel(), _stream()))
    return _out(out, sq)


def _offs(offsets) -> tuple[ctypes.Array, int]:
    o = np.ascontiguousarray(np.asarray(offsets, dtype=np.int32).reshape(-1, 2))
    arr = (ctypes.c_int32 * o.size)(*o.ravel().tolist())
    return arr, o.shape[0]


def offsets_max(t: torch.Tensor, offsets) -> torch.Tensor:
    x, sq = _as_batch(t)
    B, H, W = x.shape
    out = torch.empty_like(x)
    arr, n = _offs(offsets)
    check(_lib.load().dfc_offsets_max(_ptr(x), _ptr(out), B, H, W, arr, n, _stream()))
    return _out(out, sq)


def offsets_min(t: torch.Tensor, offsets) -> torch.Tensor:
    x, sq = _as_batch(t)
    B, H, W = x.shape
    out = torch.empty_like(x)
    arr, n = _offs(offsets)
    check(_lib.load().dfc_offsets_min(_ptr(x), _ptr(out), B, H, W, arr, n, _stream()))
    return _out(out, sq)


def median(t: torch.Tensor, size: int) -> torch.Tensor:
    x, sq = _as_batch(t)
    B, H, W = x.shape
    out = torch.empty_like(x)
    check(_lib.load().dfc_median(_ptr(x), _ptr(out), B, H, W, int(size), _stream()))
    return _out(out, sq)


def gaussian_separable(t: torch.Tensor, weights, exact: bool = False) -> torch.Tensor:
    x, sq = _as_batch(t)
    B, H, W = x.shape
    out = torch.empty_like(x)
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    warr = (ctypes.c_double * w.size)(*w.tolist())
    ws = _op_ws(B, H, W, x.device)
    check(_lib.load().dfc_gaussian_separable(_ptr(x), _ptr(out), B, H, W, warr, w.size, int(bool(exact)), _ptr(ws),
                                             ws.numel(), _stream()))
    return _out(out, sq)


def bilateral(t: torch.Tensor, size: int, sigma_value: float, sigma_space: float, exact: bool = False):
    x, sq = _as_batch(t)
    B, H, W = x.shape
    out = torch.empty_like(x)
    check(_lib.load().dfc_bilateral(_ptr(x), _ptr(out), B, H, W, int(size), float(sigma_value), float(sigma_space),
                                    int(bool(exact)), _stream()))
    return _out(out, sq)


def invert(t: torch.Tensor, offset: float = 100.0) -> tuple[torch.Tensor, torch.Tensor]:
    """_flip: returns (out, status[B]) with DFC_ST_RANGE set where any v >= offset."""
    x, sq = _as_batch(t)
    B, H, W = x.shape
    out = torch.empty_like(x)
    st = torch.zeros(B, dtype=torch.int32, device=x.device)
    check(_lib.load().dfc_invert(_ptr(x), _ptr(out), B, H, W, float(offset), _ptr(st), _stream()))
    return _out(out, sq), st


def validate(t: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    x, _ = _as_batch(t)
    B, H, W = x.shape
    st = torch.zeros(B, dtype=torch.int32, device=x.device)
    nv = torch.zeros(B, dtype=torch.int64, device=x.device)
    check(_lib.load().dfc_validate(_ptr(x), B, H, W, _ptr(st), _ptr(nv), _stream()))
    return st, nv


def masked_fill(cur: torch.Tensor, dilated: torch.Tensor) -> torch.Tensor:
    x, sq = _as_batch(cur)
    d, _ = _as_batch(dilated)
    B, H, W = x.shape
    out = torch.empty_like(x)
    check(_lib.load().dfc_masked_fill(_ptr(x), _ptr(d), _ptr(out), B, H, W, _stream()))
    return _out(out, sq)


def extend_to_top(t: torch.Tensor) -> torch.Tensor:
    x, sq = _as_batch(t)
    B, H, W = x.shape
    out = torch.empty_like(x)
    check(_lib.load().dfc_extend_to_top(_ptr(x), _ptr(out), B, H, W, _stream()))
    return _out(out, sq)


def count_empty(t: torch.Tensor) -> torch.Tensor:
    x, _ = _as_batch(t)
    B, H, W = x.shape
    c = torch.empty(B, dtype=torch.int64, device=x.device)
    check(_lib.load().dfc_count_empty(_ptr(x), B, H, W, _ptr(c), _stream()))
    return c


def reimpose(blurred: torch.Tensor, mask_src: torch.Tensor) -> torch.Tensor:
    b, sq = _as_batch(blurred)
    m, _ = _as_batch(mask_src)
    B, H, W = b.shape
    out = torch.empty_like(b)
    check(_lib.load().dfc_reimpose(_ptr(b), _ptr(m), _ptr(out), B, H, W, _stream()))
    return _out(out, sq)


# ---------------------------------------------------------------------------
# fused batch pipeline
# ---------------------------------------------------------------------------

@dataclass
class FillResult:
    dense: torch.Tensor        # [B, H, W] float32, direct encoding
    status: torch.Tensor       # [B] int32 DFC_ST_* bits
    iterations: torch.Tensor   # [B] int32 large-fill iterations
    valid_counts: torch.Tensor | None = None  # [B, 2] int32: input / output pixels > 0.1 (RunStats densities)

    def densities(self) -> tuple[np.ndarray, np.ndarray]:
        """RunStats.input_density / output_density per frame (pipeline.py:138-141, 192-202)."""
        if self.valid_counts is None:
            raise ValueError("no valid-pixel counts for this result")
        n = self.dense.shape[-1] * self.dense.shape[-2]
        c = self.valid_counts.cpu().numpy().astype(np.int64)
        return c[:, 0] / n, c[:, 1] / n


class Workspace:
    """Device workspace for dfc_fill_batch, grown on demand.

    A workspace belongs to one stream at a time: the library keeps per-call
    counters in it (work queue, fallback count, validation maxima), so two
    calls in flight on different streams must not share one.  The default
    workspaces are therefore keyed by (device, stream) and locked for the
    duration of a call; a buffer dropped on growth is first recorded on the
    stream that last used it, so the caching allocator cannot hand it out
    while that stream's kernels may still read it.
    """

    def __init__(self):
        self.buf = None
        self.stream = None  # the stream of the last call that used buf
        self.lock = threading.Lock()

    def get(self, nbytes: int, device) -> torch.Tensor:
        """The buffer for a call about to run on torch's current stream of ``device``."""
        cur = torch.cuda.current_stream(device)
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            if self.buf is not None and self.stream is not None:
                self.buf.record_stream(self.stream)
            self.buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        elif self.stream is not None and self.stream != cur:
            # reused on another stream: keep the allocator from recycling it
            # while the earlier stream may still be running on it
            self.buf.record_stream(cur)
            cur.wait_stream(self.stream)
        self.stream = cur
        return self.buf


_default_ws: dict = {}
_default_ws_lock = threading.Lock()


def _workspace_for(device) -> Workspace:
    """The default workspace of (device, current stream)."""
    key = (device, torch.cuda.current_stream(device).cuda_stream)
    with _default_ws_lock:
        ws = _default_ws.get(key)
        if ws is None:
            ws = _default_ws[key] = Workspace()
    return ws


def fill_batch(frames: torch.Tensor, cfg: "_lib.DfcConfig", out: torch.Tensor | None = None,
               workspace: Workspace | None = None, status: torch.Tensor | None = None,
               iterations: torch.Tensor | None = None, counts: bool = True) -> FillResult:
    """Run the depth-completion pipeline on B frames via dfc_fill_batch (and
    dfc_fill_counts for the per-frame valid-pixel counts unless counts=False)."""
    x, _ = _as_batch(frames)
    B, H, W = x.shape
    L = _lib.load()
    need = int(L.dfc_workspace_bytes(ctypes.byref(cfg), B, H, W))
    if need == 0:
        # invalid config: let dfc_fill_batch report the reason
        check(L.dfc_fill_batch(None, None, B, H, W, ctypes.byref(cfg), None, None, None, 0, _stream()))
    if workspace is None:
        workspace = _workspace_for(x.device)
    if out is None:
        out = torch.empty_like(x)
    if status is None:
        status = torch.empty(B, dtype=torch.int32, device=x.device)
    if iterations is None:
        iterations = torch.empty(B, dtype=torch.int32, device=x.device)
    vc = torch.empty((B, 2), dtype=torch.int32, device=x.device) if counts else None
    with workspace.lock:
        ws = workspace.get(need, x.device)
        check(L.dfc_fill_batch(_ptr(x), _ptr(out), B, H, W, ctypes.byref(cfg), _ptr(status), _ptr(iterations),
                               _ptr(ws), ws.numel(), _stream()))
        if counts and B > 0 and not (cfg.flags & _lib.F_NO_FINISH):
            check(L.dfc_fill_counts(ctypes.byref(cfg), B, H, W, _ptr(ws), ws.numel(), _ptr(vc), _stream()))
    return FillResult(out, status, iterations, vc if counts and not (cfg.flags & _lib.F_NO_FINISH) else None)


# ---------------------------------------------------------------------------
# KITTI 16-bit raw at the boundary (kitti_io.py:36-66)
# ---------------------------------------------------------------------------

def fill_batch_raw16(raw: torch.Tensor, cfg: "_lib.DfcConfig", out_raw: bool = True,
                     workspace: Workspace | None = None, out: torch.Tensor | None = None,
                     status: torch.Tensor | None = None, iterations: torch.Tensor | None = None) -> FillResult:
    """dfc_fill_batch_raw16: uint16 raw frames in; uint16 raw (or float32 depth) out."""
    if raw.dtype != torch.uint16:
        raise TypeError("raw frames must be torch.uint16")
    x = raw.contiguous()
    if x.dim() == 2:
        x = x.unsqueeze(0)
    B, H, W = x.shape
    L = _lib.load()
    need = int(L.dfc_workspace_bytes_raw16(ctypes.byref(cfg), B, H, W))
    if need == 0:
        check(L.dfc_fill_batch_raw16(None, None, int(out_raw), B, H, W, ctypes.byref(cfg), None, None, None, 0,
                                     _stream()))
    if workspace is None:
        workspace = _workspace_for(x.device)
    if out is None:
        out = torch.empty(x.shape, dtype=torch.uint16 if out_raw else torch.float32, device=x.device)
    if status is None:
        status = torch.empty(B, dtype=torch.int32, device=x.device)
    if iterations is None:
        iterations = torch.empty(B, dtype=torch.int32, device=x.device)
    with workspace.lock:
        ws = workspace.get(need, x.device)
        check(L.dfc_fill_batch_raw16(_ptr(x), _ptr(out), int(out_raw), B, H, W, ctypes.byref(cfg), _ptr(status),
                                     _ptr(iterations), _ptr(ws), ws.numel(), _stream()))
    return FillResult(out, status, iterations)


def decode_raw16(raw: torch.Tensor) -> torch.Tensor:
    """depth = raw / 256 (kitti_io.py:53), exact."""
    x = raw.contiguous()
    out = torch.empty(x.shape, dtype=torch.float32, device=x.device)
    check(_lib.load().dfc_decode_raw16(_ptr(x), _ptr(out), x.numel(), _stream()))
    return out


def encode_raw16(depth: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """raw = rint(depth * 256) clipped (kitti_io.py:62-65); per-frame status (DFC_ST_ENCODE if any >= 256 m)."""
    x, _ = _as_batch(depth)
    B = x.shape[0]
    out = torch.empty(x.shape, dtype=torch.uint16, device=x.device)
    status = torch.zeros(B, dtype=torch.int32, device=x.device)
    check(_lib.load().dfc_encode_raw16(_ptr(x), _ptr(out), B, x[0].numel(), _ptr(status), _stream()))
    return out.reshape(depth.shape), status

