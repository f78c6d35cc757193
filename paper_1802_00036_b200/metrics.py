"""Depth-completion error metrics on the GPU.

Mirrors the reference's `depthfill.metrics` (metrics.py:1-149): RMSE / MAE in
mm and iRMSE / iMAE in 1/km over pixels where both prediction and ground truth
are valid (> 0.1f); ground-truth-valid pixels the prediction leaves empty are
counted as skipped; dataset numbers aggregate per pixel (sums, then finalize).
The per-frame float64 sums run in one CUDA kernel per batch (csrc/metrics.cu,
`dfc_error_sums`); `finalize` is the reference's arithmetic on the host.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .completion import _device
from .domain import DepthEncoding, DepthMap, EncodingError
from .ops import _ptr, _stream

_M_TO_MM = 1000.0
_INV_M_TO_INV_KM = 1000.0


@dataclass(frozen=True)
class MetricsReport:
    """metrics.MetricsReport (metrics.py:27-54)."""

    rmse_mm: float
    mae_mm: float
    irmse_invkm: float
    imae_invkm: float
    evaluated_pixels: int
    skipped_pixels: int

    CSV_HEADER = "rmse_mm,mae_mm,irmse_invkm,imae_invkm,evaluated_pixels,skipped_pixels"

    def to_text(self) -> str:
        return (f"rmse_mm={self.rmse_mm:.6f}\nmae_mm={self.mae_mm:.6f}\nirmse_invkm={self.irmse_invkm:.6f}\n"
                f"imae_invkm={self.imae_invkm:.6f}\nevaluated_pixels={self.evaluated_pixels}\n"
                f"skipped_pixels={self.skipped_pixels}\n")

    def to_csv_row(self) -> str:
        return (f"{self.rmse_mm:.6f},{self.mae_mm:.6f},{self.irmse_invkm:.6f},{self.imae_invkm:.6f},"
                f"{self.evaluated_pixels},{self.skipped_pixels}")


def _as_batch(x) -> torch.Tensor:
    if isinstance(x, DepthMap):
        if x.encoding is not DepthEncoding.DIRECT:
            raise EncodingError("metrics expect direct-encoded maps")  # metrics.py:116-117
        x = x.values
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    if x.device.type != "cuda":
        x = x.to(_device())
    if x.dtype != torch.float32:  # the kernels read float32 (metrics.py:110-117 works on float32 maps)
        x = x.to(torch.float32)
    x = x.contiguous()
    return x.unsqueeze(0) if x.dim() == 2 else x


def _pair(pred, gt) -> tuple[torch.Tensor, torch.Tensor]:
    p, g = _as_batch(pred), _as_batch(gt)
    if p.shape != g.shape:  # metrics._check_pair (metrics.py:110-117)
        raise ValueError(f"dimension mismatch: prediction {p.shape[-1]}x{p.shape[-2]} vs "
                         f"ground truth {g.shape[-1]}x{g.shape[-2]}")
    return p, g


def error_sums(pred, gt) -> tuple[np.ndarray, np.ndarray]:
    """Per-frame [B, 4] float64 sums (sq, abs, inv_sq, inv_abs) and [B, 2] counts (evaluated, skipped)."""
    p, g = _pair(pred, gt)
    B, H, W = p.shape
    sums = torch.empty((B, 4), dtype=torch.float64, device=p.device)
    counts = torch.empty((B, 2), dtype=torch.int64, device=p.device)
    _lib.check(_lib.load().dfc_error_sums(_ptr(p), _ptr(g), B, H, W, _ptr(sums), _ptr(counts), _stream()))
    return sums.cpu().numpy(), counts.cpu().numpy()


def _finalize(sum_sq, sum_abs, sum_inv_sq, sum_inv_abs, n, skipped) -> MetricsReport:
    """metrics._finalize (metrics.py:140-149)."""
    return MetricsReport(rmse_mm=float(np.sqrt(sum_sq / n) * _M_TO_MM), mae_mm=float(sum_abs / n * _M_TO_MM),
                         irmse_invkm=float(np.sqrt(sum_inv_sq / n) * _INV_M_TO_INV_KM),
                         imae_invkm=float(sum_inv_abs / n * _INV_M_TO_INV_KM), evaluated_pixels=int(n),
                         skipped_pixels=int(skipped))


def evaluate(pred, gt) -> MetricsReport:
    """metrics.evaluate (metrics.py:93-98) for one pair."""
    s, c = error_sums(pred, gt)
    if s.shape[0] != 1:
        raise ValueError("evaluate takes one frame; use evaluate_batch or MetricsAccumulator")
    if c[0, 0] == 0:
        raise ValueError("prediction and ground truth share no valid pixels")
    return _finalize(*s[0], c[0, 0], c[0, 1])


def evaluate_batch(pred, gt) -> list[MetricsReport]:
    """evaluate() per frame of a [B, H, W] batch (one kernel launch)."""
    s, c = error_sums(pred, gt)
    out = []
    for b in range(s.shape[0]):
        if c[b, 0] == 0:
            raise ValueError(f"prediction and ground truth share no valid pixels (frame {b})")
        out.append(_finalize(*s[b], c[b, 0], c[b, 1]))
    return out


def error_map(pred, gt) -> torch.Tensor:
    """metrics.error_map (metrics.py:101-108): |pred - gt| where both valid, 0 elsewhere."""
    p, g = _pair(pred, gt)
    B, H, W = p.shape
    out = torch.empty_like(p)
    _lib.check(_lib.load().dfc_error_map(_ptr(p), _ptr(g), _ptr(out), B, H, W, _stream()))
    return out


class MetricsAccumulator:
    """metrics.MetricsAccumulator (metrics.py:56-90): per-pixel dataset aggregation."""

    def __init__(self):
        self.sum_sq = self.sum_abs = self.sum_inv_sq = self.sum_inv_abs = 0.0
        self.evaluated = self.skipped = 0

    def add(self, pred, gt) -> None:
        """Add one frame or a [B, H, W] batch (frames are added in order)."""
        s, c = error_sums(pred, gt)
        for b in range(s.shape[0]):
            self.sum_sq += float(s[b, 0])
            self.sum_abs += float(s[b, 1])
            self.sum_inv_sq += float(s[b, 2])
            self.sum_inv_abs += float(s[b, 3])
            self.evaluated += int(c[b, 0])
            self.skipped += int(c[b, 1])

    def finalize(self) -> MetricsReport:
        if self.evaluated == 0:
            raise ValueError("no overlapping valid pixels were accumulated")
        return _finalize(self.sum_sq, self.sum_abs, self.sum_inv_sq, self.sum_inv_abs, self.evaluated, self.skipped)


__all__ = ["MetricsReport", "MetricsAccumulator", "evaluate", "evaluate_batch", "error_map", "error_sums"]
