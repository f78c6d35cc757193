"""CPU restatement of the reference's metrics and KITTI value conversion.

TEST INFRASTRUCTURE ONLY (the checker for tests/ -- never imported by the
product path).  Each function cites the reference line it follows; the
outputs are pinned against the unmodified reference by
tests/golden/make_golden.py (metrics_small.*, kitti_small.npz) and
tests/test_oracle_golden.py.
"""

from __future__ import annotations

import numpy as np

VALIDITY_THRESHOLD = 0.1  # depth_core.py:20 (compared as a weak scalar against float32 maps)
DEPTH_SCALE = 256.0       # kitti_io.py:22


def error_sums(pred: np.ndarray, gt: np.ndarray):
    """metrics._error_sums (metrics.py:119-137)."""
    if pred.shape != gt.shape:
        raise ValueError("dimension mismatch")
    gt_valid = gt > VALIDITY_THRESHOLD
    pred_valid = pred > VALIDITY_THRESHOLD
    both = gt_valid & pred_valid
    skipped = int(np.count_nonzero(gt_valid & ~pred_valid))
    d = pred[both].astype(np.float64)
    g = gt[both].astype(np.float64)
    err = d - g
    inv_err = 1.0 / d - 1.0 / g
    return (float(np.dot(err, err)), float(np.abs(err).sum()), float(np.dot(inv_err, inv_err)),
            float(np.abs(inv_err).sum()), int(both.sum()), skipped)


def finalize(sum_sq, sum_abs, sum_inv_sq, sum_inv_abs, n, skipped):
    """metrics._finalize (metrics.py:140-149): (rmse_mm, mae_mm, irmse_invkm, imae_invkm, n, skipped)."""
    return (float(np.sqrt(sum_sq / n) * 1000.0), float(sum_abs / n * 1000.0), float(np.sqrt(sum_inv_sq / n) * 1000.0),
            float(sum_inv_abs / n * 1000.0), int(n), int(skipped))


def error_map(pred: np.ndarray, gt: np.ndarray) -> np.ndarray:
    """metrics.error_map (metrics.py:101-108)."""
    both = (pred > VALIDITY_THRESHOLD) & (gt > VALIDITY_THRESHOLD)
    diff = np.abs(pred.astype(np.float64) - gt.astype(np.float64)).astype(np.float32)
    return np.where(both, diff, np.float32(0.0))


def decode_raw16(raw: np.ndarray) -> np.ndarray:
    """kitti_io.read_depth_png value conversion (kitti_io.py:53)."""
    return raw.astype(np.float32) / np.float32(DEPTH_SCALE)


def encode_raw16(values: np.ndarray) -> np.ndarray:
    """kitti_io.write_depth_png value conversion (kitti_io.py:60-65)."""
    if (values >= 256.0).any():
        raise ValueError("depth values must be < 256 m to be encodable")
    raw = np.rint(values.astype(np.float64) * DEPTH_SCALE)
    return np.clip(raw, 0, 65535).astype(np.uint16)


_RAMP_X = np.array([0.0, 0.25, 0.5, 0.75, 1.0])           # kitti_io.py:27
_RAMP = (np.array([0.0, 0.0, 0.0, 255.0, 255.0]),        # red    kitti_io.py:28
         np.array([0.0, 255.0, 255.0, 255.0, 0.0]),      # green  kitti_io.py:29
         np.array([255.0, 255.0, 0.0, 0.0, 0.0]))        # blue   kitti_io.py:30


def colormap(values: np.ndarray, range_min: float, range_max: float) -> np.ndarray:
    """kitti_io.write_colormap_png's pixel array (kitti_io.py:69-85), before PNG encoding."""
    if range_max <= range_min:
        raise ValueError(f"degenerate range [{range_min}, {range_max}]")
    t = np.clip((values.astype(np.float64) - range_min) / (range_max - range_min), 0.0, 1.0)
    rgb = np.stack([np.rint(np.interp(t, _RAMP_X, ch)) for ch in _RAMP], axis=-1).astype(np.uint8)
    rgb[values == 0.0] = 0
    return rgb

