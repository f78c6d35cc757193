"""Seeded synthetic sparse-LIDAR depth frames.

KITTI is not available in this environment, so every benchmark and parity
case uses these frames instead: a ground plane whose depth falls linearly from
``far_m`` at the top LIDAR row to 3 m at the bottom row, 5-15 axis-aligned
boxes (occlusion = min depth), sampled along ``beams`` near-horizontal
scanlines with a random-phase sinusoidal wobble, per-sample keep probability
``density * H / beams``, N(0, 0.02^2) noise, clipped to
[0.5, max_depth - 0.2].  Frame ``i`` of config ``c`` is seeded by
``SeedSequence([c, i])`` so any frame can be regenerated on the CPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SynthSpec:
    width: int = 1216
    height: int = 352
    beams: int = 64
    density: tuple[float, float] = (0.05, 0.05)  # U(lo, hi) whole-frame valid fraction
    max_depth: float = 100.0
    far_m: float = 80.0
    box_depth: tuple[float, float] = (5.0, 40.0)
    noise_m: float = 0.02


# BASELINE.json configs 0..4.
CONFIG_SPECS = {
    0: SynthSpec(),
    1: SynthSpec(density=(0.04, 0.06)),
    2: SynthSpec(density=(0.04, 0.06)),
    3: SynthSpec(width=1242, height=375),
    4: SynthSpec(width=4096, height=1024, beams=128, density=(0.02, 0.02), max_depth=120.0,
                 far_m=115.0, box_depth=(0.5, 60.0)),
}


def make_frame(spec: SynthSpec, seed) -> np.ndarray:
    """One float32 [H, W] frame in meters, 0.0 = empty."""
    rng = np.random.default_rng(np.random.SeedSequence(seed))
    W, H, L = spec.width, spec.height, spec.beams
    y0 = int(round(120 * H / 352))
    density = rng.uniform(*spec.density) if spec.density[0] != spec.density[1] else spec.density[0]

    # scene: ground plane + boxes (min = occlusion)
    rows = np.arange(H, dtype=np.float64)
    ground = spec.far_m + (3.0 - spec.far_m) * (rows - y0) / max(H - 1 - y0, 1)
    scene = np.repeat(ground[:, None], W, axis=1)
    n_boxes = int(rng.integers(5, 16))
    for _ in range(n_boxes):
        bw = rng.uniform(W / 40, W / 6)
        bh = rng.uniform((H - y0) / 6, (H - y0) * 0.8)
        bx = rng.uniform(-bw / 2, W - bw / 2)
        by = rng.uniform(y0 + (H - y0) / 3, H)  # bottom edge
        d = rng.uniform(*spec.box_depth)
        x_lo, x_hi = int(max(bx, 0)), int(min(bx + bw, W))
        y_lo, y_hi = int(max(by - bh, 0)), int(min(by, H))
        if x_hi > x_lo and y_hi > y_lo:
            blk = scene[y_lo:y_hi, x_lo:x_hi]
            np.minimum(blk, d, out=blk)

    # scanlines
    base = y0 + np.arange(L) * (H - 1 - y0) / max(L - 1, 1)
    amp = rng.uniform(0.5, 2.0, size=L)
    period = rng.uniform(W / 4, W, size=L)
    phase = rng.uniform(0, 2 * np.pi, size=L)
    xs = np.arange(W, dtype=np.float64)
    beam_rows = np.rint(base[:, None] + amp[:, None] * np.sin(2 * np.pi * xs[None, :] / period[:, None]
                                                               + phase[:, None]))
    beam_rows = np.clip(beam_rows, y0, H - 1).astype(np.int64)
    p = min(1.0, density * H / L)
    keep = rng.random((L, W)) < p
    noise = rng.normal(0.0, spec.noise_m, size=(L, W))

    out = np.zeros((H, W), dtype=np.float32)
    r = beam_rows[keep]
    c = np.broadcast_to(xs.astype(np.int64)[None, :], (L, W))[keep]
    d = scene[r, c] + noise[keep]
    d = np.clip(d, 0.5, spec.max_depth - 0.2)
    out[r, c] = d.astype(np.float32)
    return out


def make_batch(config: int, start: int, count: int, spec: SynthSpec | None = None) -> np.ndarray:
    """Frames ``start .. start+count-1`` of ``config`` as a [count, H, W] array."""
    spec = spec or CONFIG_SPECS[config]
    out = np.empty((count, spec.height, spec.width), dtype=np.float32)
    for k in range(count):
        out[k] = make_frame(spec, [config, start + k])
    return out
