"""Host-side value types mirroring the reference's public types.

Mirrors (same names, argument meaning and exceptions):
  depth_core.py:17-167  VALIDITY_THRESHOLD, INVERSION_OFFSET, DepthEncoding,
                        EncodingError, DepthRangeError, DepthMap, ValidityMask,
                        new_depth_map, validity_mask, density
  kernels.py:15-78      KernelShape, Kernel, make_kernel, kernel_offsets
  pipeline.py:44-45     DegenerateInputError

Only validation and bookkeeping live here; all pixel work runs in libdfc.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

VALIDITY_THRESHOLD = 0.1      # compared as float32(0.1) against float32 maps
INVERSION_OFFSET = 100.0      # BASELINE "max_depth" default
_MAX_PIXELS = 2 ** 31


class DepthEncoding(Enum):
    DIRECT = "direct"
    INVERTED = "inverted"


class EncodingError(ValueError):
    """Operation applied to a map in the wrong encoding (depth_core.py:38-39)."""


class DepthRangeError(ValueError):
    """Depth values outside the invertible range (depth_core.py:42-43)."""


class DegenerateInputError(ValueError):
    """Input with no valid pixels (pipeline.py:44-45)."""


def _checked_array(values) -> np.ndarray:
    """The DepthMap constructor checks, in the reference's order."""
    a = np.asarray(values)
    if a.ndim != 2:
        raise ValueError(f"depth map must be 2-D, got shape {a.shape}")
    rows, cols = a.shape
    if rows < 1 or cols < 1:
        raise ValueError(f"depth map dimensions must be >= 1, got {cols}x{rows}")
    if rows * cols > _MAX_PIXELS:
        raise ValueError(f"depth map dimensions {cols}x{rows} exceed supported size")
    a = np.ascontiguousarray(a, dtype=np.float32)
    if not np.isfinite(a).all():
        raise ValueError("depth values must be finite")
    if (a < 0).any():
        raise ValueError("depth values must be non-negative")
    return a


@dataclass(frozen=True, eq=False)
class DepthMap:
    """Immutable float32 [H, W] depth grid with its encoding tag."""

    values: np.ndarray = field(repr=False)
    encoding: DepthEncoding = DepthEncoding.DIRECT

    def __post_init__(self):
        a = _checked_array(self.values)
        if a is self.values:
            a = a.copy()
        a.setflags(write=False)
        object.__setattr__(self, "values", a)

    @classmethod
    def _wrap(cls, values: np.ndarray, encoding: DepthEncoding) -> "DepthMap":
        obj = object.__new__(cls)
        values.setflags(write=False)
        object.__setattr__(obj, "values", values)
        object.__setattr__(obj, "encoding", encoding)
        return obj

    @classmethod
    def coerce(cls, m) -> "DepthMap":
        """Accept our DepthMap, the reference's DepthMap (duck-typed) or an array."""
        if isinstance(m, DepthMap):
            return m
        if hasattr(m, "values") and hasattr(m, "encoding"):
            enc = DepthEncoding(getattr(m.encoding, "value", m.encoding))
            return cls(np.asarray(m.values), enc)
        return cls(m)

    @property
    def width(self) -> int:
        return self.values.shape[1]

    @property
    def height(self) -> int:
        return self.values.shape[0]

    def __repr__(self):
        return f"DepthMap({self.width}x{self.height}, {self.encoding.value})"


@dataclass(frozen=True, eq=False)
class ValidityMask:
    bits: np.ndarray = field(repr=False)

    def __post_init__(self):
        b = np.ascontiguousarray(self.bits, dtype=bool)
        b.setflags(write=False)
        object.__setattr__(self, "bits", b)

    @property
    def width(self) -> int:
        return self.bits.shape[1]

    @property
    def height(self) -> int:
        return self.bits.shape[0]


def new_depth_map(width: int, height: int) -> DepthMap:
    width, height = int(width), int(height)
    if width < 1 or height < 1:
        raise ValueError(f"dimensions must be >= 1, got {width}x{height}")
    if width * height > _MAX_PIXELS:
        raise ValueError(f"dimensions {width}x{height} exceed supported size")
    return DepthMap(np.zeros((height, width), dtype=np.float32))


def validity_mask(depth_map: DepthMap) -> ValidityMask:
    return ValidityMask(depth_map.values > np.float32(VALIDITY_THRESHOLD))


def density(depth_map: DepthMap) -> float:
    v = depth_map.values > np.float32(VALIDITY_THRESHOLD)
    return float(np.count_nonzero(v)) / v.size


# ---------------------------------------------------------------------------
# structuring elements (kernels.py)
# ---------------------------------------------------------------------------

class KernelShape(Enum):
    FULL = "full"
    CIRCLE = "circle"
    CROSS = "cross"
    DIAMOND = "diamond"


@dataclass(frozen=True, eq=False)
class Kernel:
    """Centred k x k boolean footprint."""

    bits: np.ndarray = field(repr=False)

    def __post_init__(self):
        b = np.ascontiguousarray(self.bits, dtype=bool)
        if b.ndim != 2 or b.shape[0] != b.shape[1] or b.shape[0] % 2 == 0:
            raise ValueError("kernel must be a square boolean array of odd size")
        b.setflags(write=False)
        object.__setattr__(self, "bits", b)

    @property
    def size(self) -> int:
        return self.bits.shape[0]

    @property
    def is_full(self) -> bool:
        return bool(self.bits.all())

    def named(self):
        """(shape, size) if this footprint is one of the Fig. 3 shapes, else None."""
        for s in (KernelShape.DIAMOND, KernelShape.FULL, KernelShape.CROSS, KernelShape.CIRCLE):
            if self.size >= 3 and np.array_equal(make_kernel(s, self.size).bits, self.bits):
                return s, self.size
        return None

    def __repr__(self):
        return f"Kernel({self.size}x{self.size}, popcount={int(self.bits.sum())})"


def _footprint(shape: KernelShape, size: int) -> np.ndarray:
    half = size // 2
    off = np.abs(np.arange(size) - half)
    ay, ax = off[:, None], off[None, :]
    if shape is KernelShape.FULL:
        return np.ones((size, size), dtype=bool)
    if shape is KernelShape.DIAMOND:
        return ay + ax <= half
    if shape is KernelShape.CROSS:
        return (ay == 0) | (ax == 0)
    if shape is KernelShape.CIRCLE:
        return 4 * (ay * ay + ax * ax) <= size * size
    raise ValueError(f"unknown kernel shape: {shape!r}")


def make_kernel(shape: KernelShape, size: int) -> Kernel:
    """Fig. 3 structuring element at an odd size >= 3 (kernels.py:45-71)."""
    size = int(size)
    if size < 3 or size % 2 == 0:
        raise ValueError(f"kernel size must be odd and >= 3, got {size}")
    return Kernel(_footprint(KernelShape(shape), size))


def kernel_offsets(kernel: Kernel) -> np.ndarray:
    """(n, 2) int32 (dy, dx) offsets of the set bits, row-major (kernels.py:74-78)."""
    ys, xs = np.nonzero(kernel.bits)
    half = kernel.size // 2
    return np.ascontiguousarray(np.stack([ys - half, xs - half], axis=1).astype(np.int32))
