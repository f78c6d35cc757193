"""The reference's compiled operator surface (oracle/_ref, built by
oracle/build_ref.sh from /root/reference/.../_native_ops.pyx) behind the same
7-function interface as the numpy oracle -- TEST/BASELINE INFRASTRUCTURE ONLY.

The shipped adapter (_native.py:16-30) cannot be used through the public API:
DepthMap arrays and ``median_pairs`` are read-only while the Cython entry
points take non-const memoryviews (SURVEY.md finding 4).  This shim passes
writable copies, exactly the "test-harness shim" of SURVEY.md 8(c) path 2.
"""

from __future__ import annotations

import importlib.machinery
import importlib.util
import sysconfig
from functools import lru_cache
from pathlib import Path

import numpy as np

_REF_DIR = Path(__file__).resolve().parent / "_ref"
_SO = _REF_DIR / ("_native_ops" + sysconfig.get_config_var("EXT_SUFFIX"))


def _cpu_ok() -> bool:
    """The .so is built for x86-64-v3 (AVX2/FMA/BMI2)."""
    try:
        flags = Path("/proc/cpuinfo").read_text()
    except OSError:
        return False
    return all(f in flags for f in (" avx2", " fma", " bmi2"))


@lru_cache(maxsize=None)
def load_native():
    """Return the compiled reference module, or None if unavailable."""
    if not _SO.exists() or not _cpu_ok():
        return None
    loader = importlib.machinery.ExtensionFileLoader("_native_ops", str(_SO))
    spec = importlib.util.spec_from_file_location("_native_ops", str(_SO), loader=loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    return mod


# --- median comparator network (restates _sorting_networks.py:17-57) --------

def _oddeven_merge_sort_pairs(n: int) -> list[tuple[int, int]]:
    """Batcher odd-even mergesort comparators for a power-of-two n."""
    pairs = []
    p = 1
    while p < n:
        k = p
        while k >= 1:
            j = k % p
            while j < n - k:
                for i in range(min(k, n - j - k)):
                    if (i + j) // (2 * p) == (i + j + k) // (2 * p):
                        pairs.append((i + j, i + j + k))
                j += 2 * k
            k //= 2
        p *= 2
    return pairs


@lru_cache(maxsize=None)
def median_network(n: int) -> np.ndarray:
    """Comparators placing the median of n inputs on wire n//2: the pruned
    power-of-two network restricted to the median's dependency cone."""
    n2 = 1 << (n - 1).bit_length()
    pairs = [(a, b) for (a, b) in _oddeven_merge_sort_pairs(n2) if b < n]
    need = {n // 2}
    keep = []
    for a, b in reversed(pairs):
        if a in need or b in need:
            keep.append((a, b))
            need.update((a, b))
    keep.reverse()
    return np.array(keep, dtype=np.int32)


class RefNativeOps:
    """_native.py surface over the compiled reference (writable-copy shim)."""

    NAME = "reference-native"

    @staticmethod
    def _w(v):
        return np.array(v, dtype=np.float32, copy=True, order="C")

    @classmethod
    def box_max(cls, v, radius):
        return load_native().box_max(cls._w(v), int(radius))

    @classmethod
    def box_min(cls, v, radius):
        return load_native().box_min(cls._w(v), int(radius))

    @classmethod
    def offsets_max(cls, v, offsets):
        return load_native().offsets_max(cls._w(v), np.array(offsets, dtype=np.int32, copy=True))

    @classmethod
    def offsets_min(cls, v, offsets):
        return load_native().offsets_min(cls._w(v), np.array(offsets, dtype=np.int32, copy=True))

    @classmethod
    def median_filter(cls, v, size):
        nat = load_native()
        if size in (3, 5):
            return nat.median_network(cls._w(v), int(size), median_network(size * size).copy())
        return nat.median_generic(cls._w(v), int(size))

    @classmethod
    def gaussian_separable(cls, v, weights):
        return load_native().gaussian_separable(cls._w(v), np.array(weights, dtype=np.float64, copy=True))

    @classmethod
    def bilateral_filter(cls, v, size, sigma_value, sigma_space):
        return load_native().bilateral_filter(cls._w(v), int(size), float(sigma_value), float(sigma_space))
