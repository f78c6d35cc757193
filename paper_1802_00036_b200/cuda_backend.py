"""``cuda`` kernel backend for the reference's operator plug-in registry.

Implements the 7-function backend surface of the reference
(_numpy_ops.py:1-7, _native.py:16-30): 2-D C-contiguous float32 in, a fresh
float32 array out, replicate borders, read-only input never modified.  Each
call runs the matching libdfc kernel on the GPU.

Registration into an installed reference (no edit of its sources; SURVEY.md
8(b) probe 17):

    from depthfill import backend
    from paper_1802_00036_b200 import cuda_backend
    cuda_backend.register(backend)      # backend._BACKENDS["cuda"] = cuda_backend
    backend.set_backend("cuda")
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops

NAME = "cuda"


def _up(values: np.ndarray) -> torch.Tensor:
    if not torch.cuda.is_available():
        raise RuntimeError("cuda backend selected but no CUDA device is present")
    a = np.ascontiguousarray(values, dtype=np.float32)
    if a.ndim != 2:
        raise ValueError("backend ops take 2-D maps")
    return torch.from_numpy(a).cuda()


def _down(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


def box_max(values: np.ndarray, radius: int) -> np.ndarray:
    return _down(ops.box_max(_up(values), radius))


def box_min(values: np.ndarray, radius: int) -> np.ndarray:
    return _down(ops.box_min(_up(values), radius))


def offsets_max(values: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    return _down(ops.offsets_max(_up(values), offsets))


def offsets_min(values: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    return _down(ops.offsets_min(_up(values), offsets))


def median_filter(values: np.ndarray, size: int) -> np.ndarray:
    return _down(ops.median(_up(values), size))


def gaussian_separable(values: np.ndarray, weights: np.ndarray) -> np.ndarray:
    # fp64 in the reference's operation order: the backend surface promises the
    # numpy backend's arithmetic (_numpy_ops.py:61-73)
    return _down(ops.gaussian_separable(_up(values), weights, exact=True))


def bilateral_filter(values: np.ndarray, size: int, sigma_value: float, sigma_space: float) -> np.ndarray:
    return _down(ops.bilateral(_up(values), size, sigma_value, sigma_space, exact=True))


def register(backend_module, name: str = NAME) -> None:
    """Insert this module into a reference ``depthfill.backend`` registry."""
    import sys

    backend_module._BACKENDS[name] = sys.modules[__name__]
