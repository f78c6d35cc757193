"""ctypes binding of libdfc.so (include/dfc.h).

The library is built in-tree (``paper_1802_00036_b200/libdfc.so``) by
``build.py``.  There is no CPU fallback: if the shared library is missing or
no CUDA device is present, the product path raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libdfc.so"

DFC_OK = 0
DFC_E_INVALID = -1
DFC_E_CUDA = -2
DFC_E_WORKSPACE = -3
DFC_E_UNSUPPORTED = -4

ST_NONFINITE = 0x1
ST_NEGATIVE = 0x2
ST_DEGENERATE = 0x4
ST_RANGE = 0x8
ST_ENCODE = 0x10
ST_FALLBACK = 0x100

F_FORCE_STAGED = 0x1
F_EXACT_BLUR = 0x2
F_NO_FINISH = 0x4
F_SPARSE = 0x8  # performance hint: register-dense large fill (frames with many empties); results unchanged

SHAPE_CODES = {"full": 0, "circle": 1, "cross": 2, "diamond": 3}
BLUR_CODES = {"none": 0, "bilateral": 1, "median": 2, "median_bilateral": 3, "gaussian": 4,
              "median_gaussian": 5}
FILL_CODES = {"full": 0, "partial": 1}

# every symbol include/dfc.h declares
EXPORTS = (
    "dfc_abi_version", "dfc_last_error_string", "dfc_kernel_launches", "dfc_config_init", "dfc_workspace_bytes",
    "dfc_fill_batch", "dfc_fill_finish", "dfc_fill_counts", "dfc_op_workspace_bytes", "dfc_box_max", "dfc_box_min",
    "dfc_offsets_max", "dfc_offsets_min", "dfc_median", "dfc_gaussian_separable", "dfc_bilateral",
    "dfc_invert", "dfc_validate", "dfc_masked_fill", "dfc_extend_to_top", "dfc_count_empty",
    "dfc_reimpose", "dfc_workspace_bytes_raw16", "dfc_fill_batch_raw16", "dfc_decode_raw16", "dfc_encode_raw16",
    "dfc_error_sums", "dfc_error_map", "dfc_colormap",
)


class DfcConfig(ctypes.Structure):
    """Mirror of ``dfc_config`` (include/dfc.h)."""

    _fields_ = [
        ("dilation_shape", ctypes.c_int32),
        ("dilation_size", ctypes.c_int32),
        ("closure_size", ctypes.c_int32),
        ("small_fill_size", ctypes.c_int32),
        ("large_fill_size", ctypes.c_int32),
        ("large_fill_max_iters", ctypes.c_int32),
        ("blur_mode", ctypes.c_int32),
        ("median_size", ctypes.c_int32),
        ("gaussian_size", ctypes.c_int32),
        ("bilateral_size", ctypes.c_int32),
        ("gaussian_sigma", ctypes.c_double),
        ("bilateral_sigma_value", ctypes.c_double),
        ("bilateral_sigma_space", ctypes.c_double),
        ("fill_mode", ctypes.c_int32),
        ("max_depth", ctypes.c_float),
        ("multiscale", ctypes.c_int32),
        ("bin_edge_near", ctypes.c_float),
        ("bin_edge_far", ctypes.c_float),
        ("near_shape", ctypes.c_int32),
        ("near_size", ctypes.c_int32),
        ("med_shape", ctypes.c_int32),
        ("med_size", ctypes.c_int32),
        ("far_shape", ctypes.c_int32),
        ("far_size", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("custom_n", ctypes.c_int32),
        ("custom_offsets", ctypes.POINTER(ctypes.c_int32)),
    ]


class DfcError(RuntimeError):
    """A libdfc call failed (CUDA error, bad workspace, unsupported config)."""


_lib = None


def lib_path() -> Path:
    return Path(os.environ.get("DFC_LIB", str(LIB_PATH)))


def load(require: bool = True):
    """Load libdfc.so once; raise (never fall back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    p = lib_path()
    if not p.exists():
        if not require:
            return None
        raise ImportError(f"libdfc.so not built at {p}; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(str(p))
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    u32p = ctypes.c_void_p
    cfgp = ctypes.POINTER(DfcConfig)
    sig = {
        "dfc_abi_version": (ctypes.c_int, []),
        "dfc_last_error_string": (ctypes.c_char_p, []),
        "dfc_kernel_launches": (ctypes.c_ulonglong, []),
        "dfc_config_init": (ctypes.c_int, [cfgp]),
        "dfc_workspace_bytes": (sz, [cfgp, i64, i32, i32]),
        "dfc_fill_batch": (ctypes.c_int, [vp, vp, i64, i32, i32, cfgp, u32p, vp, vp, sz, vp]),
        "dfc_fill_finish": (ctypes.c_int, [vp, vp, i64, i32, i32, cfgp, u32p, vp, vp, sz, vp]),
        "dfc_fill_counts": (ctypes.c_int, [cfgp, i64, i32, i32, vp, sz, vp, vp]),
        "dfc_op_workspace_bytes": (sz, [i64, i32, i32]),
        "dfc_box_max": (ctypes.c_int, [vp, vp, i64, i32, i32, i32, vp, sz, vp]),
        "dfc_box_min": (ctypes.c_int, [vp, vp, i64, i32, i32, i32, vp, sz, vp]),
        "dfc_offsets_max": (ctypes.c_int, [vp, vp, i64, i32, i32, ctypes.POINTER(ctypes.c_int32), i32, vp]),
        "dfc_offsets_min": (ctypes.c_int, [vp, vp, i64, i32, i32, ctypes.POINTER(ctypes.c_int32), i32, vp]),
        "dfc_median": (ctypes.c_int, [vp, vp, i64, i32, i32, i32, vp]),
        "dfc_gaussian_separable": (ctypes.c_int, [vp, vp, i64, i32, i32, ctypes.POINTER(ctypes.c_double), i32,
                                                  i32, vp, sz, vp]),
        "dfc_bilateral": (ctypes.c_int, [vp, vp, i64, i32, i32, i32, ctypes.c_double, ctypes.c_double, i32, vp]),
        "dfc_invert": (ctypes.c_int, [vp, vp, i64, i32, i32, ctypes.c_float, vp, vp]),
        "dfc_validate": (ctypes.c_int, [vp, i64, i32, i32, vp, vp, vp]),
        "dfc_masked_fill": (ctypes.c_int, [vp, vp, vp, i64, i32, i32, vp]),
        "dfc_extend_to_top": (ctypes.c_int, [vp, vp, i64, i32, i32, vp]),
        "dfc_count_empty": (ctypes.c_int, [vp, i64, i32, i32, vp, vp]),
        "dfc_reimpose": (ctypes.c_int, [vp, vp, vp, i64, i32, i32, vp]),
        "dfc_workspace_bytes_raw16": (sz, [cfgp, i64, i32, i32]),
        "dfc_fill_batch_raw16": (ctypes.c_int, [vp, vp, i32, i64, i32, i32, cfgp, u32p, vp, vp, sz, vp]),
        "dfc_decode_raw16": (ctypes.c_int, [vp, vp, i64, vp]),
        "dfc_encode_raw16": (ctypes.c_int, [vp, vp, i64, i64, vp, vp]),
        "dfc_error_sums": (ctypes.c_int, [vp, vp, i64, i32, i32, vp, vp, vp]),
        "dfc_error_map": (ctypes.c_int, [vp, vp, vp, i64, i32, i32, vp]),
        "dfc_colormap": (ctypes.c_int, [vp, vp, i64, ctypes.c_double, ctypes.c_double, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.dfc_abi_version() != 1:
        raise ImportError("libdfc ABI version mismatch")
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a DFC_E_* return code to a Python exception."""
    if rc == DFC_OK:
        return
    msg = load().dfc_last_error_string().decode(errors="replace")
    if rc == DFC_E_INVALID:
        raise ValueError(msg)
    raise DfcError(f"libdfc error {rc}: {msg}")
