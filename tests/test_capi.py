"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/dfc.h declares, the ctypes struct mirrors dfc_config, and argument
validation fails loudly before any CUDA call."""

import ctypes
import re
import subprocess
import textwrap
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HDR = ROOT / "include" / "dfc.h"


@pytest.fixture(scope="module")
def L():
    from paper_1802_00036_b200 import _lib, build

    build.build()
    return _lib.load()


def declared_symbols():
    txt = HDR.read_text()
    return sorted(set(re.findall(r"^\s*(?:[a-z_0-9 ]+\*?\s+\**)(dfc_[a-z_0-9]+)\(", txt, re.M)))


def test_header_declares_expected(L):
    from paper_1802_00036_b200 import _lib

    syms = declared_symbols()
    assert len(syms) >= 20
    assert set(syms) == set(_lib.EXPORTS)


def test_library_exports_every_symbol(L):
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_1802_00036_b200" / "libdfc.so")],
                         capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), f"{s} not exported"


def test_sm100a_code_present():
    out = subprocess.run(["cuobjdump", "--list-elf", str(ROOT / "paper_1802_00036_b200" / "libdfc.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_c(tmp_path, L):
    from paper_1802_00036_b200 import _lib

    src = tmp_path / "lay.c"
    fields = [f for f, _ in _lib.DfcConfig._fields_]
    body = "\n".join(f'  printf("%s %zu\\n", "{f}", offsetof(dfc_config, {f}));' for f in fields)
    src.write_text(textwrap.dedent(f"""
        #include <stdio.h>
        #include <stddef.h>
        #include "dfc.h"
        int main(void) {{
          printf("sizeof %zu\\n", sizeof(dfc_config));
        {body}
          return 0;
        }}
    """))
    exe = tmp_path / "lay"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = dict(ln.split() for ln in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    assert int(got["sizeof"]) == ctypes.sizeof(_lib.DfcConfig)
    for f in fields:
        assert int(got[f]) == getattr(_lib.DfcConfig, f).offset, f


def test_config_defaults(L):
    from paper_1802_00036_b200 import _lib

    c = _lib.DfcConfig()
    assert L.dfc_config_init(ctypes.byref(c)) == 0
    assert (c.dilation_shape, c.dilation_size, c.closure_size, c.small_fill_size, c.large_fill_size) == (3, 5, 5, 7, 31)
    assert c.large_fill_max_iters == 100 and c.blur_mode == 5 and c.fill_mode == 0
    assert c.gaussian_sigma == 1.1 and c.max_depth == 100.0


def test_invalid_arguments_rejected_without_gpu(L):
    from paper_1802_00036_b200 import _lib

    c = _lib.DfcConfig()
    L.dfc_config_init(ctypes.byref(c))
    c.dilation_size = 4
    rc = L.dfc_fill_batch(None, None, 1, 10, 10, ctypes.byref(c), None, None, None, 0, None)
    assert rc == _lib.DFC_E_INVALID
    assert b"dilation_size must be an odd integer >= 3, got 4" in L.dfc_last_error_string()
    L.dfc_config_init(ctypes.byref(c))
    assert L.dfc_fill_batch(None, None, 1, 0, 10, ctypes.byref(c), None, None, None, 0, None) == _lib.DFC_E_INVALID
    assert L.dfc_workspace_bytes(ctypes.byref(c), 4, 352, 1216) > 0
    # a batch of zero frames is a no-op
    assert L.dfc_fill_batch(None, None, 0, 352, 1216, ctypes.byref(c), None, None, None, 0, None) == 0
    # workspace too small is reported, not a crash
    assert L.dfc_fill_batch(ctypes.c_void_p(16), ctypes.c_void_p(16), 1, 352, 1216, ctypes.byref(c),
                            ctypes.c_void_p(16), None, None, 0, None) == _lib.DFC_E_WORKSPACE
    assert L.dfc_median(ctypes.c_void_p(16), ctypes.c_void_p(16), 1, 4, 4, 4, None) == _lib.DFC_E_INVALID
