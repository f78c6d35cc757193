"""Pin the CPU oracle to the reference: every golden vector produced by running
the unmodified reference (tests/golden/make_golden.py) must be reproduced
bit-for-bit by oracle/depthfill_oracle.py."""

import hashlib
import json

import numpy as np
import pytest

from oracle import depthfill_oracle as O
from paper_1802_00036_b200 import synth


def _bits_equal(a, b):
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.fixture(scope="module")
def ops_npz(golden_dir):
    return np.load(golden_dir / "ops_small.npz")


def test_ops_golden(ops_npz):
    keys = [k[3:] for k in ops_npz.files if k.startswith("in_")]
    assert len(keys) >= 18
    n_checked = 0
    for key in keys:
        v = ops_npz[f"in_{key}"]
        for r in (1, 2, 3, 15):
            assert _bits_equal(O.box_max(v, r), ops_npz[f"box_max_r{r}_{key}"])
            assert _bits_equal(O.box_min(v, r), ops_npz[f"box_min_r{r}_{key}"])
            n_checked += 2
        for shape in O.KernelShape:
            for size in (3, 5, 7):
                offs = O.kernel_offsets(O.make_kernel(shape, size))
                assert _bits_equal(O.offsets_max(v, offs), ops_npz[f"offs_max_{shape.value}{size}_{key}"])
                assert _bits_equal(O.offsets_min(v, offs), ops_npz[f"offs_min_{shape.value}{size}_{key}"])
                n_checked += 2
        for size in (3, 5, 7):
            assert _bits_equal(O.median_filter(v, size), ops_npz[f"median{size}_{key}"])
        for (size, sigma) in ((5, 1.1), (3, 0.8), (7, 2.0)):
            got = O.gaussian_separable(v, O.gaussian_weights(size, sigma))
            assert _bits_equal(got, ops_npz[f"gauss{size}_{sigma}_{key}"])
        for (size, sv, ss) in ((5, 1.5, 2.0), (3, 0.5, 1.0), (7, 3.0, 1.5)):
            got = O.bilateral_filter(v, size, sv, ss)
            assert _bits_equal(got, ops_npz[f"bilat{size}_{sv}_{ss}_{key}"])
    assert n_checked > 500


def test_stages_golden(golden_dir):
    z = np.load(golden_dir / "stages_small.npz")
    keys = [k[3:] for k in z.files if k.startswith("in_")]
    for key in keys:
        v = z[f"in_{key}"]
        inv = O.flip(v)
        assert _bits_equal(inv, z[f"invert_{key}"])
        assert _bits_equal(O.flip(inv), z[f"invert_back_{key}"])
        assert _bits_equal(O.extend_to_top(inv), z[f"extend_{key}"])
        for size in (3, 7, 31):
            k = f"mfill{size}_{key}"
            if k in z.files:
                assert _bits_equal(O.masked_fill_dilate(inv, O.make_kernel(O.KernelShape.FULL, size)), z[k])


def _cfg(kw, offset=100.0):
    conv = {"blur_mode": O.BlurMode, "fill_mode": O.FillMode, "dilation_shape": O.KernelShape}
    return O.OracleConfig(**{k: conv[k](x) if k in conv else x for k, x in kw.items()}, max_depth=offset)


def test_pipeline_small_golden(golden_dir):
    z = np.load(golden_dir / "pipeline_small.npz")
    meta = json.loads((golden_dir / "pipeline_small.json").read_text())
    assert len(meta) > 80
    errors = {"DegenerateInputError": O.DegenerateInputError, "DepthRangeError": O.DepthRangeError,
              "ValueError": ValueError}
    for m in meta:
        v = z[f"in_{m['key']}"]
        cfg = _cfg(m["cfg"], m["offset"])
        if m["error"]:
            with pytest.raises(errors[m["error"]]):
                O.complete_with_stats(v, cfg)
            continue
        dense, info = O.complete_with_stats(v, cfg)
        assert _bits_equal(dense, z[f"out_{m['key']}"]), m
        assert info["large_fill_iterations"] == m["iters"], m
        assert info["output_density"] == pytest.approx(m["out_density"], abs=0)


def test_single_pixel_kat(golden_dir):
    """a lone valid 50 m pixel -> every output pixel 50 m."""
    one = np.zeros((48, 128), np.float32)
    one[30, 77] = 50.0
    out = O.complete(one)
    assert np.all(out == np.float32(50.0))


def test_multiscale_composed_golden(golden_dir):
    z = np.load(golden_dir / "multiscale_small.npz")
    meta = json.loads((golden_dir / "multiscale_small.json").read_text())
    for m in meta:
        (sn, zn), (sm, zm), (sf, zf) = m["kernels"]
        ms = (tuple(m["edges"]), (O.KernelShape(sn), zn), (O.KernelShape(sm), zm), (O.KernelShape(sf), zf))
        cfg = O.OracleConfig(blur_mode=O.BlurMode(m["blur"]), multiscale=ms, max_depth=m["offset"])
        dense, info = O.complete_with_stats(z[f"in_{m['key']}"], cfg)
        assert _bits_equal(dense, z[f"out_{m['key']}"]), m
        assert info["large_fill_iterations"] == m["iters"]


def test_multiscale_equal_kernels_is_fast():
    """Max-merge definition: identical bin kernels reproduce fill_in_fast stage 2."""
    v = synth.make_frame(synth.SynthSpec(width=96, height=40, beams=12, density=(0.1, 0.1)), [7, 7])
    d5 = (O.KernelShape.DIAMOND, 5)
    cfg_ms = O.OracleConfig(multiscale=((15.0, 30.0), d5, d5, d5))
    assert _bits_equal(O.complete(v, cfg_ms), O.complete(v, O.OracleConfig()))


@pytest.mark.parametrize("case", range(6))
def test_pipeline_full_golden(golden_dir, case):
    meta = json.loads((golden_dir / "pipeline_full.json").read_text())[case]
    v = synth.make_frame(synth.CONFIG_SPECS[meta["config"]], [meta["config"], meta["frame"]])
    assert hashlib.sha256(v.tobytes()).hexdigest() == meta["input_sha256"], "generator drifted"
    dense, info = O.complete_with_stats(v, _cfg(meta["cfg"], meta["offset"]))
    assert hashlib.sha256(dense.tobytes()).hexdigest() == meta["output_sha256"]
    assert info["large_fill_iterations"] == meta["iters"]


def _ms_cfg(m):
    (sn, zn), (sm, zm), (sf, zf) = m["kernels"]
    ms = (tuple(m["edges"]), (O.KernelShape(sn), zn), (O.KernelShape(sm), zm), (O.KernelShape(sf), zf))
    return O.OracleConfig(blur_mode=O.BlurMode(m["blur"]), multiscale=ms, max_depth=m["offset"])


@pytest.mark.parametrize("case", range(3))
def test_multiscale_full_golden(golden_dir, case):
    """BASELINE config 2 / 4 full-size frames (4096x1024, max_depth 120 for config 4)
    through the composed multiscale oracle, pinned by SHA-256 to the composition of
    the reference's own primitives (make_golden.py: ref_multiscale)."""
    m = json.loads((golden_dir / "multiscale_full.json").read_text())[case]
    v = synth.make_frame(synth.CONFIG_SPECS[m["config"]], [m["config"], m["frame"]])
    assert hashlib.sha256(v.tobytes()).hexdigest() == m["input_sha256"], "generator drifted"
    dense, info = O.complete_with_stats(v, _ms_cfg(m))
    assert hashlib.sha256(dense.tobytes()).hexdigest() == m["output_sha256"]
    assert info["large_fill_iterations"] == m["iters"]


def test_metrics_oracle_matches_reference(golden_dir):
    """oracle/metrics_oracle.py against depthfill.metrics outputs."""
    from oracle import metrics_oracle as M

    z = np.load(golden_dir / "metrics_small.npz")
    meta = json.loads((golden_dir / "metrics_small.json").read_text())
    tot = np.zeros(4)
    n = s = 0
    for m in meta[:-1]:
        k = m["key"]
        sums = M.error_sums(z[f"pred_{k}"], z[f"gt_{k}"])
        assert list(sums) == m["sums"]
        assert list(M.finalize(*sums)) == m["report"]
        assert np.array_equal(M.error_map(z[f"pred_{k}"], z[f"gt_{k}"]), z[f"emap_{k}"])
        tot += np.array(sums[:4])
        n += sums[4]
        s += sums[5]
    assert list(M.finalize(*tot, n, s)) == meta[-1]["accumulated"]


def test_kitti_oracle_matches_reference_png_roundtrip(golden_dir):
    """decode / encode against kitti_io.write_depth_png -> read_depth_png through real PNG files."""
    from oracle import metrics_oracle as M

    z = np.load(golden_dir / "kitti_small.npz")
    for k in range(3):
        back = M.decode_raw16(M.encode_raw16(z[f"in_{k}"]))
        assert np.array_equal(back.view(np.uint32), z[f"back_{k}"].view(np.uint32))
    raw = np.arange(65536, dtype=np.uint16).reshape(256, 256)
    assert np.array_equal(M.decode_raw16(raw).view(np.uint32), z["all_raw_decoded"].view(np.uint32))


def test_colormap_oracle_matches_reference_png(golden_dir):
    """oracle colormap against kitti_io.write_colormap_png's PNG pixels."""
    from oracle import metrics_oracle as M

    z = np.load(golden_dir / "kitti_small.npz")
    for k in range(3):
        lo, hi = z[f"cmap_range_{k}"]
        assert np.array_equal(M.colormap(z[f"cmap_in_{k}"], float(lo), float(hi)), z[f"cmap_rgb_{k}"])
