"""End-to-end GPU parity of the pipeline (fused and staged paths) against the
CPU oracle, which tests/test_oracle_golden.py pins to the reference.

Bar (BASELINE north_star): bit-exact for inversion, dilation, close, fills,
extrapolation and median; within 1e-4 m absolute for Gaussian / bilateral.
"""

import hashlib
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import depthfill_oracle as O  # noqa: E402
from paper_1802_00036_b200 import synth  # noqa: E402

TOL = 1e-4  # meters, Gaussian / bilateral (north_star)
BLURRY = {"gaussian", "median_gaussian", "bilateral", "median_bilateral"}


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_00036_b200 as pkg

    return pkg


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def _cmp(got, ref, blur):
    got = np.asarray(got, np.float32)
    ref = np.asarray(ref, np.float32)
    assert got.shape == ref.shape
    if blur in BLURRY:
        err = float(np.abs(got - ref).max())
        assert err <= TOL, f"max |err| {err}"
        # validity (empty vs filled) must agree exactly
        assert np.array_equal(got > np.float32(0.1), ref > np.float32(0.1))
    else:
        assert np.array_equal(_bits(got), _bits(ref)), "not bit-exact"


def _pcfg(P, kw, offset=100.0, exact=False):
    conv = {"blur_mode": P.BlurMode, "fill_mode": P.FillMode, "dilation_shape": P.KernelShape}
    return P.PipelineConfig(**{k: conv[k](x) if k in conv else x for k, x in kw.items()}, max_depth=offset,
                            exact_blur=exact)


def _ocfg(kw, offset=100.0):
    conv = {"blur_mode": O.BlurMode, "fill_mode": O.FillMode, "dilation_shape": O.KernelShape}
    return O.OracleConfig(**{k: conv[k](x) if k in conv else x for k, x in kw.items()}, max_depth=offset)


ERRORS = {"DegenerateInputError": "DegenerateInputError", "DepthRangeError": "DepthRangeError"}


@pytest.mark.parametrize("force_staged", [False, True])
def test_pipeline_small_golden(P, golden_dir, force_staged):
    z = np.load(golden_dir / "pipeline_small.npz")
    meta = json.loads((golden_dir / "pipeline_small.json").read_text())
    for m in meta:
        v = z[f"in_{m['key']}"]
        cfg = _pcfg(P, m["cfg"], m["offset"])
        if m["error"]:
            with pytest.raises(getattr(P, m["error"])):
                P.complete_batch(v[None], cfg, force_staged=force_staged)
            continue
        res = P.complete_batch(v[None], cfg, force_staged=force_staged)
        blur = m["cfg"].get("blur_mode", "median_gaussian")
        _cmp(res.dense[0].cpu().numpy(), z[f"out_{m['key']}"], blur)
        assert int(res.iterations[0]) == m["iters"], m


def test_pipeline_small_exact_blur_bit_exact(P, golden_dir):
    """fp64 exact-blur mode reproduces the reference Gaussian bit for bit."""
    z = np.load(golden_dir / "pipeline_small.npz")
    meta = json.loads((golden_dir / "pipeline_small.json").read_text())
    n = 0
    for m in meta:
        blur = m["cfg"].get("blur_mode", "median_gaussian")
        if m["error"] or "bilateral" in blur:
            continue
        v = z[f"in_{m['key']}"]
        res = P.complete_batch(v[None], _pcfg(P, m["cfg"], m["offset"], exact=True))
        assert np.array_equal(_bits(res.dense[0].cpu().numpy()), _bits(z[f"out_{m['key']}"])), m
        n += 1
    assert n > 20


def test_multiscale_golden(P, golden_dir):
    z = np.load(golden_dir / "multiscale_small.npz")
    meta = json.loads((golden_dir / "multiscale_small.json").read_text())
    for m in meta:
        (sn, zn), (sm, zm), (sf, zf) = m["kernels"]
        blur = m["blur"]
        got = P.fill_in_multiscale(z[f"in_{m['key']}"], max_depth=m["offset"], near_kernel=(sn, zn),
                                   medium_kernel=(sm, zm), far_kernel=(sf, zf), bin_edges=m["edges"],
                                   extrapolate=True, blur_type=blur.replace("median_", ""),
                                   median_blur=blur.startswith("median"))
        _cmp(got, z[f"out_{m['key']}"], blur)


@pytest.mark.parametrize("case", range(6))
def test_full_size_golden_frames(P, golden_dir, case):
    meta = json.loads((golden_dir / "pipeline_full.json").read_text())[case]
    v = synth.make_frame(synth.CONFIG_SPECS[meta["config"]], [meta["config"], meta["frame"]])
    assert hashlib.sha256(v.tobytes()).hexdigest() == meta["input_sha256"]
    ref, info = O.complete_with_stats(v, _ocfg(meta["cfg"], meta["offset"]))
    assert hashlib.sha256(ref.tobytes()).hexdigest() == meta["output_sha256"]
    res = P.complete_batch(v[None], _pcfg(P, meta["cfg"], meta["offset"]))
    _cmp(res.dense[0].cpu().numpy(), ref, meta["cfg"].get("blur_mode", "median_gaussian"))
    assert int(res.iterations[0]) == info["large_fill_iterations"]


@pytest.mark.parametrize("config_id,blur,fill,n", [(1, "gaussian", "full", 24), (0, "bilateral", "partial", 8),
                                                   (3, "gaussian", "full", 6), (1, "none", "full", 6),
                                                   (1, "median_gaussian", "full", 4),
                                                   (2, "median_bilateral", "full", 4)])
def test_config_batches_vs_oracle(P, config_id, blur, fill, n):
    frames = synth.make_batch(config_id, 100, n)
    kw = {"blur_mode": blur, "fill_mode": fill}
    res = P.complete_batch(torch.from_numpy(frames).cuda(), _pcfg(P, kw))
    got = res.dense.cpu().numpy()
    for i in range(n):
        ref, info = O.complete_with_stats(frames[i], _ocfg(kw))
        _cmp(got[i], ref, blur)
        assert int(res.iterations[i]) == info["large_fill_iterations"]


def test_multi_iteration_frames_inside_batch(P):
    """Frames needing >1 large-fill iteration are finished by the staged path."""
    frames = synth.make_batch(1, 200, 6)
    rng = np.random.default_rng(9)
    for j in (1, 4):
        f = np.zeros_like(frames[j])
        idx = rng.choice(f.size, 4, replace=False)
        f.flat[idx] = rng.uniform(2, 80, 4).astype(np.float32)
        frames[j] = f
    kw = {"blur_mode": "gaussian", "fill_mode": "full"}
    res = P.complete_batch(torch.from_numpy(frames).cuda(), _pcfg(P, kw))
    got = res.dense.cpu().numpy()
    for i in range(6):
        ref, info = O.complete_with_stats(frames[i], _ocfg(kw))
        _cmp(got[i], ref, "gaussian")
        assert int(res.iterations[i]) == info["large_fill_iterations"]
    assert int(res.iterations[1]) > 1


def test_batch_errors_name_the_frame(P):
    frames = synth.make_batch(1, 300, 4)
    frames[2] = 0.0
    with pytest.raises(P.DegenerateInputError, match="frame 2"):
        P.complete_batch(frames, _pcfg(P, {"blur_mode": "gaussian"}))
    frames[2] = synth.make_batch(1, 301, 1)[0]
    frames[3, 0, 0] = 100.0
    with pytest.raises(P.DepthRangeError, match="frame 3"):
        P.complete_batch(frames, _pcfg(P, {"blur_mode": "gaussian"}))
    frames[3, 0, 0] = np.nan
    with pytest.raises(ValueError, match="finite"):
        P.complete_batch(frames, _pcfg(P, {"blur_mode": "gaussian"}))
    res = P.complete_batch(frames, _pcfg(P, {"blur_mode": "gaussian"}), raise_on_error=False)
    st = res.status.cpu().tolist()
    assert st[0] == st[1] == st[2] == 0 and st[3] & 1


def test_determinism_across_batch_sizes(P):
    """SPEC.md:594 analogue: identical bits regardless of batch composition."""
    frames = synth.make_batch(1, 400, 12)
    cfg = _pcfg(P, {"blur_mode": "gaussian", "fill_mode": "full"})
    a = P.complete_batch(frames, cfg).dense.cpu().numpy()
    b = np.concatenate([P.complete_batch(frames[i:i + 5], cfg).dense.cpu().numpy() for i in range(0, 12, 5)])
    c = P.complete_batch(frames, cfg).dense.cpu().numpy()
    assert np.array_equal(_bits(a), _bits(b)) and np.array_equal(_bits(a), _bits(c))


@pytest.mark.parametrize("blur,fill", [("gaussian", "full"), ("bilateral", "partial"), ("median_bilateral", "full")])
def test_many_items_per_cta(P, blur, fill):
    """More frames than SMs: each persistent CTA takes several items in a row, so
    the tensor-memory carry rows, the mbarrier phases and the shared ring carry
    on across items (and the raw mode runs several fused -> blur-tail rounds,
    the median blur tail's persistent CTAs several double-buffered tiles).
    The big batch must equal the same frames run in chunks small enough for one
    item per CTA, bit for bit, and late frames must match the oracle."""
    n = 320
    frames = synth.make_batch(1, 600, n)
    kw = {"blur_mode": blur, "fill_mode": fill}
    cfg = _pcfg(P, kw)
    big = P.complete_batch(frames, cfg)
    got = big.dense.cpu().numpy()
    small = np.concatenate([P.complete_batch(frames[i:i + 80], cfg).dense.cpu().numpy() for i in range(0, n, 80)])
    assert np.array_equal(_bits(got), _bits(small))
    for i in (148, 297, n - 1):
        ref, info = O.complete_with_stats(frames[i], _ocfg(kw))
        _cmp(got[i], ref, blur)
        assert int(big.iterations[i]) == info["large_fill_iterations"]


def test_full_mode_properties(P):
    """density 1.0 and range envelope on generated frames."""
    frames = synth.make_batch(1, 500, 8)
    res = P.complete_batch(frames, _pcfg(P, {"blur_mode": "median_gaussian", "fill_mode": "full"}))
    got = res.dense.cpu().numpy()
    for i in range(8):
        valid = frames[i][frames[i] > np.float32(0.1)]
        assert (got[i] > np.float32(0.1)).all()
        assert got[i].min() >= valid.min() - TOL and got[i].max() <= valid.max() + TOL


def test_single_pixel_and_constant(P):
    one = np.zeros((352, 1216), np.float32)
    one[200, 600] = 50.0
    out = P.fill_in_fast(one, extrapolate=True, blur_type="median_gaussian")
    assert np.all(out == np.float32(50.0))
    const = np.full((40, 60), 30.0, np.float32)
    assert np.all(P.fill_in_fast(const, extrapolate=True, blur_type="median") == np.float32(30.0))


def test_fill_in_fast_api(P):
    v = synth.make_frame(synth.CONFIG_SPECS[0], [0, 0])
    out = P.fill_in_fast(v)  # config 0 defaults: partial + bilateral
    ref = O.complete(v, O.OracleConfig(blur_mode=O.BlurMode.BILATERAL, fill_mode=O.FillMode.PARTIAL))
    _cmp(out, ref, "bilateral")
    t = torch.from_numpy(v).cuda()
    out_t = P.fill_in_fast(t, extrapolate=True, blur_type="gaussian")
    assert isinstance(out_t, torch.Tensor) and out_t.is_cuda
    ref = O.complete(v, O.OracleConfig(blur_mode=O.BlurMode.GAUSSIAN, fill_mode=O.FillMode.FULL))
    _cmp(out_t.cpu().numpy(), ref, "gaussian")
    # custom kernel: named shape given as a boolean array, and an arbitrary footprint
    k = P.make_kernel(P.KernelShape.CROSS, 5)
    out = P.fill_in_fast(v, custom_kernel=k.bits, extrapolate=True, blur_type="none")
    ref = O.complete(v, O.OracleConfig(dilation_shape=O.KernelShape.CROSS, blur_mode=O.BlurMode.NONE))
    _cmp(out, ref, "none")
    odd = np.zeros((5, 5), bool)
    odd[2, :] = True
    odd[0, 0] = odd[4, 4] = True
    out = P.fill_in_fast(v, custom_kernel=odd, extrapolate=True, blur_type="none")
    inv = O.flip(v)
    st2 = O.offsets_max(inv, O.kernel_offsets(odd))
    st3 = O.close(st2, O.make_kernel(O.KernelShape.FULL, 5))
    st4 = O.masked_fill_dilate(st3, O.make_kernel(O.KernelShape.FULL, 7))
    cur = O.extend_to_top(st4)
    while (cur <= np.float32(0.1)).any():
        cur = O.masked_fill_dilate(cur, O.make_kernel(O.KernelShape.FULL, 31))
    _cmp(out, O.flip(cur), "none")


def test_complete_mirror_and_stats(P):
    v = synth.make_frame(synth.CONFIG_SPECS[1], [1, 0])
    dm = P.complete(P.DepthMap(v))
    ref, info = O.complete_with_stats(v)
    _cmp(dm.values, ref, "median_gaussian")
    dense, stats = P.complete_with_stats(P.DepthMap(v))
    _cmp(dense.values, ref, "median_gaussian")
    assert [n for n, _ in stats.stage_ms] == list(P.STAGE_NAMES)
    assert stats.large_fill_iterations == info["large_fill_iterations"]
    assert stats.output_density == pytest.approx(info["output_density"])
    with pytest.raises(P.EncodingError):
        P.complete(P.DepthMap(v, P.DepthEncoding.INVERTED))


def test_host_pipeline_matches_device(P):
    from paper_1802_00036_b200.completion import HostPipeline

    frames = synth.make_batch(1, 600, 20)
    cfg = _pcfg(P, {"blur_mode": "gaussian", "fill_mode": "full"})
    dev = P.complete_batch(frames, cfg).dense.cpu()
    pipe = HostPipeline(cfg, chunk=6)
    h_in = torch.from_numpy(frames).pin_memory()
    out, st, it = pipe.run(h_in)
    assert torch.equal(out, dev)
    assert (st == 0).all()


def test_cuda_backend_plugin(P):
    """The `cuda` backend module satisfies the reference's 7-function surface."""
    import types

    from paper_1802_00036_b200 import cuda_backend

    reg = types.SimpleNamespace(_BACKENDS={})
    cuda_backend.register(reg)
    be = reg._BACKENDS["cuda"]
    assert be.NAME == "cuda"
    rng = np.random.default_rng(1)
    v = rng.uniform(0, 90, (30, 41)).astype(np.float32)
    v[rng.random(v.shape) < 0.5] = 0
    offs = O.kernel_offsets(O.make_kernel(O.KernelShape.DIAMOND, 5))
    assert np.array_equal(be.box_max(v, 2), O.box_max(v, 2))
    assert np.array_equal(be.box_min(v, 3), O.box_min(v, 3))
    assert np.array_equal(be.offsets_max(v, offs), O.offsets_max(v, offs))
    assert np.array_equal(be.offsets_min(v, offs), O.offsets_min(v, offs))
    assert np.array_equal(be.median_filter(v, 5), O.median_filter(v, 5))
    w = O.gaussian_weights(5, 1.1)
    assert np.array_equal(be.gaussian_separable(v, w), O.gaussian_separable(v, w))
    assert np.abs(be.bilateral_filter(v, 5, 1.5, 2.0) - O.bilateral_filter(v, 5, 1.5, 2.0)).max() <= 1e-5


GEOMS = [(352, 1216), (375, 1242), (40, 130), (16, 16), (17, 203), (100, 1250), (64, 2600), (200, 333), (33, 129)]


def _geom_frames(h, w, n, seed):
    spec = synth.SynthSpec(width=w, height=h, beams=max(4, min(64, h // 3)), density=(0.04, 0.12))
    return np.stack([synth.make_frame(spec, [900 + seed, i]) for i in range(n)])


@pytest.mark.parametrize("h,w", GEOMS)
@pytest.mark.parametrize("blur,fill", [("gaussian", "full"), ("none", "full"), ("gaussian", "partial"),
                                       ("none", "partial"), ("median_bilateral", "full"), ("median", "partial"),
                                       ("bilateral", "partial"), ("median_gaussian", "partial")])
def test_fused_geometries_vs_oracle(P, h, w, blur, fill):
    """Frame shapes that exercise strips, W % 4 != 0, lane halos and tiny H."""
    frames = _geom_frames(h, w, 3, h * 7 + w)
    kw = {"blur_mode": blur, "fill_mode": fill}
    res = P.complete_batch(frames, _pcfg(P, kw))
    got = res.dense.cpu().numpy()
    st = res.status.cpu().numpy()
    for i in range(frames.shape[0]):
        ref, info = O.complete_with_stats(frames[i], _ocfg(kw))
        _cmp(got[i], ref, blur)
        assert int(res.iterations[i]) == info["large_fill_iterations"], (i, st[i])


def test_fused_matches_staged_bits_for_selection(P):
    """Selection-only config: fused and staged paths agree bit for bit."""
    frames = synth.make_batch(1, 700, 16)
    kw = {"blur_mode": "none", "fill_mode": "full"}
    a = P.complete_batch(frames, _pcfg(P, kw)).dense.cpu().numpy()
    b = P.complete_batch(frames, _pcfg(P, kw), force_staged=True).dense.cpu().numpy()
    assert np.array_equal(_bits(a), _bits(b))


def test_fused_random_sparse_frames(P):
    """Uniform random sparse points (not scanlines): many empties, columns
    without points, values near max_depth."""
    rng = np.random.default_rng(77)
    frames = np.zeros((6, 120, 300), np.float32)
    for i in range(6):
        m = rng.random(frames[i].shape) < [0.002, 0.01, 0.03, 0.08, 0.2, 0.5][i]
        frames[i][m] = rng.uniform(0.05, 99.99, m.sum()).astype(np.float32)
    frames[2, :, 100:140] = 0  # empty column band
    for blur in ("gaussian", "none", "median_bilateral", "median"):
        kw = {"blur_mode": blur, "fill_mode": "full"}
        res = P.complete_batch(frames, _pcfg(P, kw))
        got = res.dense.cpu().numpy()
        for i in range(6):
            ref, info = O.complete_with_stats(frames[i], _ocfg(kw))
            _cmp(got[i], ref, blur)
            assert int(res.iterations[i]) == info["large_fill_iterations"]


@pytest.mark.parametrize("density", [0.01, 0.002])
def test_low_density_scanline_frames(P, density):
    """BASELINE config-1 frames at 1 % / 0.2 % density (~12 % / ~60 % of the
    pixels still empty after the small fill): the register-dense large fill
    (warp blocks with many empties), the per-pixel passes around it and, at
    0.2 %, the batched multi-iteration fallback, against the oracle."""
    import dataclasses

    spec = dataclasses.replace(synth.CONFIG_SPECS[1], density=(density, density))
    frames = np.stack([synth.make_frame(spec, [1, 9000 + i]) for i in range(2)])
    for blur in ("none", "gaussian"):
        kw = {"blur_mode": blur, "fill_mode": "full"}
        refs = [O.complete_with_stats(frames[i], _ocfg(kw)) for i in range(frames.shape[0])]
        for hint in (True, False):  # DFC_F_SPARSE: the register-dense large fill or the per-pixel passes
            res = P.complete_batch(frames, _pcfg(P, kw), sparse_hint=hint)
            got = res.dense.cpu().numpy()
            for i, (ref, info) in enumerate(refs):
                _cmp(got[i], ref, blur)
                assert int(res.iterations[i]) == info["large_fill_iterations"]


MS_DEFAULT = ((15.0, 30.0), (O.KernelShape.FULL, 7), (O.KernelShape.DIAMOND, 7), (O.KernelShape.DIAMOND, 5))


@pytest.mark.parametrize("h,w", GEOMS)
@pytest.mark.parametrize("blur,fill", [("none", "full"), ("median_bilateral", "full"), ("median", "partial")])
def test_multiscale_geometries_vs_oracle(P, h, w, blur, fill):
    """fill_in_multiscale (default bin kernels: streaming stage-2 kernel) on odd shapes, vs the composed oracle."""
    frames = _geom_frames(h, w, 3, h * 5 + w + 1)
    kw = {"blur_mode": blur, "fill_mode": fill}
    res = P.complete_batch(frames, _pcfg(P, kw), multiscale=P.MultiscaleConfig())
    got = res.dense.cpu().numpy()
    for i in range(frames.shape[0]):
        ref, info = O.complete_with_stats(frames[i], O.OracleConfig(**{**_ocfg(kw).__dict__, "multiscale": MS_DEFAULT}))
        _cmp(got[i], ref, blur)
        assert int(res.iterations[i]) == info["large_fill_iterations"]


@pytest.mark.parametrize("multi", [False, True])
def test_rounds_bit_identical(P, multi, monkeypatch):
    """Raw-mode / multiscale batches run in rounds whose intermediate maps live in the workspace; the round
    length (an 8 GiB budget by default) must not change a bit: 3 and 2 rounds against one."""
    frames = synth.make_batch(2, 700, 20)
    cfg = _pcfg(P, {"blur_mode": "median_bilateral", "fill_mode": "full"})
    ms = P.MultiscaleConfig() if multi else None
    outs = []
    for chunk in ("8", "12", None):
        if chunk:
            monkeypatch.setenv("DFC_RAW_CHUNK", chunk)
        else:
            monkeypatch.delenv("DFC_RAW_CHUNK")
        res = P.complete_batch(frames, cfg, multiscale=ms)
        outs.append((res.dense.cpu().numpy(), res.valid_counts.cpu().numpy(), res.iterations.cpu().numpy()))
        assert not (res.status.cpu().numpy() & 0xFF).any()
    for d, n, it in outs[:-1]:
        assert d.tobytes() == outs[-1][0].tobytes()
        assert np.array_equal(n, outs[-1][1]) and np.array_equal(it, outs[-1][2])


@pytest.mark.parametrize("h,w", [(352, 1216), (100, 250), (67, 130), (1024, 512)])
def test_multiscale_row_segments_bit_identical(P, h, w, monkeypatch):
    """The stage-2 streaming kernel cuts column slices into row segments (one warm-up block each) when whole
    columns do not fill the SMs evenly; every segment count gives the whole-column result bit for bit, the
    same valid-input counts, and matches the composed oracle."""
    frames = synth.make_batch(2, 900, 2) if (h, w) == (352, 1216) else _geom_frames(h, w, 2, h + w)
    kw = {"blur_mode": "none", "fill_mode": "full"}
    outs = {}
    for nseg in ("1", "2", "3", "4", "16"):
        monkeypatch.setenv("DFC_MS_NSEG", nseg)
        res = P.complete_batch(frames, _pcfg(P, kw), multiscale=P.MultiscaleConfig())
        outs[nseg] = (res.dense.cpu().numpy(), res.valid_counts.cpu().numpy()[:, 0])
    monkeypatch.delenv("DFC_MS_NSEG")
    res = P.complete_batch(frames, _pcfg(P, kw), multiscale=P.MultiscaleConfig())
    outs["auto"] = (res.dense.cpu().numpy(), res.valid_counts.cpu().numpy()[:, 0])
    for k, (d, n) in outs.items():
        assert d.tobytes() == outs["1"][0].tobytes(), k
        assert np.array_equal(n, outs["1"][1]), k
    for i in range(frames.shape[0]):
        ref = O.complete(frames[i], O.OracleConfig(**{**_ocfg(kw).__dict__, "multiscale": MS_DEFAULT}))
        _cmp(outs["auto"][0][i], ref, "none")
        assert int(outs["auto"][1][i]) == int(np.count_nonzero(frames[i] > 0.1))


@pytest.mark.parametrize("kernels", [((O.KernelShape.CROSS, 5), (O.KernelShape.CIRCLE, 7), (O.KernelShape.FULL, 3)),
                                     ((O.KernelShape.DIAMOND, 3), (O.KernelShape.FULL, 5), (O.KernelShape.CIRCLE, 5))])
def test_multiscale_other_kernels_vs_oracle(P, kernels):
    """Non-default bin kernels take the generic offsets stage-2 kernel."""
    frames = synth.make_batch(2, 300, 3)
    kw = {"blur_mode": "none", "fill_mode": "full"}
    ms = P.MultiscaleConfig(near=(P.KernelShape(kernels[0][0].value), kernels[0][1]),
                            medium=(P.KernelShape(kernels[1][0].value), kernels[1][1]),
                            far=(P.KernelShape(kernels[2][0].value), kernels[2][1]))
    res = P.complete_batch(frames, _pcfg(P, kw), multiscale=ms)
    got = res.dense.cpu().numpy()
    for i in range(frames.shape[0]):
        ref = O.complete(frames[i], O.OracleConfig(**{**_ocfg(kw).__dict__, "multiscale": ((15.0, 30.0), *kernels)}))
        _cmp(got[i], ref, "none")


@pytest.mark.parametrize("blur", ["none", "gaussian", "median_bilateral"])
def test_wide_sparse_frames_dense_large_fill(P, blur):
    """~1% density on multi-strip frames: many empty pixels per warp block take
    the dense large-fill path (shared vertical maxima) instead of per-pixel passes."""
    spec = synth.SynthSpec(width=2600, height=256, beams=48, density=(0.008, 0.012))
    frames = np.stack([synth.make_frame(spec, [950, i]) for i in range(2)])
    kw = {"blur_mode": blur, "fill_mode": "full"}
    res = P.complete_batch(frames, _pcfg(P, kw))
    got = res.dense.cpu().numpy()
    for i in range(frames.shape[0]):
        ref, info = O.complete_with_stats(frames[i], _ocfg(kw))
        _cmp(got[i], ref, blur)
        assert int(res.iterations[i]) == info["large_fill_iterations"]


def _rand_case(rng):
    h, w = int(rng.integers(16, 160)), int(rng.integers(16, 700))
    spec = synth.SynthSpec(width=w, height=h, beams=int(rng.integers(4, max(5, min(64, h // 2)))),
                           density=(float(rng.uniform(0.005, 0.05)),) * 2,
                           max_depth=float(rng.choice([100.0, 120.0, 60.0])))
    blur = str(rng.choice(["none", "gaussian", "median", "bilateral", "median_gaussian", "median_bilateral"]))
    fill = str(rng.choice(["full", "partial"]))
    shape = str(rng.choice(["diamond", "full", "cross", "circle"]))
    size = int(rng.choice([3, 5, 7]))
    multi = bool(rng.random() < 0.3)
    return spec, blur, fill, shape, size, multi


@pytest.mark.parametrize("case", range(100))
def test_randomized_configs_vs_oracle(P, case):
    """Seeded random shapes, densities, max_depth, blur / fill modes, stage-2 kernels
    and multiscale bins: every device path (fused, raw + blur tail, PRE, staged) vs the oracle."""
    rng = np.random.default_rng(10_000 + case)
    spec, blur, fill, shape, size, multi = _rand_case(rng)
    frames = np.stack([synth.make_frame(spec, [1234, case, i]) for i in range(2)])
    kw = {"blur_mode": blur, "fill_mode": fill}
    md = spec.max_depth
    if multi:
        ms = P.MultiscaleConfig(near=(P.KernelShape(shape), size))
        res = P.complete_batch(frames, _pcfg(P, kw, offset=md), multiscale=ms, raise_on_error=False)
        ocfg = O.OracleConfig(**{**_ocfg(kw, md).__dict__, "multiscale": (
            (15.0, 30.0), (O.KernelShape(shape), size), (O.KernelShape.DIAMOND, 7), (O.KernelShape.DIAMOND, 5))})
    else:
        kw2 = {**kw, "dilation_shape": shape, "dilation_size": size}
        res = P.complete_batch(frames, _pcfg(P, kw2, offset=md), raise_on_error=False)
        ocfg = _ocfg(kw2, md)
    got = res.dense.cpu().numpy()
    st = res.status.cpu().numpy()
    for i in range(frames.shape[0]):
        try:
            ref, info = O.complete_with_stats(frames[i], ocfg)
        except Exception as e:  # the reference raises: the device must flag the frame
            assert st[i] & 0xFF, (type(e).__name__, st[i])
            continue
        assert not st[i] & 0xFF, st[i]
        _cmp(got[i], ref, blur)
        assert int(res.iterations[i]) == info["large_fill_iterations"]


def _counts_ref(frames, ocfg):
    out = []
    for f in frames:
        _, info = O.complete_with_stats(f, ocfg)
        n = f.size
        out.append((round(info["input_density"] * n), round(info["output_density"] * n)))
    return np.array(out)


@pytest.mark.parametrize("blur,fill,multi,staged", [("gaussian", "full", False, False),
                                                    ("bilateral", "partial", False, False),
                                                    ("median_bilateral", "full", True, False),
                                                    ("none", "full", False, False),
                                                    ("gaussian", "partial", False, True)])
def test_density_counters_vs_oracle(P, blur, fill, multi, staged):
    """(f)3: per-frame valid-pixel counts from the fused read / store passes
    (dfc_fill_counts) equal RunStats' input / output densities times H*W
    (pipeline.py:138-141, 192-202) exactly -- including frames with inputs
    within 0.1 of max_depth (valid, but invalid once inverted) and a frame
    finished by the staged fallback."""
    frames = synth.make_batch(1, 800, 6)
    frames[2][frames[2] > 0] = np.float32(99.95)  # every valid input inverts to an empty pixel
    frames[3].flat[::97] = np.float32(99.95)
    f4 = np.zeros_like(frames[4])
    f4[100, 50] = 20.0
    f4[300, 1100] = 40.0
    frames[4] = f4  # needs many large-fill iterations (staged fallback in FULL mode)
    kw = {"blur_mode": blur, "fill_mode": fill}
    ocfg = _ocfg(kw)
    if multi:
        ocfg = O.OracleConfig(**{**ocfg.__dict__, "multiscale": MS_DEFAULT})
    res = P.complete_batch(frames, _pcfg(P, kw), multiscale=P.MultiscaleConfig() if multi else None,
                           force_staged=staged, raise_on_error=False)
    got = res.valid_counts.cpu().numpy()
    ok = [i for i in range(6) if not res.status.cpu().numpy()[i] & 0xFF]
    want = _counts_ref(frames[ok], ocfg)
    assert np.array_equal(got[ok], want), (got[ok], want)
    din, dout = res.densities()
    assert np.allclose(din[ok] * frames[0].size, want[:, 0])


@pytest.mark.parametrize("blur", ["none", "bilateral", "median"])
@pytest.mark.parametrize("gsize", [7, 63])
def test_fused_path_other_blur_any_gaussian_size(P, blur, gsize):
    """gaussian_size only matters to the Gaussian: the fused path with another blur
    and a non-default gaussian_size runs and matches the oracle."""
    frames = synth.make_batch(1, 850, 2)
    kw = {"blur_mode": blur, "fill_mode": "full", "gaussian_size": gsize}
    res = P.complete_batch(frames, _pcfg(P, kw))
    got = res.dense.cpu().numpy()
    for i in range(2):
        ref = O.complete(frames[i], _ocfg(kw))
        _cmp(got[i], ref, blur)


def test_sparse_batch_fallback_batched(P):
    """A batch of very sparse frames (uniform ~0.05 % points: many large-fill
    iterations each) goes through the batched, device-gated fallback: every
    frame matches the oracle with its own iteration count."""
    rng = np.random.default_rng(123)
    n = 40
    frames = np.zeros((n, 352, 1216), np.float32)
    for i in range(n):
        m = rng.random(frames[i].shape) < rng.uniform(0.0002, 0.001)
        frames[i][m] = rng.uniform(1, 90, m.sum()).astype(np.float32)
    kw = {"blur_mode": "gaussian", "fill_mode": "full"}
    res = P.complete_batch(frames, _pcfg(P, kw))
    got = res.dense.cpu().numpy()
    st = res.status.cpu().numpy()
    its = res.iterations.cpu().numpy()
    assert (st & 0x100).sum() > n // 2, "expected most frames on the fallback"
    for i in range(0, n, 5):
        ref, info = O.complete_with_stats(frames[i], _ocfg(kw))
        _cmp(got[i], ref, "gaussian")
        assert int(its[i]) == info["large_fill_iterations"]
    assert len(set(its.tolist())) > 1
