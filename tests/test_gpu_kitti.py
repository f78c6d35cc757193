"""KITTI 16-bit raw at the boundary: value conversion of
kitti_io.read_depth_png (depth = raw / 256, kitti_io.py:53) and
write_depth_png (raw = rint(f64(depth) * 256) clipped, < 256 m, kitti_io.py:60-65)
fused into the pipeline's read / write passes, against the oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import depthfill_oracle as O  # noqa: E402
from paper_1802_00036_b200 import synth  # noqa: E402

TOL = 1e-4


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_00036_b200.kitti as kitti

    return kitti


def ref_decode(raw):  # kitti_io.py:53
    return raw.astype(np.float32) / np.float32(256.0)


def ref_encode(v):  # kitti_io.py:64-65
    return np.clip(np.rint(v.astype(np.float64) * 256.0), 0, 65535).astype(np.uint16)


def test_decode_encode_all_raw_values(K):
    raw = np.arange(65536, dtype=np.uint16).reshape(256, 256)
    d = K.decode(raw).cpu().numpy()
    assert np.array_equal(d.view(np.uint32), ref_decode(raw).view(np.uint32))
    assert np.array_equal(K.encode(d).cpu().numpy(), raw)


def test_encode_rounding_and_range(K):
    rng = np.random.default_rng(3)
    v = np.concatenate([rng.uniform(0, 255.99, 5000), np.arange(0, 512) / 512.0 + 0.5 / 256.0,  # ties (x.5 raw)
                        [0.0, 1e-9, 255.998, 255.9999]]).astype(np.float32)
    assert np.array_equal(K.encode(v[None]).cpu().numpy()[0], ref_encode(v))
    with pytest.raises(ValueError, match="encodable"):
        K.encode(np.array([[1.0, 256.0]], np.float32))


def _raw_frames(cid, n, seed, spec=None):
    spec = spec or synth.CONFIG_SPECS[cid]
    return np.stack([ref_encode(synth.make_frame(spec, [seed, i])) for i in range(n)])


def _ocfg(kw, offset=100.0):
    conv = {"blur_mode": O.BlurMode, "fill_mode": O.FillMode}
    return O.OracleConfig(**{k: conv[k](x) if k in conv else x for k, x in kw.items()}, max_depth=offset)


def _pcfg(P, kw):
    conv = {"blur_mode": P.BlurMode, "fill_mode": P.FillMode}
    return P.PipelineConfig(**{k: conv[k](x) if k in conv else x for k, x in kw.items()})


@pytest.mark.parametrize("shape", [(352, 1216), (375, 1242), (64, 300), (96, 2600)])
@pytest.mark.parametrize("blur,fill", [("none", "full"), ("gaussian", "full"), ("median_bilateral", "full"),
                                       ("bilateral", "partial"), ("none", "partial")])
def test_raw16_pipeline_vs_oracle(K, shape, blur, fill):
    import paper_1802_00036_b200 as P

    h, w = shape
    spec = synth.SynthSpec(width=w, height=h, beams=max(8, min(64, h // 4)), density=(0.04, 0.07))
    raw = _raw_frames(None, 2, 777 + h, spec)
    kw = {"blur_mode": blur, "fill_mode": fill}
    res_raw = K.complete_raw16_batch(raw, _pcfg(P, kw), out_raw=True)
    res_f = K.complete_raw16_batch(raw, _pcfg(P, kw), out_raw=False)
    got_raw = res_raw.dense.cpu().numpy()
    got_f = res_f.dense.cpu().numpy()
    for i in range(raw.shape[0]):
        ref, info = O.complete_with_stats(ref_decode(raw[i]), _ocfg(kw))
        if blur == "none":
            assert np.array_equal(got_f[i].view(np.uint32), ref.view(np.uint32))
            assert np.array_equal(got_raw[i], ref_encode(ref))
        else:
            assert float(np.abs(got_f[i] - ref).max()) <= TOL
            # a float within 1e-4 m of the reference encodes to within one raw unit
            assert int(np.abs(got_raw[i].astype(np.int32) - ref_encode(ref).astype(np.int32)).max()) <= 1
            assert np.array_equal(got_raw[i], ref_encode(got_f[i]))  # fused encode == encode of the float path
        assert int(res_raw.iterations[i]) == info["large_fill_iterations"]


def test_raw16_multiscale_and_staged(K):
    import paper_1802_00036_b200 as P

    raw = _raw_frames(2, 2, 31)
    kw = {"blur_mode": "none", "fill_mode": "full"}
    ms = ((15.0, 30.0), (O.KernelShape.FULL, 7), (O.KernelShape.DIAMOND, 7), (O.KernelShape.DIAMOND, 5))
    a = K.complete_raw16_batch(raw, _pcfg(P, kw), multiscale=P.MultiscaleConfig()).dense.cpu().numpy()
    b = K.complete_raw16_batch(raw, _pcfg(P, kw), force_staged=True).dense.cpu().numpy()
    for i in range(2):
        ref_ms = O.complete(ref_decode(raw[i]), O.OracleConfig(**{**_ocfg(kw).__dict__, "multiscale": ms}))
        assert np.array_equal(a[i], ref_encode(ref_ms))
        assert np.array_equal(b[i], ref_encode(O.complete(ref_decode(raw[i]), _ocfg(kw))))


def test_raw16_errors(K):
    import paper_1802_00036_b200 as P

    raw = _raw_frames(1, 2, 5)
    raw[1, 200, 300] = 25600  # 100.0 m == max_depth
    with pytest.raises(P.DepthRangeError, match="frame 1"):
        K.complete_raw16_batch(raw, P.PipelineConfig())
    empty = np.full((1, 64, 128), 25, np.uint16)  # 25 / 256 <= 0.1 m: every pixel empty
    with pytest.raises(P.DegenerateInputError):
        K.complete_raw16_batch(empty, P.PipelineConfig())


def test_colormap_vs_oracle(K, golden_dir):
    """GPU colormap pixels bit-identical to the oracle (pinned to write_colormap_png) and to the golden PNGs."""
    from oracle import metrics_oracle as M

    z = np.load(golden_dir / "kitti_small.npz")
    for k in range(3):
        lo, hi = (float(x) for x in z[f"cmap_range_{k}"])
        assert np.array_equal(K.colormap(z[f"cmap_in_{k}"], lo, hi).cpu().numpy(), z[f"cmap_rgb_{k}"])
    rng = np.random.default_rng(8)
    v = rng.uniform(-10, 120, size=(2, 200, 300)).astype(np.float32)
    v[rng.random(v.shape) < 0.3] = 0.0
    assert np.array_equal(K.colormap(v, 0.0, 100.0).cpu().numpy(), M.colormap(v, 0.0, 100.0))
    with pytest.raises(ValueError, match="degenerate range"):
        K.colormap(v, 5.0, 5.0)


def test_raw_pipeline_matches_batch_api(K):
    """Pinned-host raw16 pipeline (3 streams, chunks) == complete_raw16_batch, incl. a frame that
    needs more than one large-fill iteration (re-run through the staged path)."""
    import paper_1802_00036_b200 as P

    raw = _raw_frames(1, 10, 61)
    rng = np.random.default_rng(4)
    f = np.zeros_like(raw[3])
    f.flat[rng.choice(f.size, 4, replace=False)] = rng.integers(600, 20000, 4).astype(np.uint16)
    raw[3] = f  # 4 isolated points: several large-fill iterations
    cfg = P.PipelineConfig(blur_mode=P.BlurMode.GAUSSIAN, fill_mode=P.FillMode.FULL)
    want = K.complete_raw16_batch(raw, cfg)
    pipe = K.RawPipeline(cfg, chunk=4)
    out, st, it = pipe.run(torch.from_numpy(raw).pin_memory())
    assert np.array_equal(out.numpy(), want.dense.cpu().numpy())
    assert np.array_equal(it.numpy(), want.iterations.cpu().numpy())
    assert int(it[3]) > 1 and int(st[3]) & 0x100  # finished by the staged path
