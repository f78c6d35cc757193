"""End-to-end GPU parity at the BASELINE.json configs' own shapes (SURVEY.md §4
tier 3): fill_in_multiscale on config 2 (1216x352 batch) and config 4
(4096x1024, 128 beams, 2 %, max_depth 120: the fused PRE + DENSE kernel with
4 column strips), against the composed multiscale oracle, which
tests/test_oracle_golden.py::test_multiscale_full_golden pins by SHA-256 to the
reference's own primitives (reference semantics: pipeline.py:124-203,
morphology.py:39-51).

Bar: <= 1e-4 m (bilateral blur, north_star), exact validity, exact large-fill
iteration counts, and the frames must stay on the fused path (no staged
fallback, status bit DFC_ST_FALLBACK clear).
"""

import hashlib
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import depthfill_oracle as O  # noqa: E402
from paper_1802_00036_b200 import synth  # noqa: E402

TOL = 1e-4


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_00036_b200 as pkg

    return pkg


def _ocfg(md):
    return O.OracleConfig(blur_mode=O.BlurMode.MEDIAN_BILATERAL, fill_mode=O.FillMode.FULL, max_depth=md,
                          multiscale=O.DEFAULT_MULTISCALE)


def _pcfg(P, md):
    return P.PipelineConfig(blur_mode=P.BlurMode.MEDIAN_BILATERAL, fill_mode=P.FillMode.FULL, max_depth=md)


def _check(got, ref):
    got = np.asarray(got, np.float32)
    err = float(np.abs(got - ref).max())
    assert err <= TOL, f"max |err| {err}"
    assert np.array_equal(got > np.float32(0.1), ref > np.float32(0.1))


def test_config4_multiscale_vs_oracle(P):
    """Config 4: two 4096x1024 frames, max_depth 120, median + bilateral, 31x31 fill."""
    frames = synth.make_batch(4, 0, 2)
    res = P.complete_batch(torch.from_numpy(frames).cuda(), _pcfg(P, 120.0), multiscale=P.MultiscaleConfig())
    st = res.status.cpu().numpy()
    assert not (st & 0x100).any(), f"frames went to the staged fallback: {st}"
    got = res.dense.cpu().numpy()
    meta = json.loads((__import__("pathlib").Path(__file__).parent / "golden" / "multiscale_full.json").read_text())
    pinned = {(m["config"], m["frame"]): m for m in meta}
    for i in range(2):
        ref, info = O.complete_with_stats(frames[i], _ocfg(120.0))
        if (4, i) in pinned:  # the oracle output is the reference's, bit for bit
            assert hashlib.sha256(ref.tobytes()).hexdigest() == pinned[(4, i)]["output_sha256"]
        _check(got[i], ref)
        assert int(res.iterations[i]) == info["large_fill_iterations"]


def test_config4_public_api(P):
    """fill_in_multiscale(max_depth=120, blur_type='bilateral', median_blur=True) on a
    device tensor returns a device tensor equal to complete_batch's output."""
    frames = synth.make_batch(4, 1, 1)
    t = torch.from_numpy(frames).cuda()
    out = P.fill_in_multiscale(t, max_depth=120.0, extrapolate=True, blur_type="bilateral", median_blur=True)
    assert isinstance(out, torch.Tensor) and out.is_cuda and tuple(out.shape) == frames.shape
    ref = O.complete(frames[0], _ocfg(120.0))
    _check(out[0].cpu().numpy(), ref)


def test_config2_multiscale_batch_vs_oracle(P):
    """Config 2: a batch of 1216x352 frames (density U(4 %, 6 %)) through the
    public fill_in_multiscale on a device tensor, vs the composed oracle."""
    n = 8
    frames = synth.make_batch(2, 0, n)
    out = P.fill_in_multiscale(torch.from_numpy(frames).cuda(), max_depth=100.0, extrapolate=True,
                               blur_type="bilateral", median_blur=True)
    got = out.cpu().numpy()
    meta = json.loads((__import__("pathlib").Path(__file__).parent / "golden" / "multiscale_full.json").read_text())
    pinned = {(m["config"], m["frame"]): m for m in meta}
    for i in range(n):
        ref, info = O.complete_with_stats(frames[i], _ocfg(100.0))
        if (2, i) in pinned:
            assert hashlib.sha256(ref.tobytes()).hexdigest() == pinned[(2, i)]["output_sha256"]
        _check(got[i], ref)
    res = P.complete_batch(torch.from_numpy(frames).cuda(), _pcfg(P, 100.0), multiscale=P.MultiscaleConfig())
    assert not (res.status.cpu().numpy() & 0x100).any()
    assert np.array_equal(res.dense.cpu().numpy().view(np.uint32), got.view(np.uint32))


def test_config3_shape_batch_vs_oracle(P):
    """Config 3 shape (1242x375, W % 4 == 2: the VEC-2 fused instantiation)."""
    frames = synth.make_batch(3, 0, 4)
    cfg = P.PipelineConfig(blur_mode=P.BlurMode.GAUSSIAN, fill_mode=P.FillMode.FULL)
    res = P.complete_batch(torch.from_numpy(frames).cuda(), cfg)
    got = res.dense.cpu().numpy()
    for i in range(4):
        ref, info = O.complete_with_stats(frames[i], O.OracleConfig(blur_mode=O.BlurMode.GAUSSIAN,
                                                                    fill_mode=O.FillMode.FULL))
        _check(got[i], ref)
        assert int(res.iterations[i]) == info["large_fill_iterations"]
