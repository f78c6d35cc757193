"""GPU error metrics against the oracle restatement of
depthfill.metrics, which tests/test_oracle_golden.py pins to the reference."""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import metrics_oracle as M  # noqa: E402
from paper_1802_00036_b200 import synth  # noqa: E402


@pytest.fixture(scope="module")
def Mx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1802_00036_b200 import metrics

    return metrics


def _close(a, b):  # float64 sums in a different (fixed) order than numpy's
    return abs(a - b) <= 1e-9 * max(abs(a), abs(b), 1e-300)


def test_metrics_golden_pairs(Mx, golden_dir):
    z = np.load(golden_dir / "metrics_small.npz")
    meta = json.loads((golden_dir / "metrics_small.json").read_text())
    acc = Mx.MetricsAccumulator()
    for m in meta[:-1]:
        k = m["key"]
        p, g = z[f"pred_{k}"], z[f"gt_{k}"]
        sums, counts = Mx.error_sums(p, g)
        ref = M.error_sums(p, g)
        assert all(_close(float(sums[0, i]), ref[i]) for i in range(4))
        assert (int(counts[0, 0]), int(counts[0, 1])) == (ref[4], ref[5])
        r = Mx.evaluate(p, g)
        assert all(_close(a, b) for a, b in zip((r.rmse_mm, r.mae_mm, r.irmse_invkm, r.imae_invkm), m["report"][:4]))
        assert (r.evaluated_pixels, r.skipped_pixels) == tuple(m["report"][4:])
        assert np.array_equal(Mx.error_map(p, g).cpu().numpy()[0], z[f"emap_{k}"])
        acc.add(p, g)
    r = acc.finalize()
    want = meta[-1]["accumulated"]
    assert all(_close(a, b) for a, b in zip((r.rmse_mm, r.mae_mm, r.irmse_invkm, r.imae_invkm), want[:4]))
    assert (r.evaluated_pixels, r.skipped_pixels) == tuple(want[4:])


def test_metrics_batch_full_size(Mx):
    """Completed frames vs a denser synthetic 'ground truth' of the same scenes, batched."""
    import paper_1802_00036_b200 as P

    sparse = synth.make_batch(1, 40, 4)
    gt = synth.make_batch(1, 40, 4) + np.float32(0.01)
    pred = P.complete_batch(sparse, P.PipelineConfig()).dense
    reps = Mx.evaluate_batch(pred, gt)
    pn = pred.cpu().numpy()
    for b in range(4):
        ref = M.finalize(*M.error_sums(pn[b], gt[b]))
        r = reps[b]
        assert all(_close(a, c) for a, c in zip((r.rmse_mm, r.mae_mm, r.irmse_invkm, r.imae_invkm), ref[:4]))
        assert (r.evaluated_pixels, r.skipped_pixels) == ref[4:]


def test_metrics_errors(Mx):
    with pytest.raises(ValueError, match="dimension mismatch"):
        Mx.evaluate(np.ones((4, 5), np.float32), np.ones((5, 4), np.float32))
    with pytest.raises(ValueError, match="share no valid pixels"):
        Mx.evaluate(np.zeros((4, 5), np.float32), np.ones((4, 5), np.float32))
    with pytest.raises(ValueError, match="no overlapping"):
        Mx.MetricsAccumulator().finalize()


def test_metrics_non_float32_tensors(Mx):
    """float64 / float16 CUDA tensors are converted, not reinterpreted as float32 bits."""
    rng = np.random.default_rng(5)
    p = rng.uniform(1, 80, (30, 40)).astype(np.float32)
    g = rng.uniform(1, 80, (30, 40)).astype(np.float32)
    g[rng.random(g.shape) < 0.3] = 0
    want = Mx.error_sums(p, g)
    got = Mx.error_sums(torch.from_numpy(p.astype(np.float64)).cuda(), torch.from_numpy(g.astype(np.float64)).cuda())
    assert np.array_equal(want[0], got[0]) and np.array_equal(want[1], got[1])
    from paper_1802_00036_b200 import kitti

    a = kitti.colormap(torch.from_numpy(p).cuda(), 0.0, 80.0).cpu()
    b = kitti.colormap(torch.from_numpy(p.astype(np.float64)).cuda(), 0.0, 80.0).cpu()
    assert torch.equal(a, b)
