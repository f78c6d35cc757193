"""The drop-in boundary through the reference's own operator registry
(backend.py:21-54; SURVEY.md 8(b) boundary 1).

* CPU (runs where /root/reference is present): ``cuda_backend.register`` puts
  this package's backend into the UNMODIFIED reference's ``_BACKENDS``,
  ``set_backend('cuda')`` selects it, and its seven functions take the same
  positional parameters as the reference's own backends.
* GPU: every operator call the reference pipeline made through its registry
  for three configs (recorded by tests/golden/make_registry_trace.py with a
  recording backend around the reference's numpy backend) is replayed through
  ``cuda_backend`` -- selection ops and the fp64 Gaussian bit-exact, the
  bilateral within 1e-4 m -- and ``complete`` on the same frames matches the
  reference's ``complete`` output.
"""

import inspect
import json
import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
GOLD = Path(__file__).resolve().parent / "golden"
OPS = ("box_max", "box_min", "offsets_max", "offsets_min", "median_filter", "gaussian_separable", "bilateral_filter")


@pytest.mark.skipif(not (REF / "depthfill" / "backend.py").exists(), reason="reference not present (GPU box)")
def test_cuda_backend_registers_in_reference_registry(monkeypatch):
    monkeypatch.setenv("DEPTHFILL_BACKEND", "python")
    monkeypatch.syspath_prepend(str(REF))
    for m in [k for k in sys.modules if k == "depthfill" or k.startswith("depthfill.")]:
        monkeypatch.delitem(sys.modules, m)
    from depthfill import _numpy_ops, backend

    from paper_1802_00036_b200 import cuda_backend

    cuda_backend.register(backend)
    try:
        assert "cuda" in backend.available_backends()
        backend.set_backend("cuda")
        assert backend.active_backend() is cuda_backend
        assert backend.active_backend_name() == "cuda"
        for op in OPS:
            ours = list(inspect.signature(getattr(cuda_backend, op)).parameters)
            ref = list(inspect.signature(getattr(_numpy_ops, op)).parameters)
            assert ours == ref, (op, ours, ref)
    finally:
        backend.set_backend("python")
        backend._BACKENDS.pop("cuda", None)


def _args(z, call):
    return [z[a["array"]] if "array" in a else a["value"] for a in call["args"]]


@pytest.mark.gpu
def test_registry_trace_replay_through_cuda_backend():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1802_00036_b200 import cuda_backend

    z = np.load(GOLD / "registry_trace.npz")
    meta = json.loads((GOLD / "registry_trace.json").read_text())
    n = 0
    for run in meta:
        for j, call in enumerate(run["calls"]):
            vin = z[f"in_{run['key']}_{j}"]
            ref = z[f"out_{run['key']}_{j}"]
            got = getattr(cuda_backend, call["op"])(vin, *_args(z, call))
            assert got.dtype == np.float32 and got.shape == ref.shape
            if call["op"] == "bilateral_filter":
                assert float(np.abs(got - ref).max()) <= 1e-4, (run["key"], j)
            else:
                assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (run["key"], j, call["op"])
            n += 1
    assert n == sum(len(r["calls"]) for r in meta) > 0


@pytest.mark.gpu
def test_complete_matches_reference_complete_on_trace_frames():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_00036_b200 as P

    z = np.load(GOLD / "registry_trace.npz")
    meta = json.loads((GOLD / "registry_trace.json").read_text())
    cfgs = {
        "default": P.PipelineConfig(),
        "partial_bilateral": P.PipelineConfig(blur_mode=P.BlurMode.BILATERAL, fill_mode=P.FillMode.PARTIAL),
        "cross_median_bilateral": P.PipelineConfig(dilation_shape=P.KernelShape.CROSS,
                                                   blur_mode=P.BlurMode.MEDIAN_BILATERAL),
    }
    for run in meta:
        fr = z[f"frame_{run['key']}"]
        ref = z[f"complete_{run['key']}"]
        got = np.asarray(P.complete(P.DepthMap(fr), cfgs[run["config"]]).values)
        assert float(np.abs(got - ref).max()) <= 1e-4, run["key"]
        assert np.array_equal(got > np.float32(0.1), ref > np.float32(0.1)), run["key"]
