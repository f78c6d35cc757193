"""Row (e): frame-sharded multi-GPU completion through libdfc.

The test box has one GPU, so N independent workers share cuda:0: they never
wait on each other (no collective on the data path), and the results must be
byte-identical to one worker (reference SPEC.md:594: identical outputs for
any worker count)."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_00036_b200 as pkg

    return pkg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_multi_device_pipeline_matches_single(P):
    from paper_1802_00036_b200 import synth
    from paper_1802_00036_b200.multi import MultiDevicePipeline

    frames = synth.make_batch(1, 1000, 13)
    cfg = P.PipelineConfig(blur_mode=P.BlurMode.GAUSSIAN, fill_mode=P.FillMode.FULL)
    ref = P.complete_batch(frames, cfg).dense.cpu()
    for devs in ([0], [0, 0], [0, 0, 0]):
        pipe = MultiDevicePipeline(cfg, devices=devs, chunk=4)
        out, st, it = pipe.run(torch.from_numpy(frames).pin_memory())
        assert torch.equal(out, ref), devs
        assert (st == 0).all()


def _run_ranks(n, out, total):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           "-m", "paper_1802_00036_b200.multi", "--dfc-config", "1", "--dfc-first", "40", "--dfc-total", str(total),
           "--dfc-out", str(out), "--dfc-device", "0", "--dfc-backend", "gloo"]
    env = {**os.environ, "PYTHONPATH": str(ROOT)}
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    parts = sorted((np.load(out / f"rank{k}.npz") for k in range(n)), key=lambda z: int(z["start"]))
    assert int(parts[0]["start"]) == 0 and int(parts[-1]["stop"]) == total
    assert all(int(parts[k]["stop"]) == int(parts[k + 1]["start"]) for k in range(n - 1))
    assert all(int(p["launches"]) > 0 for p in parts)  # every rank ran libdfc kernels
    return (np.concatenate([p["dense"] for p in parts]), np.concatenate([p["status"] for p in parts]),
            np.concatenate([p["iterations"] for p in parts]))


def test_torchrun_two_ranks_byte_identical_to_one(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    total = 9
    d1, s1, i1 = _run_ranks(1, tmp_path / "one", total)
    d2, s2, i2 = _run_ranks(2, tmp_path / "two", total)
    assert d1.tobytes() == d2.tobytes()
    assert np.array_equal(s1, s2) and np.array_equal(i1, i2)
    assert not (s1 & 0xFF).any()
