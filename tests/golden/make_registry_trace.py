"""Record the operator calls the UNMODIFIED reference pipeline makes through its
backend registry, for the drop-in replay test (tests/test_gpu_registry.py).

A recording backend module is inserted into ``depthfill.backend._BACKENDS``
(the same mechanism ``cuda_backend.register`` uses, backend.py:21-54) and
selected with ``set_backend``; it forwards every call to the reference's own
numpy backend (``_numpy_ops``) and stores the op name, its arguments, the
input map and the returned map.  ``pipeline.complete`` is then run on seeded
synthetic frames for three configs (the reference defaults: median + Gaussian,
FULL; bilateral, PARTIAL; custom cross kernel + median + bilateral).  The GPU
test replays each recorded call through ``cuda_backend`` and compares outputs;
the final ``complete`` outputs are stored too.

Usage: python tests/golden/make_registry_trace.py   (needs /root/reference)
Writes tests/golden/registry_trace.npz (+ .json).  Inputs come from seeds.
"""

from __future__ import annotations

import json
import os
import sys
import types
from pathlib import Path

os.environ["DEPTHFILL_BACKEND"] = "python"
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

from depthfill import backend, pipeline  # noqa: E402
from depthfill import _numpy_ops  # noqa: E402
from depthfill.depth_core import DepthMap  # noqa: E402

from paper_1802_00036_b200 import synth  # noqa: E402

OPS = ("box_max", "box_min", "offsets_max", "offsets_min", "median_filter", "gaussian_separable", "bilateral_filter")


def main():
    calls = []
    rec = types.ModuleType("trace_backend")
    rec.NAME = "trace"

    def wrap(name):
        fn = getattr(_numpy_ops, name)

        def f(values, *args):
            out = fn(values, *args)
            calls.append((name, np.array(values, copy=True), [np.array(a) if isinstance(a, np.ndarray) else a
                                                             for a in args], np.array(out, copy=True)))
            return out
        return f

    for n in OPS:
        setattr(rec, n, wrap(n))
    backend._BACKENDS["trace"] = rec
    backend.set_backend("trace")
    assert backend.active_backend_name() == "trace"

    spec = synth.SynthSpec(width=96, height=64, beams=16, density=(0.06, 0.06))
    frames = [synth.make_frame(spec, [31, i]) for i in range(2)]
    configs = {
        "default": {},
        "partial_bilateral": {"blur_mode": pipeline.BlurMode.BILATERAL, "fill_mode": pipeline.FillMode.PARTIAL},
        "cross_median_bilateral": {"dilation_shape": pipeline.KernelShape.CROSS,
                                   "blur_mode": pipeline.BlurMode.MEDIAN_BILATERAL},
    }
    arrays, meta = {}, []
    for ck, kw in configs.items():
        for i, fr in enumerate(frames):
            calls.clear()
            cfg = pipeline.PipelineConfig(**kw)
            out = pipeline.complete(DepthMap(fr), cfg).values
            key = f"{ck}_{i}"
            arrays[f"frame_{key}"] = fr
            arrays[f"complete_{key}"] = np.asarray(out)
            entry = {"key": key, "config": ck, "calls": []}
            for j, (name, vin, args, vout) in enumerate(calls):
                arrays[f"in_{key}_{j}"] = vin
                arrays[f"out_{key}_{j}"] = vout
                a_meta = []
                for k, a in enumerate(args):
                    if isinstance(a, np.ndarray):
                        arrays[f"arg_{key}_{j}_{k}"] = a
                        a_meta.append({"array": f"arg_{key}_{j}_{k}"})
                    else:
                        a_meta.append({"value": a})
                entry["calls"].append({"op": name, "args": a_meta})
            meta.append(entry)
    backend.set_backend("python")
    np.savez_compressed(HERE / "registry_trace.npz", **arrays)
    (HERE / "registry_trace.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(f"{sum(len(m['calls']) for m in meta)} calls over {len(meta)} runs")


if __name__ == "__main__":
    main()
