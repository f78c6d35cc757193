"""Generate the golden vectors that pin the oracle to the reference.

Runs the UNMODIFIED reference package ``depthfill`` from
``/root/reference/pkg/src`` (numpy backend, exactly as shipped: nothing is
built there, so ``backend.auto`` resolves to ``_numpy_ops``) on seeded inputs
and stores its outputs:

* ``ops_small.npz``      -- the 7-function operator surface on random grids,
* ``stages_small.npz``   -- invert / masked fill / extend_to_top,
* ``pipeline_small.npz`` -- complete_with_stats on small synthetic frames over
                            the config matrix, plus edge cases,
* ``pipeline_full.json`` -- full-size BASELINE config frames: sha256 of the
                            reference output bytes (inputs are regenerated
                            from their seeds and also hashed),
* ``multiscale_small.npz`` -- the composed multiscale oracle built from the
                            reference's own morphology.dilate per depth bin,
* ``multiscale_full.json`` -- full-size BASELINE config 2 / 4 frames through the
                            composed multiscale oracle: sha256 of the output,
* ``metrics_small.npz`` / ``metrics_small.json`` -- metrics.evaluate, error_map
                            and MetricsAccumulator on seeded prediction / ground
                            truth pairs,
* ``kitti_small.npz``    -- kitti_io.write_depth_png -> read_depth_png on
                            seeded maps through real 16-bit PNG files (written
                            to a scratch directory inside the repo, removed).

Nothing here is copied from a dataset; every input is generated from a seed.
Usage:  python tests/golden/make_golden.py [name ...]   (needs /root/reference;
        names: ops stages pipeline multiscale full metrics kitti multiscale_full; default all)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

os.environ["DEPTHFILL_BACKEND"] = "python"
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, REF)
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from depthfill import backend, depth_core, kernels, morphology, pipeline  # noqa: E402
from paper_1802_00036_b200 import synth  # noqa: E402

assert backend.active_backend_name() == "python"
OPS = backend.active_backend()


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rand_map(rng, h, w, p_empty=0.5, tiny=0.05):
    v = rng.uniform(0.0, 99.0, size=(h, w)).astype(np.float32)
    u = rng.random((h, w))
    v[u < p_empty] = 0.0
    v[(u >= p_empty) & (u < p_empty + tiny)] = rng.uniform(0.0, 0.1)
    return v


SIZES = [(1, 1), (1, 7), (7, 1), (2, 3), (5, 5), (13, 29), (33, 17), (64, 64), (48, 61)]


def gen_ops():
    rng = np.random.default_rng(1234)
    out = {}
    n = 0
    for (h, w) in SIZES:
        for rep in range(2):
            v = rand_map(rng, h, w)
            key = f"{n:03d}"
            out[f"in_{key}"] = v
            for r in (1, 2, 3, 15):
                out[f"box_max_r{r}_{key}"] = OPS.box_max(v, r)
                out[f"box_min_r{r}_{key}"] = OPS.box_min(v, r)
            for shape in kernels.KernelShape:
                for size in (3, 5, 7):
                    offs = kernels.kernel_offsets(kernels.make_kernel(shape, size))
                    out[f"offs_max_{shape.value}{size}_{key}"] = OPS.offsets_max(v, offs)
                    out[f"offs_min_{shape.value}{size}_{key}"] = OPS.offsets_min(v, offs)
            for size in (3, 5, 7):
                out[f"median{size}_{key}"] = OPS.median_filter(v, size)
            for (size, sigma) in ((5, 1.1), (3, 0.8), (7, 2.0)):
                wts = morphology.gaussian_weights(size, sigma)
                out[f"gauss{size}_{sigma}_{key}"] = OPS.gaussian_separable(v, wts)
            for (size, sv, ss) in ((5, 1.5, 2.0), (3, 0.5, 1.0), (7, 3.0, 1.5)):
                out[f"bilat{size}_{sv}_{ss}_{key}"] = OPS.bilateral_filter(v, size, sv, ss)
            n += 1
    np.savez_compressed(HERE / "ops_small.npz", **out)


def gen_stages():
    rng = np.random.default_rng(99)
    out = {}
    for n, (h, w) in enumerate(SIZES):
        v = rand_map(rng, h, w)
        v = np.minimum(v, np.float32(99.95))
        key = f"{n:03d}"
        out[f"in_{key}"] = v
        dm = depth_core.DepthMap(v)
        inv = depth_core.invert(dm)
        out[f"invert_{key}"] = inv.values
        out[f"invert_back_{key}"] = depth_core.invert_back(inv).values
        out[f"extend_{key}"] = morphology.extend_to_top(inv).values
        for size in (3, 7, 31):
            k = kernels.make_kernel(kernels.KernelShape.FULL, size)
            if size <= 2 * min(h, w) + 1:
                out[f"mfill{size}_{key}"] = morphology.masked_fill_dilate(inv, k).values
    np.savez_compressed(HERE / "stages_small.npz", **out)


SMALL_SPEC = synth.SynthSpec(width=128, height=48, beams=16, density=(0.06, 0.12))


def run_ref(v, cfg, offset=100.0):
    old = depth_core.INVERSION_OFFSET
    depth_core.INVERSION_OFFSET = offset
    try:
        dense, st = pipeline.complete_with_stats(depth_core.DepthMap(v), cfg)
    finally:
        depth_core.INVERSION_OFFSET = old
    return dense.values, st


def gen_pipeline_small():
    out = {}
    meta = []
    n = 0

    def add(v, cfgkw, offset=100.0, tag=""):
        nonlocal n
        cfg = pipeline.PipelineConfig(**{k: (pipeline.BlurMode(x) if k == "blur_mode" else
                                             pipeline.FillMode(x) if k == "fill_mode" else
                                             kernels.KernelShape(x) if k == "dilation_shape" else x)
                                         for k, x in cfgkw.items()})
        key = f"{n:03d}"
        try:
            dense, st = run_ref(v, cfg, offset)
            out[f"out_{key}"] = dense
            res = {"iters": st.large_fill_iterations, "in_density": st.input_density,
                   "out_density": st.output_density, "error": None}
        except ValueError as e:
            res = {"error": type(e).__name__}
        out[f"in_{key}"] = v
        meta.append({"key": key, "cfg": cfgkw, "offset": offset, "tag": tag, **res})
        n += 1

    for i in range(6):
        v = synth.make_frame(SMALL_SPEC, [100, i])
        for blur in [b.value for b in pipeline.BlurMode]:
            for fill in ("full", "partial"):
                add(v, {"blur_mode": blur, "fill_mode": fill}, tag="matrix")
    for i, shape in enumerate(kernels.KernelShape):
        for size in (3, 5, 7):
            v = synth.make_frame(SMALL_SPEC, [101, 10 * i + size])
            add(v, {"dilation_shape": shape.value, "dilation_size": size,
                    "blur_mode": "gaussian", "fill_mode": "full"}, tag="shapes")
    # non-default sizes
    v = synth.make_frame(SMALL_SPEC, [102, 0])
    add(v, {"closure_size": 3, "small_fill_size": 5, "large_fill_size": 9, "median_size": 3,
            "gaussian_size": 7, "gaussian_sigma": 2.0, "blur_mode": "median_gaussian"}, tag="sizes")
    add(v, {"bilateral_size": 3, "bilateral_sigma_value": 0.7, "bilateral_sigma_space": 1.3,
            "median_size": 7, "blur_mode": "median_bilateral"}, tag="sizes")
    add(v, {"large_fill_max_iters": 1, "large_fill_size": 5, "blur_mode": "gaussian"}, tag="sizes")

    # edge cases
    one = np.zeros((48, 128), np.float32)
    one[30, 77] = 50.0
    add(one, {}, tag="single_pixel")  # every output pixel 50.0
    add(np.full((20, 30), 30.0, np.float32), {}, tag="constant")
    add(np.full((1, 1), 7.5, np.float32), {}, tag="1x1")
    add(np.array([[0.0, 12.0, 0.0], [0.0, 0.0, 40.0]], np.float32), {}, tag="2x3")
    add(np.zeros((10, 10), np.float32), {}, tag="degenerate")
    add(np.array([[0.05, 0.1, 0.0], [0.0, 0.0, 0.1]], np.float32), {}, tag="degenerate_sub")
    bad = np.full((8, 8), 5.0, np.float32)
    bad[3, 3] = 100.0
    add(bad, {}, tag="range")
    rng = np.random.default_rng(5)
    sparse = np.zeros((200, 300), np.float32)
    idx = rng.choice(sparse.size, 3, replace=False)
    sparse.flat[idx] = rng.uniform(1, 80, 3).astype(np.float32)
    add(sparse, {"blur_mode": "gaussian"}, tag="multi_iter")
    add(sparse, {"blur_mode": "gaussian", "large_fill_max_iters": 2}, tag="iter_cap")
    v = synth.make_frame(SMALL_SPEC, [103, 0])
    v[:, 40:52] = 0.0  # empty column band
    v[5, 100] = 99.95  # inverts to a tiny (empty) value
    v[6, 101] = 0.07   # sub-threshold input
    add(v, {"blur_mode": "median_gaussian"}, tag="edge_values")
    add(v, {"blur_mode": "bilateral", "fill_mode": "partial"}, tag="edge_values")
    v120 = synth.make_frame(synth.SynthSpec(width=128, height=48, beams=16, density=(0.1, 0.1),
                                            max_depth=120.0, far_m=115.0), [104, 0])
    add(v120, {"blur_mode": "median_bilateral"}, offset=120.0, tag="max_depth_120")
    tiny = np.zeros((3, 40), np.float32)
    tiny[1, ::7] = 20.0
    add(tiny, {}, tag="tiny_frame")  # _fit_to_frame clamps kernels
    np.savez_compressed(HERE / "pipeline_small.npz", **out)
    (HERE / "pipeline_small.json").write_text(json.dumps(meta, indent=1))


FULL_CASES = [
    # (config, frame index, cfg kwargs, offset)
    (0, 0, {"blur_mode": "bilateral", "fill_mode": "partial"}, 100.0),
    (1, 0, {"blur_mode": "gaussian", "fill_mode": "full"}, 100.0),
    (1, 1, {"blur_mode": "gaussian", "fill_mode": "full"}, 100.0),
    (1, 2, {}, 100.0),  # reference default median_gaussian
    (2, 0, {"blur_mode": "median_bilateral", "fill_mode": "full"}, 100.0),
    (3, 0, {"blur_mode": "gaussian", "fill_mode": "full"}, 100.0),
]


def gen_pipeline_full():
    meta = []
    for (c, i, kw, off) in FULL_CASES:
        v = synth.make_frame(synth.CONFIG_SPECS[c], [c, i])
        cfg = pipeline.PipelineConfig(**{k: (pipeline.BlurMode(x) if k == "blur_mode" else
                                             pipeline.FillMode(x)) for k, x in kw.items()})
        dense, st = run_ref(v, cfg, off)
        meta.append({"config": c, "frame": i, "cfg": kw, "offset": off,
                     "input_sha256": sha(v), "output_sha256": sha(dense),
                     "iters": st.large_fill_iterations,
                     "out_density": st.output_density,
                     "samples": [[int(y), int(x), float(dense[y, x])]
                                 for y, x in ((0, 0), (v.shape[0] // 2, v.shape[1] // 2),
                                              (v.shape[0] - 1, v.shape[1] - 1), (150, 600))]})
    (HERE / "pipeline_full.json").write_text(json.dumps(meta, indent=1))


MS_EDGES = (15.0, 30.0)
MS_KERNELS = [(("full", 7), ("diamond", 7), ("diamond", 5)),
              (("diamond", 5), ("diamond", 5), ("diamond", 5)),
              (("cross", 5), ("circle", 7), ("full", 3))]


def ref_multiscale(v, kern, blur, offset=100.0):
    """Composed oracle from reference primitives only."""
    old = depth_core.INVERSION_OFFSET
    depth_core.INVERSION_OFFSET = offset
    try:
        dm = depth_core.DepthMap(v)
        inv = depth_core.invert(dm)
        d = dm.values
        near = d <= np.float32(MS_EDGES[0])
        med = (d > np.float32(MS_EDGES[0])) & (d <= np.float32(MS_EDGES[1]))
        far = d > np.float32(MS_EDGES[1])
        merged = None
        for sel, (shape, size) in zip((near, med, far), kern):
            part = depth_core.DepthMap._wrap(np.where(sel, inv.values, np.float32(0.0)),
                                             depth_core.DepthEncoding.INVERTED)
            r = morphology.dilate(part, kernels.make_kernel(kernels.KernelShape(shape), size)).values
            merged = r if merged is None else np.maximum(merged, r)
        cur = depth_core.DepthMap._wrap(merged, depth_core.DepthEncoding.INVERTED)
        cfg = pipeline.PipelineConfig(blur_mode=pipeline.BlurMode(blur))
        cur = morphology.close(cur, kernels.make_kernel(kernels.KernelShape.FULL, cfg.closure_size))
        cur = morphology.masked_fill_dilate(cur, kernels.make_kernel(kernels.KernelShape.FULL,
                                                                     cfg.small_fill_size))
        cur = morphology.extend_to_top(cur)
        big = kernels.make_kernel(kernels.KernelShape.FULL, cfg.large_fill_size)
        it = 0
        while it < cfg.large_fill_max_iters and (cur.values <= depth_core.VALIDITY_THRESHOLD).any():
            cur = morphology.masked_fill_dilate(cur, big)
            it += 1
        cur = pipeline._blur_stage(cur, cfg)
        return depth_core.invert_back(cur).values, it
    finally:
        depth_core.INVERSION_OFFSET = old


def gen_multiscale():
    out = {}
    meta = []
    spec = synth.SynthSpec(width=128, height=48, beams=16, density=(0.08, 0.12))
    n = 0
    for ki, kern in enumerate(MS_KERNELS):
        for blur in ("median_bilateral", "gaussian"):
            v = synth.make_frame(spec, [105, n])
            dense, it = ref_multiscale(v, kern, blur)
            key = f"{n:03d}"
            out[f"in_{key}"] = v
            out[f"out_{key}"] = dense
            meta.append({"key": key, "kernels": kern, "edges": MS_EDGES, "blur": blur, "iters": it,
                         "offset": 100.0})
            n += 1
    spec120 = synth.SynthSpec(width=128, height=48, beams=16, density=(0.05, 0.05), max_depth=120.0,
                              far_m=115.0, box_depth=(0.5, 60.0))
    v = synth.make_frame(spec120, [105, 99])
    dense, it = ref_multiscale(v, MS_KERNELS[0], "median_bilateral", 120.0)
    out["in_100"] = v
    out["out_100"] = dense
    meta.append({"key": "100", "kernels": MS_KERNELS[0], "edges": MS_EDGES, "blur": "median_bilateral",
                 "iters": it, "offset": 120.0})
    np.savez_compressed(HERE / "multiscale_small.npz", **out)
    (HERE / "multiscale_small.json").write_text(json.dumps(meta, indent=1))


def gen_metrics():
    from depthfill import metrics

    rng = np.random.default_rng(2024)
    out, meta = {}, []
    acc = metrics.MetricsAccumulator()
    for k, (h, w) in enumerate([(1, 1), (3, 5), (17, 31), (64, 80), (120, 300)]):
        gt = rand_map(rng, h, w, p_empty=0.6)
        pred = gt + rng.normal(0, 0.5, size=gt.shape).astype(np.float32)
        pred = np.where(rng.random(gt.shape) < 0.2, np.float32(0.0), np.abs(pred)).astype(np.float32)
        pred[0, 0] = gt[0, 0] = np.float32(5.0)  # at least one shared valid pixel
        p = depth_core.DepthMap(pred)
        g = depth_core.DepthMap(gt)
        rep = metrics.evaluate(p, g)
        acc.add(p, g)
        out[f"pred_{k}"] = pred
        out[f"gt_{k}"] = gt
        out[f"emap_{k}"] = metrics.error_map(p, g)
        meta.append({"key": k, "sums": list(metrics._error_sums(p, g)), "report": [
            rep.rmse_mm, rep.mae_mm, rep.irmse_invkm, rep.imae_invkm, rep.evaluated_pixels, rep.skipped_pixels]})
    r = acc.finalize()
    meta.append({"accumulated": [r.rmse_mm, r.mae_mm, r.irmse_invkm, r.imae_invkm, r.evaluated_pixels,
                                 r.skipped_pixels]})
    np.savez_compressed(HERE / "metrics_small.npz", **out)
    (HERE / "metrics_small.json").write_text(json.dumps(meta, indent=1))


def gen_kitti():
    import shutil

    from depthfill import kitti_io

    rng = np.random.default_rng(99)
    tmp = ROOT / "gpurun_out" / "_golden_png"
    tmp.mkdir(parents=True, exist_ok=True)
    out = {}
    try:
        for k, (h, w) in enumerate([(1, 1), (7, 9), (40, 64)]):
            v = rng.uniform(0.0, 255.99, size=(h, w)).astype(np.float32)
            v[rng.random((h, w)) < 0.3] = 0.0
            v.flat[0] = np.float32(1.5 / 256.0)  # an exact tie (raw 1.5 -> 2)
            path = tmp / f"k{k}.png"
            kitti_io.write_depth_png(depth_core.DepthMap(v), path)
            back = kitti_io.read_depth_png(path).values
            out[f"in_{k}"] = v
            out[f"back_{k}"] = np.array(back)
        raw = np.arange(65536, dtype=np.uint16).reshape(256, 256)
        path = tmp / "all.png"
        from PIL import Image

        Image.fromarray(raw).save(path)
        out["all_raw_decoded"] = np.array(kitti_io.read_depth_png(path).values)
        # colormap rendering (kitti_io.write_colormap_png): pixels read back from the PNG
        ranges = [(0.0, 80.0), (2.5, 7.25), (-1.0, 0.5)]
        for k, (lo, hi) in enumerate(ranges):
            v = rng.uniform(lo - 5.0, hi + 5.0, size=(33, 47)).astype(np.float32)
            v[rng.random(v.shape) < 0.2] = 0.0
            v.flat[1:6] = np.float32(lo + (hi - lo) * np.array([0.0, 0.25, 0.5, 0.75, 1.0]))  # ramp stops
            path = tmp / f"c{k}.png"
            kitti_io.write_colormap_png(v, path, lo, hi)
            with Image.open(path) as img:
                out[f"cmap_rgb_{k}"] = np.array(img.convert("RGB"))
            out[f"cmap_in_{k}"] = v
            out[f"cmap_range_{k}"] = np.array([lo, hi])
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    np.savez_compressed(HERE / "kitti_small.npz", **out)


# full-size BASELINE fill_in_multiscale frames (config 2: 1216x352, config 4:
# 4096x1024 with max_depth 120), pinned by SHA-256 of the composed reference output
MS_FULL_CASES = [(2, 0, 100.0), (2, 1, 100.0), (4, 0, 120.0)]


def gen_multiscale_full():
    meta = []
    for (c, i, off) in MS_FULL_CASES:
        v = synth.make_frame(synth.CONFIG_SPECS[c], [c, i])
        dense, it = ref_multiscale(v, MS_KERNELS[0], "median_bilateral", off)
        meta.append({"config": c, "frame": i, "kernels": MS_KERNELS[0], "edges": MS_EDGES,
                     "blur": "median_bilateral", "offset": off, "input_sha256": sha(v),
                     "output_sha256": sha(dense), "iters": it,
                     "samples": [[int(y), int(x), float(dense[y, x])]
                                 for y, x in ((0, 0), (v.shape[0] // 2, v.shape[1] // 2),
                                              (v.shape[0] - 1, v.shape[1] - 1), (150, 600))]})
    (HERE / "multiscale_full.json").write_text(json.dumps(meta, indent=1))


GENS = {"ops": gen_ops, "stages": gen_stages, "pipeline": gen_pipeline_small, "multiscale": gen_multiscale,
        "full": gen_pipeline_full, "metrics": gen_metrics, "kitti": gen_kitti,
        "multiscale_full": gen_multiscale_full}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(GENS):
        GENS[name]()
    print("golden vectors written to", HERE)
