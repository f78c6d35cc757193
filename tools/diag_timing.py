"""Per-warp cycle breakdown of the fused kernel (diagnostics build).

    python tools/diag_timing.py build      # here: libdfc_timing.so with -DDFC_TIMING
    python tools/diag_timing.py run        # on a GPU box: config-1 frames, prints the table

The timing build accumulates clock64 deltas per (CTA, warp): producer,
barrier wait, consumer, phase 1.  It perturbs register allocation, so use it
for the shape of the imbalance, not for absolute speed.
"""
import ctypes
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
LIB = ROOT / "paper_1802_00036_b200" / "libdfc_timing.so"


def build():
    from paper_1802_00036_b200 import build as B

    B.build()
    objdir = ROOT / "paper_1802_00036_b200" / "build_obj"
    tim = objdir / "timing"
    tim.mkdir(exist_ok=True)
    srcs = ["fused.cu", "fused_vec4.cu"]
    for s in srcs:
        cmd = [B.nvcc(), *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-c", "-DDFC_TIMING",
               "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{B.CSRC}", str(B.CSRC / s), "-o",
               str(tim / (Path(s).stem + ".o"))]
        subprocess.run(cmd, check=True)
    objs = [str(tim / (Path(s).stem + ".o")) for s in srcs]
    objs += [str(o) for o in sorted(objdir.glob("*.o")) if o.name not in ("fused.o", "fused_vec4.o")]
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", *objs, "-o", str(LIB)], check=True)
    print(LIB)


def run(frames=1024):
    import numpy as np
    import torch

    from paper_1802_00036_b200 import _lib, synth
    from paper_1802_00036_b200.completion import BlurMode, FillMode, PipelineConfig, to_dfc_config

    L = ctypes.CDLL(str(LIB))
    _lib._declare(L) if hasattr(_lib, "_declare") else None
    x = torch.from_numpy(synth.make_batch(1, 0, frames)).cuda()
    out = torch.empty_like(x)
    B, H, W = x.shape
    st = torch.empty(B, dtype=torch.int32, device="cuda")
    it = torch.empty(B, dtype=torch.int32, device="cuda")
    cfg = to_dfc_config(PipelineConfig(blur_mode=BlurMode.GAUSSIAN, fill_mode=FillMode.FULL))
    cfg.flags |= _lib.F_NO_FINISH
    L.dfc_workspace_bytes.restype = ctypes.c_size_t
    need = L.dfc_workspace_bytes(ctypes.byref(cfg), ctypes.c_int64(B), H, W)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    tim = torch.zeros(148 * 12 * 6, dtype=torch.int64, device="cuda")
    os.environ["DFC_TIM_PTR"] = hex(tim.data_ptr())
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    for _ in range(2):
        tim.zero_()
        rc = L.dfc_fill_batch(P(x), P(out), ctypes.c_int64(B), H, W, ctypes.byref(cfg), P(st), P(it), P(ws),
                              ctypes.c_size_t(need), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0, rc
        torch.cuda.synchronize()
    t = tim.view(148, 12, 6).cpu().numpy().astype(np.float64)
    names = ["producer", "(ring wait)", "consumer", "item-end wait", "(cons:ring+LF)", "fast blocks"]
    tot = t[:, :, [0, 2, 3]].sum(axis=2)
    t[:, :, 5] *= 1e6 / frames  # fast-block count per frame (scaled to print as-is)
    print("per-warp mean cycles (over CTAs), share of warp time:")
    print("warp " + " ".join(f"{n:>10s}" for n in names) + "      total")
    for w in range(12):
        m = t[:, w, :].mean(axis=0)
        print(f"{w:4d} " + " ".join(f"{v / 1e6:9.2f}M" for v in m) + f" {tot[:, w].mean() / 1e6:9.2f}M")
    allm = t.sum(axis=(0, 1))
    print("all  " + " ".join(f"{v / allm[[0, 2, 3]].sum() * 100:9.1f}%" for v in allm))
    print("(parenthesised columns are parts of the producer / consumer columns)")


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
