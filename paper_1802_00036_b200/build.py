"""Build libdfc.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libdfc.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    deps = list(CSRC.glob("*")) + [ROOT / "include" / "dfc.h", Path(__file__)]
    return all(p.stat().st_mtime <= t for p in deps)


def _compile(src: Path, obj: Path) -> subprocess.CompletedProcess:
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-c",
           "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{CSRC}", "-Xptxas", "-v", str(src), "-o", str(obj)]
    return subprocess.run(cmd, capture_output=True, text=True)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every csrc/*.cu in parallel (the fused kernel's instantiations are
    split over fused_vec{1,2,4}.cu for this), then link libdfc.so."""
    if not force and up_to_date():
        return OUT
    from concurrent.futures import ThreadPoolExecutor

    objdir = PKG / "build_obj"
    objdir.mkdir(exist_ok=True)
    srcs = sources()
    objs = [objdir / (s.stem + ".o") for s in srcs]
    # longest first: the fused instantiations dominate
    order = sorted(range(len(srcs)), key=lambda i: -srcs[i].stat().st_size)
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        results = dict(zip(order, ex.map(lambda i: _compile(srcs[i], objs[i]), order)))
    log = []
    for i in range(len(srcs)):
        res = results[i]
        log.append(res.stderr)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {srcs[i].name}")
    link = subprocess.run([nvcc(), *ARCH, "-shared", *[str(o) for o in objs], "-o", str(OUT) + ".tmp"],
                          capture_output=True, text=True)
    if link.returncode != 0:
        sys.stderr.write(link.stdout + link.stderr)
        raise RuntimeError("nvcc failed linking libdfc.so")
    (PKG / "build_ptxas.log").write_text("".join(log))
    os.replace(str(OUT) + ".tmp", OUT)
    if verbose:
        print("".join(log))
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
