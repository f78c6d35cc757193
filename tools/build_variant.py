"""Build an experimental libdfc variant with extra -D flags on the fused kernel.

    python tools/build_variant.py NAME -DFLAG[=V] ...   ->  paper_1802_00036_b200/libdfc_NAME.so

Only fused.cu / fused_vec4.cu (or $VARIANT_SRCS) are recompiled; select the variant at run time
with DFC_LIB=paper_1802_00036_b200/libdfc_NAME.so (bench.py, tests).
"""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(name, flags):
    from paper_1802_00036_b200 import build as B

    B.build()
    objdir = ROOT / "paper_1802_00036_b200" / "build_obj"
    vdir = objdir / f"var_{name}"
    vdir.mkdir(exist_ok=True)
    import os
    srcs = os.environ.get("VARIANT_SRCS", "fused.cu fused_vec4.cu").split()

    def cc(s):
        cmd = [B.nvcc(), *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-c", *flags,
               "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{B.CSRC}", "-Xptxas", "-v",
               str(B.CSRC / s), "-o", str(vdir / (Path(s).stem + ".o"))]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(r.stderr)
            raise SystemExit(1)
        return r.stderr

    with ThreadPoolExecutor(2) as ex:
        logs = list(ex.map(cc, srcs))
    (vdir / "ptxas.log").write_text("".join(logs))
    objs = [str(vdir / (Path(s).stem + ".o")) for s in srcs]
    objs += [str(o) for o in sorted(objdir.glob("*.o")) if o.name not in {Path(x).stem + ".o" for x in srcs}]
    out = ROOT / "paper_1802_00036_b200" / f"libdfc_{name}.so"
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", *objs, "-o", str(out)], check=True)
    print(out)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
