"""Static SASS opcode histogram of libdfc kernels (cuobjdump), e.g.

    python tools/sass_hist.py paper_1802_00036_b200/build_obj/fused_vec4.o 'fused_kernelILi4ELb1ELi4ELb0ELb0ELi0E'

Prints the count of each opcode in the kernel's SASS (static instruction
sites, not executed counts) plus the tcgen05 / TMA / async-copy markers the
profiling guide names (STTM/LDTM, UTMALDG/UBLKCP, LDGSTS, SYNCS)."""

import collections
import re
import subprocess
import sys


def sass(obj: str, pattern: str) -> dict[str, list[str]]:
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for ln in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            cur = m.group(1) if re.search(pattern, m.group(1)) else None
            if cur:
                funcs[cur] = []
            continue
        if cur:
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
            if m:
                funcs[cur].append(m.group(2))
    return funcs


def main():
    obj, pattern = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "."
    for name, ops in sass(obj, pattern).items():
        base = collections.Counter(o.split(".")[0] for o in ops)
        print(f"== {name}: {len(ops)} instructions")
        for op, n in base.most_common():
            print(f"  {op:12s} {n}")


if __name__ == "__main__":
    main()
