#!/usr/bin/env python
"""Per-CUDA-line executed warp instructions and stall samples from
    ncu -i REP --page source --csv --print-source cuda,sass -k regex:NAME > mix.csv
    python tools/line_profile.py mix.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = "?"
hdr = None
agg = collections.defaultdict(lambda: [0, 0, collections.Counter(), ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r) if k}
        # the second "Source" column (SASS) shadows the first; metrics come after it
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        n = int(r[hdr["Instructions Executed"]] or 0)
        s = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    a = agg[(fname, int(r[0]))]
    a[0] += n
    a[1] += s
    a[3] = r[1][:70]
    for k, i in hdr.items():
        if k.startswith("stall_") and "Not Issued" not in k and r[i].isdigit() and int(r[i]):
            a[2][k[6:]] += int(r[i])
tn = sum(a[0] for a in agg.values())
ts = sum(a[1] for a in agg.values())
print(f"total instr {tn}, samples {ts}")
for key, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:N]:
    top = ", ".join(f"{k} {v / max(1, a[1]):.0%}" for k, v in a[2].most_common(2))
    print(f"{key[0][:14]:14s}:{key[1]:<5d} instr {a[0] / tn:6.2%} samp {a[1] / ts:6.2%}  [{top}]  {a[3]}")
