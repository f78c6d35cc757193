#!/usr/bin/env python
"""Opcode histogram (executed warp instructions) and stall samples per opcode
from an ncu source-page export:
    ncu -i REP --page source --csv --print-source sass -k regex:NAME > src.csv
    python tools/sass_profile.py src.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
ex = collections.Counter()
samp = collections.Counter()
stall = collections.defaultdict(collections.Counter)
tot_ex = 0
tot_s = 0
for r in rows[2:]:
    if len(r) < len(h) or not r[ix["Instructions Executed"]].isdigit():
        continue
    src = r[1].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex[op] += n
    samp[op] += s
    tot_ex += n
    tot_s += s
    for k in h:
        if k.startswith("stall_") and "Not Issued" not in k:
            v = int(r[ix[k]] or 0)
            if v:
                stall[op][k[6:]] += v
print(f"total executed warp instructions {tot_ex}, stall samples {tot_s}")
print(f"{'opcode':12s} {'executed':>12s} {'%':>6s} {'samples%':>9s}  top stalls")
for op, n in ex.most_common(40):
    top = ", ".join(f"{k} {v / max(1, samp[op]):.0%}" for k, v in stall[op].most_common(3))
    print(f"{op:12s} {n:12d} {n / tot_ex:6.1%} {samp[op] / max(1, tot_s):9.1%}  {top}")
