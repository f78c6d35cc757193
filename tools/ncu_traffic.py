#!/usr/bin/env python
"""Aggregate ncu launch lists (gpu__time_duration / dram__bytes_read / _write
per launch, `--csv --log-file`) into per-config DRAM bytes per frame and write
them into profiles/traffic.json under the config id.

    python tools/ncu_traffic.py CONFIG FRAMES_PROCESSED launches.csv [--label fused] [--write]

FRAMES_PROCESSED = frames every dfc_fill_batch call of the profiled run
covered together ((warmup + steps) x frames per step with --no-e2e).  Only
libdfc kernels count (torch's own kernels are the harness's).
"""

from __future__ import annotations

import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OURS = ("fused_kernel", "r0_kernel", "finalize_kernel", "ms_fast_kernel", "ms_tile", "blur_tail", "lf_",
        "large_fill", "count_kernel", "fill_counts")


def load(path):
    rows = [ln for ln in Path(path).read_text().splitlines() if ln.startswith('"')]
    per = defaultdict(dict)
    names = {}
    for r in csv.DictReader(rows):
        i = int(r["ID"])
        names[i] = r["Kernel Name"]
        per[i][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return names, per


def short(name):
    n = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    return n.split("(")[0].replace("void ", "")


def summarise(path, frames):
    names, per = load(path)
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])  # launches, ns, read, write
    for i, n in names.items():
        s = short(n)
        if not any(k in s for k in OURS):
            continue
        m = per[i]
        a = agg[s]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
    tot_r = sum(a[2] for a in agg.values())
    tot_w = sum(a[3] for a in agg.values())
    tot_t = sum(a[1] for a in agg.values())
    return agg, tot_r / frames, tot_w / frames, tot_t


def main():
    cfg, frames, path = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    label = sys.argv[sys.argv.index("--label") + 1] if "--label" in sys.argv else "fused"
    agg, rpf, wpf, tot_t = summarise(path, frames)
    print(f"{'kernel':60s} {'n':>5s} {'ms total':>10s} {'share':>7s} {'MB read/fr':>11s} {'MB write/fr':>12s}")
    for s, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{s[:60]:60s} {a[0]:5d} {a[1] / 1e6:10.3f} {a[1] / tot_t:7.1%} {a[2] / frames / 1e6:11.3f} "
              f"{a[3] / frames / 1e6:12.3f}")
    print(f"DRAM bytes per frame: {rpf + wpf:.0f} (read {rpf:.0f}, write {wpf:.0f})")
    if "--write" in sys.argv:
        tf = ROOT / "profiles" / "traffic.json"
        d = json.loads(tf.read_text()) if tf.exists() else {}
        d.setdefault(str(cfg), {})[label] = {
            "dram_bytes_per_frame": round(rpf + wpf),
            "read_bytes_per_frame": round(rpf),
            "write_bytes_per_frame": round(wpf),
            "source": f"ncu launch list {Path(path).name}: dram__bytes_read/write.sum of every libdfc kernel "
                      f"over {frames} frames (cold-cache, serialised launches)",
        }
        tf.write_text(json.dumps(d, indent=1) + "\n")


if __name__ == "__main__":
    main()
