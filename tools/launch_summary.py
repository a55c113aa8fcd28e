"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum
--clock-control none --csv --log-file FILE python bench.py ...`) by kernel
family: launches, total device ms and share.  Generated candidate kernels
(`k<i>_<stage>`) are one family; the best candidate's kernel is reported by
grid/block when given.

  python tools/launch_summary.py gpurun_out/launches_v3.csv [--grid G --block B]
"""

from __future__ import annotations

import argparse
import csv
import io
import re
from collections import defaultdict


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--grid", default="")
    ap.add_argument("--block", default="")
    a = ap.parse_args()
    text = open(a.csv, encoding="utf-8", errors="replace").read()
    start = text.find('"ID"')
    rows = csv.DictReader(io.StringIO(text[start:]))
    fam = defaultdict(lambda: [0, 0.0])
    best = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ms = ns / 1e6 if unit == "ns" else ns / 1e3 if unit == "us" else ns
        name = r["Kernel Name"]
        key = "candidate kernels (generated, k<i>_<stage>)" if re.match(r"k\d+_", name) else name.split("(")[0]
        fam[key][0] += 1
        fam[key][1] += ms
        if a.grid and r["Grid Size"].strip("()").split(",")[0].strip() == a.grid and \
                r["Block Size"].strip("()").split(",")[0].strip() == a.block and re.match(r"k\d+_", name):
            best.append(ms)
    total = sum(v[1] for v in fam.values())
    print(f"{'kernel':48s} {'launches':>9s} {'total ms':>10s} {'share':>7s}")
    for k, (n, ms) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:48s} {n:9d} {ms:10.2f} {100 * ms / total:6.1f}%")
    if best:
        print(f"# best candidate's kernel ({a.block} thr x {a.grid} blocks): {len(best)} launches, "
              f"mean {1e3 * sum(best) / len(best):.1f} us")


if __name__ == "__main__":
    main()
