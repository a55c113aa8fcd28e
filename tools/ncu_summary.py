"""Condense an ncu report (`--set full`) into the per-kernel summary kept under
profiles/: speed-of-light, issue, memory, launch and occupancy lines, plus the
DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum).

  python tools/ncu_summary.py REPORT.ncu-rep [--header TEXT] [--traffic-key SHA1 --config CFG]

With --traffic-key the DRAM bytes are also merged into profiles/traffic.json
(bench.py's `roofline.traffic` for that candidate source).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import OrderedDict

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
KEEP = ("Memory Throughput", "DRAM Throughput", "Duration", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate", "Block Size", "Grid Size", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Waves Per SM", "Theoretical Occupancy", "Achieved Occupancy")


def ncu_csv(rep: str, page: str, extra=()) -> list:
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True,
                         check=True).stdout
    start = out.find('"')
    return list(csv.reader(io.StringIO(out[start:])))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--header", default="")
    ap.add_argument("--traffic-key", default="")
    ap.add_argument("--config", default="RC")
    a = ap.parse_args()
    rows = ncu_csv(a.report, "details")
    head, body = rows[0], rows[1:]
    ix = {k: i for i, k in enumerate(head)}
    if a.header:
        print(f"# {a.header}")
    seen = set()
    for r in body:
        name = r[ix["Kernel Name"]].split("(")[0]
        key = (name, r[ix["Metric Name"]])          # first launch of each kernel
        if r[ix["Metric Name"]] in KEEP and key not in seen:
            seen.add(key)
            print(f"{name:14s} {r[ix['Section Name']]:34s} {r[ix['Metric Name']]:34s} "
                  f"{r[ix['Metric Value']]:>12s} {r[ix['Metric Unit']]}")
    raw = ncu_csv(a.report, "raw", ("--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"))
    rh, units, rb = raw[0], raw[1], raw[2:]
    rix = {k: i for i, k in enumerate(rh)}
    kernels = OrderedDict()
    for r in rb:
        name = r[rix["Kernel Name"]].split("(")[0]
        if name in kernels:
            continue

        def val(m):
            v = float(r[rix[m]].replace(",", ""))
            u = units[rix[m]]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
                     "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3, "s": 1e6, "second": 1e6}.get(u, 1)
            return v * scale
        kernels[name] = {"dram_read_bytes": val("dram__bytes_read.sum"),
                         "dram_write_bytes": val("dram__bytes_write.sum"),
                         "us": val("gpu__time_duration.sum")}
    total = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in kernels.values())
    for n, k in kernels.items():
        print(f"# {n}: DRAM read {k['dram_read_bytes'] / 1e6:.2f} MB, write {k['dram_write_bytes'] / 1e6:.2f} MB, "
              f"{k['us']:.1f} us")
    print(f"# DRAM bytes per launch of the candidate: {total / 1e6:.2f} MB")
    if a.traffic_key:
        path = os.path.join(ROOT, "profiles", "traffic.json")
        data = json.load(open(path)) if os.path.exists(path) else {}
        data[a.traffic_key] = {"config": a.config, "dram_bytes_per_launch": total, "kernels": kernels,
                               "source": f"ncu --set full --clock-control none (cold L2 per replay), {a.report}"}
        with open(path, "w") as fh:
            json.dump(data, fh, indent=1)


if __name__ == "__main__":
    main()
