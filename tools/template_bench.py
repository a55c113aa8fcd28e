"""Template-quality benchmark: run a FIXED set of candidate States through the
runner and summarise per config (best / median / geomean TFLOP/s and total
device time).  Used before/after every template change; the set is the first
K States of each golden stream (the reference sampler's own candidates) plus
the hand-built tilings in tools/hand_states.py.

  python tools/template_bench.py [K] [--backend ptx|nvrtc] [--out FILE]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("k", type=int, nargs="?", default=48)
    ap.add_argument("--backend", default="ptx")
    ap.add_argument("--configs", default="RC,G10,CL,TBG")
    ap.add_argument("--out", default="")
    ap.add_argument("--offset", type=int, default=0)
    ap.add_argument("--no-hand", action="store_true")
    args = ap.parse_args()
    from bench import FLOPS, load_stream
    from hand_states import states
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200.state import replay
    r = measure.configure(device=0, cache_dir="", backend=args.backend)
    lines = []
    for cfg in args.configs.split(","):
        dag, stream = load_stream(cfg)
        progs = [replay(dag, h) for h in stream[args.offset:args.offset + args.k]]
        recs = r.measure_programs(progs)
        tf = [FLOPS[cfg] / (x.cost_us * 1e-6) / 1e12 for x in recs if x.status == "valid"]
        bad = [x.status + ":" + x.detail[:60] for x in recs if x.status != "valid"]
        line = {"config": cfg, "n": len(progs), "valid": len(tf),
                "best_tflops": max(tf) if tf else None,
                "median_tflops": statistics.median(tf) if tf else None,
                "geomean_tflops": math.exp(sum(math.log(t) for t in tf) / len(tf)) if tf else None,
                "sum_us": sum(x.cost_us for x in recs if x.status == "valid"),
                "invalid": bad[:5]}
        lines.append(line)
        print(json.dumps(line), flush=True)
        for i, x in enumerate(recs):
            lines.append({"cand": cfg, "i": i, "status": x.status, "us": x.cost_us,
                          "kernels": [{k: v for k, v in kk.items() if k != "factors"} | {"factors": kk.get("factors")}
                                      for kk in x.info.get("kernels", [])]})
    for name, p in ([] if args.no_hand else states()):
        (rec,) = r.measure_programs([p])
        cfg = name.split()[0]
        line = {"hand": name, "status": rec.status, "us": rec.cost_us,
                "tflops": FLOPS[cfg] / (rec.cost_us * 1e-6) / 1e12 if rec.status == "valid" else None}
        lines.append(line)
        print(json.dumps(line), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            for ln in lines:
                fh.write(json.dumps(ln) + "\n")
    measure._shutdown()


if __name__ == "__main__":
    main()
