"""Where a measured candidate's time goes: per-candidate lowering, ptxas and
device seconds over a slice of a golden stream, summarised (sum, percentiles).

  python tools/pipeline_probe.py [CFG] [K] [--ptxas "-O3 ..."] [--out FILE]

--ptxas overrides the candidates' ptxas options (LT_PTXAS_OPT, newline- or
space-separated) so compile-time / kernel-time trade-offs can be compared on
the same States.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


def pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(q * len(xs)))] if xs else None


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", nargs="?", default="RC")
    ap.add_argument("k", type=int, nargs="?", default=128)
    ap.add_argument("--offset", type=int, default=64)
    ap.add_argument("--ptxas", default="")
    ap.add_argument("--min-ms", type=float, default=1.0)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    if args.ptxas:
        os.environ["LT_PTXAS_OPT"] = "\n".join(args.ptxas.split())
    from bench import FLOPS, load_stream
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200.state import replay
    r = measure.configure(device=0, cache_dir=tempfile.mkdtemp(), min_ms=args.min_ms)
    dag, stream = load_stream(args.cfg)
    r.prepare(dag, 0)
    r.measure_programs([replay(dag, h) for h in stream[:16]])           # warm the pools
    progs = [replay(dag, h) for h in stream[args.offset:args.offset + args.k]]
    s0 = dict(r.stats)
    recs = r.measure_programs(progs)
    st = {k: r.stats[k] - s0.get(k, 0) for k in r.stats if isinstance(r.stats[k], (int, float))}
    valid = [x for x in recs if x.status == "valid"]
    dev_us = [x.first_us + x.cost_us * x.repeats for x in valid]
    out = {"cfg": args.cfg, "k": args.k, "ptxas": args.ptxas or "default", "min_ms": args.min_ms,
           "valid": len(valid), "wall_s": st["wall_s"], "rate": args.k / st["wall_s"],
           "compile_s_sum": sum(x.compile_s for x in recs), "lower_s_sum": sum(x.lower_s for x in recs),
           "gpu_s": st["gpu_s"], "idle_s": st["idle_s"], "kernel_s_sum": sum(dev_us) / 1e6,
           "prep_s": st.get("prep_s"), "lt_measure_s": st.get("lt_measure_s"),
           "first_us_p50": pct([x.first_us for x in valid], 0.5), "first_us_p90": pct([x.first_us for x in valid], 0.9),
           "first_us_max": max((x.first_us for x in valid), default=None),
           "compile_s_p50": pct([x.compile_s for x in recs], 0.5), "compile_s_p90": pct([x.compile_s for x in recs], 0.9),
           "compile_s_max": max(x.compile_s for x in recs),
           "best_us": min((x.cost_us for x in valid), default=None),
           "best_tflops": max((FLOPS[args.cfg] / x.cost_us / 1e6 for x in valid), default=None),
           "sum_cost_us": sum(x.cost_us for x in valid)}
    # batch timeline: when lowering finished, when the device started / finished each candidate
    lw = [x.t["lowered"] for x in recs if "lowered" in x.t]
    ends = sorted((x.t["start"], x.t["end"]) for x in recs if "start" in x.t)
    busy = sum(e - b for b, e in ends)
    out["timeline"] = {"last_lowered": max(lw, default=None), "first_device_start": ends[0][0] if ends else None,
                       "last_device_end": ends[-1][1] if ends else None, "device_busy": busy,
                       "device_start_p50": pct([b for b, _ in ends], 0.5),
                       "device_start_p90": pct([b for b, _ in ends], 0.9)}
    print(json.dumps(out), flush=True)
    if args.out:
        with open(args.out, "a") as fh:
            fh.write(json.dumps(out) + "\n")
            for x in recs:
                fh.write(json.dumps({"status": x.status, "first_us": x.first_us, "cost_us": x.cost_us,
                                     "repeats": x.repeats, "compile_s": x.compile_s, "lower_s": x.lower_s,
                                     "key": x.key}) + "\n")
    measure._shutdown()


if __name__ == "__main__":
    main()
