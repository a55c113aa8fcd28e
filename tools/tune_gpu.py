"""Run the reference's unchanged tuner with the B200 hot path installed.

  python tools/tune_gpu.py CFG BUDGET [SEED] [--gpu-sampler] [--gpu-features] [--gpu-sketches] [--gpu-rules]

Imports `loomtune` from baseline/_ref (pip-installed copy of the reference;
falls back to /root/reference when present), installs the drop-ins
(`paper_2006_06762_b200.integrate.install`), tunes one BASELINE config with
structure SSSRRSRS, and writes gpurun_out/tune_<CFG>.json: per-unit best cost,
time split (evolve / measure / train), every measured history, and the best
program's GFLOP/s.
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "loomtune")):
        sys.path.insert(0, cand)
        break

import importlib  # noqa: E402

import loomtune as LT  # noqa: E402

from bench import FLOPS  # noqa: E402
from paper_2006_06762_b200 import integrate, measure  # noqa: E402
from paper_2006_06762_b200.state import workloads as W  # noqa: E402


def main() -> None:
    cfg, budget = sys.argv[1], int(sys.argv[2])
    seed = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 0
    gpu_sampler = "--gpu-sampler" in sys.argv
    gpu_features = "--gpu-features" in sys.argv
    gpu_sketches = "--gpu-sketches" in sys.argv or "--gpu-rules" in sys.argv
    gpu_rules = "--gpu-rules" in sys.argv
    name, kw = W.CONFIGS[cfg]
    dag = LT.ComputeDAG.from_json(W.build(name, **kw).to_json())
    runner = measure.configure(device=0, cache_dir="")
    sched = importlib.import_module("loomtune.sched")
    orig = integrate.install(LT, gpu_sampler=gpu_sampler, gpu_features=gpu_features)
    timers = {"evolve": 0.0, "measure": 0.0, "train": 0.0}

    def timed(key, fn):
        def w(*a, **k):
            t = time.perf_counter()
            try:
                return fn(*a, **k)
            finally:
                timers[key] += time.perf_counter() - t
        return w
    sched.evolve = timed("evolve", sched.evolve)
    sched.measure_batch = timed("measure", sched.measure_batch)
    sched.train = timed("train", sched.train)
    measured = []

    def sink(rec):
        if rec.get("kind") == "measure":
            measured.append({"history": LT.ir.history_to_json(rec["history"]) if hasattr(LT, "ir") else
                             importlib.import_module("loomtune.ir").history_to_json(rec["history"]),
                             "cost": rec["cost"], "status": rec["status"], "iteration": rec["iteration"]})
    task = LT.make_task(cfg, dag, structure="SSSRRSRS")
    paths = integrate.gpu_sketch_policy(LT, task, gpu_rules=gpu_rules) if gpu_sketches else None
    t0 = time.perf_counter()
    res = LT.tune([task], LT.Objective(), budget, LT.TuneSettings(), LT.SchedulerParams(), seed=seed, log_sink=sink)
    wall = time.perf_counter() - t0
    integrate.uninstall(LT, orig)
    best = task.best_cost
    out = {"config": cfg, "budget": budget, "seed": seed, "gpu_sampler": gpu_sampler, "gpu_features": gpu_features,
           "gpu_rules": gpu_rules,
           "gpu_sketches": [list(map(str, p)) for p in paths] if paths else None, "wall_s": wall, "timers": timers,
           "measured": len(measured), "valid": sum(m["status"] == "valid" for m in measured),
           "best_us": best, "best_tflops": FLOPS[cfg] / (best * 1e-6) / 1e12,
           "latency_curve": task.latency, "runner": runner.stats,
           "best_history": importlib.import_module("loomtune.ir").history_to_json(task.best_program.history),
           "history": measured}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    import gzip
    # every measured history is kept, gzip-compressed (a 2000-trial tune is ~8 MB as JSON)
    with gzip.open(os.path.join(ROOT, "gpurun_out", f"tune_{cfg}_s{seed}{'_rules' if gpu_rules else ''}.json.gz"),
                   "wt") as fh:
        json.dump(out, fh)
    print(json.dumps({k: v for k, v in out.items() if k not in ("history", "best_history", "latency_curve")}))
    print("latency curve (us):", [round(x, 1) for x in task.latency])
    measure._shutdown()


if __name__ == "__main__":
    main()
