"""Whole-network tuning (BASELINE.json configs[4]): the
reference's unchanged multi-task `tune` (gradient task scheduler,
`src/sched.py:276-375`) over every distinct ResNet-50 subgraph, with the B200
hot path installed.

  python tools/tune_network.py BUDGET [SEED] [--batch N] [--gpu-sampler] [--gpu-sketches] [--gpu-rules] [--tasks K] [--fused]

Tasks come from `paper_2006_06762_b200.resnet50.tasks` (--fused: each conv with its BN + ReLU; 23 conv shapes + the
classifier, weights = instance counts).  Under torchrun each rank measures its
shard of every batch and the records are all-gathered
(`paper_2006_06762_b200.dist.measure_batch_sharded`); every rank runs the same
deterministic scheduler.  Writes gpurun_out/tune_network.json: per-task best
latency and TFLOP/s, the weighted network latency sum, the scheduler's
allocation, time split and runner statistics.
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

from paper_2006_06762_b200 import integrate, measure, resnet50  # noqa: E402


def main() -> None:
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    budget = int(args[0])
    seed = int(args[1]) if len(args) > 1 else 0
    opt = {a.split("=")[0]: (a.split("=")[1] if "=" in a else True) for a in sys.argv[1:] if a.startswith("--")}
    batch = int(opt.get("--batch", 16))
    n_tasks = int(opt.get("--tasks", 0)) or None
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://")
        torch.cuda.set_device(local)
    runner = measure.configure(device=local, cache_dir="",
                               workers=max(1, (os.cpu_count() or 2) // world - (1 if world == 1 else 0)),
                               lower_workers=max(1, min(8, (os.cpu_count() or 2) // (2 * world))))
    sched = importlib.import_module("loomtune.sched")
    orig = integrate.install(LT, gpu_sampler=bool(opt.get("--gpu-sampler")),
                             gpu_features=bool(opt.get("--gpu-features")))
    # under torchrun install() shards every measurement batch and every evolution
    # population across the ranks (dist.measure_batch_sharded / score_batch_sharded)
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

    counts = {"measured": 0, "valid": 0}

    def sink(rec):
        if rec.get("kind") == "measure":
            counts["measured"] += 1
            counts["valid"] += rec["status"] == "valid"

    specs = resnet50.tasks(batch, fusion="conv_bn_relu" if opt.get("--fused") else "conv")[:n_tasks]
    tasks = []
    t0 = time.perf_counter()
    for name, dag, weight in specs:
        ldag = LT.ComputeDAG.from_json(dag.to_json())
        tasks.append(LT.make_task(name, ldag, weight=float(weight), dnn="resnet50", structure="SSSRRSRS"))
        if opt.get("--gpu-sketches") or opt.get("--gpu-rules"):
            integrate.gpu_sketch_policy(LT, tasks[-1], gpu_rules=bool(opt.get("--gpu-rules")))
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    LT.tune(tasks, LT.Objective(), budget, LT.TuneSettings(batch_size=16), LT.SchedulerParams(), seed=seed,
            log_sink=sink)
    wall = time.perf_counter() - t0
    integrate.uninstall(LT, orig)
    per_task = []
    net_us = 0.0
    for (name, dag, weight), t in zip(specs, tasks):
        fl = resnet50.flops(dag)
        per_task.append({"task": name, "weight": weight, "units": t.units, "naive_us": t.naive_cost,
                         "best_us": t.best_cost, "tflops": fl / (t.best_cost * 1e-6) / 1e12,
                         "speedup_vs_naive": (t.naive_cost / t.best_cost) if t.naive_cost else None})
        net_us += weight * t.best_cost
    naive_net = sum(w * t.naive_cost for (_, _, w), t in zip(specs, tasks))
    out = {"config": "resnet50 whole network", "batch": batch, "budget": budget, "seed": seed, "n_gpus": world,
           "tasks": len(tasks), "gpu_sketches": bool(opt.get("--gpu-sketches")), "wall_s": wall, "setup_s": t_setup, "timers": timers, **counts,
           "measured_per_s": counts["measured"] / timers["measure"] if timers["measure"] else None,
           "network_latency_us": net_us, "naive_network_latency_us": naive_net,
           "network_tflops": sum(w * resnet50.flops(d) for _, d, w in specs) / (net_us * 1e-6) / 1e12,
           "runner": runner.stats, "per_task": per_task}
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", "tune_network.json"), "w") as fh:
            json.dump(out, fh)
        print(json.dumps({k: v for k, v in out.items() if k != "per_task"}))
        for t in per_task:
            print(json.dumps(t))
    measure._shutdown()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
