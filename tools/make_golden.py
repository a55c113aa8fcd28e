"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (the reference is importable there, not on the GPU
box):  PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py

Writes
  corpus.json    DAG JSON per workload key + (dag key, history JSON, origin) per State
  features.npz   reference `extract_features` rows for every State (+ row offsets)
  model.json     a CostModel trained by the reference's `train` on corpus features
  scores.npy     reference `CostModel.predict` of every State under model.json
  measure.json   reference `measure_batch` results (status/detail/cost/throughput) and
                 `validate` results for a subset, incl. hand-broken States
  outputs.npz    reference `reference_outputs` (seed-0 `random_inputs`) for small DAGs
Everything is deterministic for the fixed seeds below.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF = os.environ.get("LOOMTUNE_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

import loomtune as LT  # noqa: E402
from loomtune.features import extract_features  # noqa: E402
from loomtune.interp import random_inputs, reference_outputs  # noqa: E402
from loomtune.ir import Annotate, apply_step, history_to_json  # noqa: E402
from loomtune.machine import machine_cost, measure_batch  # noqa: E402
from loomtune.model import TrainHyper, TrainingRecord, train  # noqa: E402
from loomtune.sched import SchedulerParams, TuneSettings, make_task, tune, Objective  # noqa: E402
from loomtune.sketch import generate_sketches  # noqa: E402

from paper_2006_06762_b200.state import workloads as W  # noqa: E402  (new DAG builders)

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")

SMALL = {
    "matmul": dict(n=64, m=64, k=64),
    "matmul_bias_relu": dict(n=32, m=32, k=32),
    "conv2d": dict(h=6, w=6, ci=8, co=8, n=2),
    "conv2d_relu": dict(h=6, w=6, ci=4, co=4),
    "grouped_conv2d": dict(h=6, w=6, ci=8, co=8),
    "norm2": dict(n=8, m=32),
    "elemwise_chain": dict(n=64),
    "batch_matmul": dict(b=4, n=16, m=16, k=8),
    "conv_bn_relu": dict(n=2, h=6, w=6, ci=8, co=8),
}


def ref_dag(name: str, kw: dict):
    """Reference DAG: registry builder, or the new builders re-expressed in the
    reference's own expression types (via the JSON codec)."""
    if name in LT.REGISTRY:
        return LT.build(name, **kw)
    ours = W.build(name, **kw)
    return LT.ComputeDAG.from_json(ours.to_json())


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    dags: dict = {}
    progs: list = []

    def add(key, dag, p, origin):
        dags.setdefault(key, dag.to_json())
        progs.append((key, dag, p, origin))

    # (a) small registry + new workloads, both structures, every sketch
    for name, kw in SMALL.items():
        dag = ref_dag(name, kw)
        key = f"{name}:" + ",".join(f"{k}={v}" for k, v in sorted(kw.items()))
        for struct in ("SSRSRS", "SSSRRSRS"):
            rng = np.random.default_rng(7)
            for sk in generate_sketches(dag, structure=struct):
                for _ in range(5):
                    add(key, dag, LT.sample_program(sk, LT.AnnotationPolicy(), rng), f"sample:{struct}")
    # (b) BASELINE configs, GPU structure
    for cfg in ("G5", "G10", "RC", "TBG", "CL"):
        name, kw = W.CONFIGS[cfg]
        dag = ref_dag(name, kw)
        rng = np.random.default_rng(11)
        for sk in generate_sketches(dag, structure="SSSRRSRS"):
            for _ in range(6):
                add(cfg, dag, LT.sample_program(sk, LT.AnnotationPolicy(), rng), "sample:SSSRRSRS")
    # (c) evolved States from short reference tune runs (mutations, crossover, moves)
    for key, name, kw, budget in (("tune:matmul_bias_relu", "matmul_bias_relu", dict(n=32, m=32, k=32), 3),
                                  ("tune:conv_bn_relu", "conv_bn_relu", dict(n=2, h=6, w=6, ci=8, co=8), 3)):
        dag = ref_dag(name, kw)
        task = make_task(key, dag, structure="SSSRRSRS")
        seen = []
        tune([task], Objective(), budget, TuneSettings(), SchedulerParams(), seed=0,
             log_sink=lambda rec: seen.append(rec) if rec.get("kind") == "measure" else None)
        for rec in seen:
            p = LT.replay(dag, rec["history"])
            add(key, dag, p, "tune")

    # features
    rows, offs = [], [0]
    for _, _, p, _ in progs:
        f = extract_features(p)
        rows.append(f)
        offs.append(offs[-1] + len(f))
    X = np.vstack(rows)
    np.savez_compressed(os.path.join(OUT, "features.npz"), rows=X, offsets=np.asarray(offs, np.int64))

    # model trained by the reference on machine-model throughputs
    best: dict = {}
    costs = []
    for key, _, p, _ in progs:
        c = machine_cost(p)
        costs.append(c)
        best[key] = min(best.get(key, math.inf), c)
    recs = [TrainingRecord(key, p.history, best[key] / c, feats=f)
            for (key, _, p, _), c, f in zip(progs, costs, rows)]
    model = train(recs, TrainHyper())
    with open(os.path.join(OUT, "model.json"), "w") as fh:
        json.dump(model.to_json(), fh)
    np.save(os.path.join(OUT, "scores.npy"), np.asarray([model.predict(p) for _, _, p, _ in progs]))

    with open(os.path.join(OUT, "corpus.json"), "w") as fh:
        json.dump({"dags": dags,
                   "programs": [{"dag": k, "history": history_to_json(p.history), "origin": o}
                                for k, _, p, o in progs]}, fh)

    # measurement semantics on small States (statuses, details, normalisation)
    meas = []
    for name in ("matmul", "matmul_bias_relu", "conv2d_relu", "batch_matmul"):
        kw = SMALL[name]
        dag = ref_dag(name, kw)
        key = f"{name}:" + ",".join(f"{k}={v}" for k, v in sorted(kw.items()))
        rng = np.random.default_rng(3)
        batch = [LT.naive_program(dag)]
        for sk in generate_sketches(dag, structure="SSSRRSRS"):
            batch.append(LT.sample_program(sk, LT.AnnotationPolicy(), rng))
        first = batch[0].stages[-1]
        broken = apply_step(apply_step(batch[0], Annotate(first.name, first.loops[0].id, "parallel")),
                            Annotate(first.name, first.loops[1].id, "parallel"))
        batch.append(broken)
        res = measure_batch(batch)
        meas.append({"dag": key, "histories": [history_to_json(p.history) for p in batch],
                     "validate": [LT.validate(p) for p in batch],
                     "results": [[r.cost if math.isfinite(r.cost) else "inf", r.throughput, r.status, r.detail]
                                 for r in res]})
    with open(os.path.join(OUT, "measure.json"), "w") as fh:
        json.dump(meas, fh)

    # State-free ground truth at small shapes
    outs = {}
    for name, kw in SMALL.items():
        dag = ref_dag(name, kw)
        ins = random_inputs(dag, np.random.default_rng(0))
        for o, arr in reference_outputs(dag, ins).items():
            outs[f"{name}/{o}"] = arr
    np.savez_compressed(os.path.join(OUT, "outputs.npz"), **outs)
    print(f"{len(progs)} States, {len(X)} rows, {len(model.trees)} trees -> {OUT}")


if __name__ == "__main__":
    main()
