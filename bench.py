"""Headline benchmark: measured candidates/sec of the B200 measurement pipeline.

Metric (both arms, identical string): "measured candidates/sec (<CFG>, SSSRRSRS)"
= candidates measured / wall seconds of the measuring region.

* A step = measuring one batch of B fresh candidate States of the BASELINE
  config (default RC = ResNet-50 conv2d N16 56x56x64->64 3x3, BASELINE.json
  configs[1]) through the drop-in `measure_batch`: validate -> lower -> ptxas
  (empty cubin cache, exact constants) -> run on the B200 -> verify every output
  against the fp64 ground truth on the device -> time.  States come from
  tests/golden/streams/<CFG>.json.gz (the reference's own sampler, filtered to
  legal launches); step s of the run measures stream[s*B*N:(s+1)*B*N] (each rank
  its own shard), so warm-up steps and timed steps never share a State.
* `value`: inputs and ground truth resident in HBM when the timed region starts;
  the region (CUDA events, synchronize + barrier on both sides, max over ranks)
  contains the whole host pipeline.  `e2e`: the same States again through the
  public `measure_batch` from scratch — a fresh measuring process (new CUDA
  context, empty cubin cache, its own untimed warm-up steps) and, every timed
  step, the DAG's inputs copied from host memory and the fp64 ground truth
  recomputed, results read back.
* `--impl reference`: the reference's own runner (`loomtune.machine.measure_batch`,
  src/machine.py:249-285, imported unchanged from baseline/_ref) on the same
  timed States, one State per task on a process pool over all host cores (a work
  queue: no per-step barrier), wall clock from first submit to last result.

Multi-GPU (torchrun): each rank measures its shard of every step's batch
(measurement units are independent); only the (status, cost)
records are gathered (NCCL all_gather).  value = candidates of all ranks /
max-over-ranks time.
"""

from __future__ import annotations

import argparse
import gzip
import json
import math
import os
import signal
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOPS = {"RC": 2 * 16 * 56 * 56 * 64 * 64 * 9, "G10": 2 * 1024 ** 3, "G5": 2 * 512 ** 3,
         "TBG": 2 * 192 * 128 * 128 * 64, "CL": 2 * 16 * 28 * 28 * 128 * 128 * 9}
NAMES = {"RC": "ResNet-50 conv2d N16 56x56x64->64 3x3 s1", "G10": "GEMM 1024^3", "G5": "GEMM 512^3",
         "TBG": "batched GEMM 192x128x128x64", "CL": "ConvLayer N16 28x28x128->128 3x3 + BN + ReLU"}
RATE_DEF = ("candidates measured / wall seconds of the measuring region; ours: device-event-bracketed steps "
            "of B candidates through measure_batch (validate+lower+compile+run+verify+time, empty cubin "
            "cache); reference: loomtune.machine.measure_batch (validate + shrunken-twin interpret + "
            "analytical cost) on the same States, work queue over all host cores")


def metric(cfg: str) -> str:
    return f"measured candidates/sec ({cfg}, SSSRRSRS)"


def load_stream(cfg: str):
    from paper_2006_06762_b200.state import ComputeDAG, history_from_json
    with gzip.open(os.path.join(ROOT, "tests", "golden", "streams", f"{cfg}.json.gz"), "rt") as fh:
        data = json.load(fh)
    return ComputeDAG.from_json(data["dag"]), [history_from_json(h) for h in data["histories"]]


def bounded_batch(args, n_states: int, world: int) -> int:
    """Candidates per rank per step: --batch, unless the stream is too short for
    every timed candidate to be a fresh State (then the largest batch it allows);
    both arms use the same value, hence the same States."""
    if (args.warmup + args.steps) * args.batch * world <= n_states:
        return args.batch
    b = n_states // ((args.warmup + args.steps) * world)
    if b < 1:
        raise SystemExit(f"stream has {n_states} States, too few for {world} ranks")
    return b


def step_slice(stream: list, step: int, batch: int, world: int) -> list:
    lo = step * batch * world
    return stream[lo:lo + batch * world]


class Clocks:
    """nvidia-smi sampler over the timed region (the recipe's clocks line)."""

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, ValueError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [r for r in rows if r[7].isdigit() and int(r[7]) > 0] or rows
        mhz = [float(r[0]) for r in busy if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in busy for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(mhz) if mhz else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(busy)}


# ---- the reference's CPU paths (work queue over all host cores) ---------------

class _Capped(Exception):
    pass


def _alarm(signum, frame):
    raise _Capped()


def _ref_worker_init():
    sys.path.insert(0, ROOT)
    from paper_2006_06762_b200.reference import loomtune  # noqa: F401  (baseline/_ref)
    import loomtune.machine  # noqa: F401
    signal.signal(signal.SIGALRM, _alarm)


def _ref_measure(item):
    """One State through the reference's own `measure_batch` (src/machine.py:249-285)."""
    dag_json, hist, cap = item
    from loomtune.graph import ComputeDAG
    from loomtune.ir import history_from_json, replay
    from loomtune.machine import measure_batch
    t0 = time.perf_counter()
    signal.setitimer(signal.ITIMER_REAL, cap)
    try:
        p = replay(ComputeDAG.from_json(json.loads(dag_json)), history_from_json(hist))
        status = measure_batch([p])[0].status
    except _Capped:
        status = "capped"
    finally:
        signal.setitimer(signal.ITIMER_REAL, 0)
    return status, time.perf_counter() - t0


def _ref_interpret(item):
    """The reference's only full-size execution of a State: `interpret` on the
    real inputs (src/interp.py:318-352) — what the B200 runner does per candidate."""
    dag_json, hist, cap = item
    import numpy as np
    from loomtune.graph import ComputeDAG
    from loomtune.interp import interpret, random_inputs
    from loomtune.ir import history_from_json, replay
    t0 = time.perf_counter()
    signal.setitimer(signal.ITIMER_REAL, cap)
    try:
        dag = ComputeDAG.from_json(json.loads(dag_json))
        interpret(replay(dag, history_from_json(hist)), random_inputs(dag, np.random.default_rng(0)))
        status = "valid"
    except _Capped:
        status = "capped"
    finally:
        signal.setitimer(signal.ITIMER_REAL, 0)
    return status, time.perf_counter() - t0


def _ref_predict(item):
    """`extract_features` + `CostModel.predict` (src/features.py:420-425,
    src/model.py:98-108) over a chunk of programs."""
    dag_json, hists, model_json = item
    from loomtune.graph import ComputeDAG
    from loomtune.ir import history_from_json, replay
    from loomtune.model import CostModel
    dag = ComputeDAG.from_json(json.loads(dag_json))
    model = CostModel.from_json(model_json)
    progs = [replay(dag, history_from_json(h)) for h in hists]
    t0 = time.perf_counter()
    for p in progs:
        model.predict(p)
    return len(progs), time.perf_counter() - t0


class RefPool:
    """Process pool over all host cores with the reference imported in every worker."""

    def __init__(self, cores: int):
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor
        self.cores = cores
        self.ex = ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("spawn"),
                                      initializer=_ref_worker_init)
        for f in [self.ex.submit(int, 0) for _ in range(cores * 2)]:     # workers up before any clock
            f.result()

    def run(self, fn, items: list) -> tuple:
        """(results, wall seconds from first submit to last result)."""
        t0 = time.perf_counter()
        res = list(self.ex.map(fn, items))
        return res, time.perf_counter() - t0

    def close(self):
        self.ex.shutdown(wait=True, cancel_futures=True)


def ref_measure_rate(pool: RefPool, dag, histories: list, cap: float) -> dict:
    from paper_2006_06762_b200.state import history_to_json
    dj = json.dumps(dag.to_json())
    items = [(dj, history_to_json(h), cap) for h in histories]
    res, wall = pool.run(_ref_measure, items)
    return {"value": len(items) / wall, "candidates": len(items), "wall_s": wall,
            "core_s": sum(t for _, t in res), "capped": sum(s == "capped" for s, _ in res)}


def ref_interpret_rate(pool: RefPool, dag, histories: list, cap: float) -> dict:
    from paper_2006_06762_b200.state import history_to_json
    dj = json.dumps(dag.to_json())
    items = [(dj, history_to_json(h), cap) for h in histories]
    res, wall = pool.run(_ref_interpret, items)
    return {"value": len(items) / wall, "candidates": len(items), "wall_s": wall,
            "capped": sum(s == "capped" for s, _ in res)}


def ref_predict_rate(pool: RefPool, dag, histories: list, model_json: dict, chunk: int = 16) -> dict:
    from paper_2006_06762_b200.state import history_to_json
    dj = json.dumps(dag.to_json())
    hj = [history_to_json(h) for h in histories]
    items = [(dj, hj[i:i + chunk], model_json) for i in range(0, len(hj), chunk)]
    res, wall = pool.run(_ref_predict, items)
    n = sum(k for k, _ in res)
    return {"value": n / wall, "programs": n, "wall_s": wall, "predict_core_s": sum(t for _, t in res)}


# ---- our scoring / training legs ----------------------------------------------

def scoring_bench(device: int, programs: list, reps: int = 20) -> dict:
    """Population scoring (features + trees) over a synthetic population of 2^16
    programs (replicated stream States): device-resident kernel times (CUDA
    events on the launching stream) and the host e2e rate through predict_batch."""
    import ctypes
    import numpy as np
    import torch
    from paper_2006_06762_b200 import runtime as rt
    from paper_2006_06762_b200.encode import encode_batch
    from paper_2006_06762_b200.model import GpuCostModel
    lib = rt.load()
    model = GpuCostModel.from_json(json.load(open(os.path.join(ROOT, "tests", "golden", "model.json"))))
    base_words, base_off, base_prog = encode_batch(programs)
    n_rep = max(1, (1 << 16) // len(programs))
    words = np.tile(base_words, n_rep)
    stmt_off = np.concatenate([base_off[:-1] + i * len(base_words) for i in range(n_rep)] + [[len(words)]])
    prog_off = np.concatenate([base_prog[:-1] + i * base_prog[-1] for i in range(n_rep)]
                              + [[base_prog[-1] * n_rep]]).astype(np.int64)
    n_stmt, n_prog = len(stmt_off) - 1, len(prog_off) - 1
    dev = torch.device("cuda", device)
    d_words = torch.from_numpy(words).to(dev)
    d_soff = torch.from_numpy(stmt_off).to(dev)
    d_poff = torch.from_numpy(prog_off).to(dev)
    d_rows = torch.empty((n_stmt, 164), dtype=torch.float64, device=dev)
    d_rs = torch.empty(n_stmt, dtype=torch.float64, device=dev)
    d_sc = torch.empty(n_prog, dtype=torch.float64, device=dev)
    d_err = torch.zeros(1, dtype=torch.int32, device=dev)
    h = model.handle()
    n_trees, n_used = ctypes.c_int(), ctypes.c_int()
    rt.check(lib.lt_model_info(h, ctypes.byref(n_trees), ctypes.byref(n_used)), "model info")
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    def feats():
        rt.check(lib.lt_features_device_cm(d_words.data_ptr(), d_soff.data_ptr(), n_stmt, d_rows.data_ptr(),
                                           d_err.data_ptr(), sp), "features")

    def trees():
        rt.check(lib.lt_predict_cols_device(h, d_rows.data_ptr(), n_stmt, d_rs.data_ptr(), sp), "trees")

    def segsum():
        rt.check(lib.lt_segment_sum_device(d_rs.data_ptr(), d_poff.data_ptr(), n_prog, d_sc.data_ptr(), sp), "sum")

    out = {}
    for name, fn in (("features", feats), ("trees", trees), ("segsum", segsum)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        out[name + "_ms"] = e0.elapsed_time(e1) / reps
    model.predict_batch(programs)                       # warm
    t0 = time.perf_counter()
    sc = model.predict_batch(programs * n_rep)          # host e2e: encode + H2D + fused scoring + D2H
    out["e2e_s"] = time.perf_counter() - t0
    out.update(n_prog=n_prog, n_stmt=n_stmt, words_bytes=int(words.nbytes), n_used=n_used.value,
               scores_finite=bool(np.isfinite(sc).all()))
    return out


def train_bench(n_prog: int = 1500) -> dict:
    """GBDT training: `gbdt.train` (trees fitted on the
    B200) vs the reference's own `train` (loomtune.model.train, 1 core) on the
    same records: stream States of four configs, labels U(0.05, 1), default
    hyper (30 trees, depth 6).  Models must be identical."""
    import numpy as np
    from loomtune.model import TrainHyper, TrainingRecord
    from loomtune.model import train as ref_train
    from paper_2006_06762_b200 import gbdt
    from paper_2006_06762_b200.features import extract_features_batch
    from paper_2006_06762_b200.state import replay
    feats, hists = [], []
    for cfg in ("RC", "G10", "CL", "TBG"):
        dag, stream = load_stream(cfg)
        progs = [replay(dag, h) for h in stream[:n_prog // 4]]
        feats += extract_features_batch(progs)
        hists += [p.history for p in progs]
    y = np.random.default_rng(0).uniform(0.05, 1.0, len(feats))
    recs = [TrainingRecord("d", h, float(v), feats=f) for h, v, f in zip(hists, y, feats)]
    gbdt.train(recs[:50], TrainHyper(trees=2))       # warm-up
    t0 = time.perf_counter()
    got = gbdt.train(recs, TrainHyper()).to_json()
    gpu_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    want = ref_train(recs, TrainHyper()).to_json()
    cpu_s = time.perf_counter() - t0
    return {"programs": len(feats), "rows": int(sum(len(f) for f in feats)), "trees": 30, "depth": 6,
            "gpu_s": gpu_s, "cpu_s": cpu_s, "speedup": cpu_s / gpu_s,
            "identical": json.dumps(got, sort_keys=True) == json.dumps(want, sort_keys=True),
            "cpu_kind": "reference (loomtune.model.train, 1 core)"}


def best_found_programs() -> dict:
    """The best program the reference's tuner found per config with the B200 path
    installed (profiles/r02_tuned_best.json: tools/tune_gpu.py at BASELINE.json's
    trial counts), as {cfg: (dag, history, provenance)}."""
    from paper_2006_06762_b200.state import config_dag, history_from_json
    try:
        with open(os.path.join(ROOT, "profiles", "r02_tuned_best.json")) as fh:
            raw = json.load(fh)
    except (OSError, ValueError):
        return {}
    return {c: (config_dag(c), history_from_json(v["history"]), v.get("source", ""))
            for c, v in raw.items() if c in FLOPS}


def traffic_of(sha1: str):
    """DRAM bytes per launch of a profiled candidate (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            hit = json.load(fh).get(sha1)
        return hit["dram_bytes_per_launch"] if hit else None
    except (OSError, ValueError, KeyError):
        return None


# ---- reference arm ---------------------------------------------------------------

def run_reference(args, cores: int) -> None:
    dag, stream = load_stream(args.config)
    world = args.gpus
    args.batch = bounded_batch(args, len(stream), world)
    timed = [h for s in range(args.warmup, args.warmup + args.steps)
             for h in step_slice(stream, s, args.batch, world)]
    pool = RefPool(cores)
    try:
        ref_measure_rate(pool, dag, step_slice(stream, 0, args.batch, world)[:cores], args.cpu_seconds)  # warm
        r = ref_measure_rate(pool, dag, timed, args.cpu_seconds)
    finally:
        pool.close()
    v = r["value"]
    print(json.dumps({
        "impl": "reference", "metric": metric(args.config), "value": v, "unit": "cand/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * r["wall_s"] / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": NAMES[args.config], "candidates_per_step": args.batch * world,
                   "stream": f"tests/golden/streams/{args.config}.json.gz", "rate": RATE_DEF},
        "cpu_baseline": {"value": v, "unit": "cand/s", "cores": cores, "kind": "reference",
                         "sample": f"the {r['candidates']} States of the timed steps through loomtune.machine."
                                   f"measure_batch on {cores} processes; {r['capped']} stopped at the "
                                   f"{args.cpu_seconds:g} s cap and counted as measured (optimistic)"},
        "e2e": {"value": v, "unit": "cand/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


# ---- our arm ------------------------------------------------------------------------

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="RC", choices=sorted(FLOPS))
    ap.add_argument("--batch", type=int, default=128, help="candidates per rank per step")
    ap.add_argument("--cpu-seconds", type=float, default=30.0,
                    help="cap on one reference candidate's CPU time (capped ones count as measured)")
    ap.add_argument("--sub-configs", default="G10,CL", help="extra configs measured in the same run ('' = none)")
    ap.add_argument("--sub-steps", type=int, default=4)
    ap.add_argument("--no-scoring", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baselines (development runs)")
    ap.add_argument("--no-stage", action="store_true",
                    help="do not lower/compile step s+1 behind step s (each step from scratch)")
    ap.add_argument("--compile-workers", type=int, default=0, help="ptxas worker processes per rank (0: auto)")
    ap.add_argument("--lower-workers", type=int, default=0, help="lowering processes per rank (0: auto)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cores = os.cpu_count() or 1

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cores)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200 import runtime as rt
    from paper_2006_06762_b200.dist import measure_batch_sharded as sharded_measure
    from paper_2006_06762_b200.state import replay

    workers = args.compile_workers or max(1, cores // world - (1 if world == 1 else 0))
    lower_workers = args.lower_workers or max(1, min(8, cores // (2 * world)))
    runner = measure.configure(device=local, workers=workers, cache_dir=tempfile.mkdtemp(prefix="lt_cubin_"),
                               lower_workers=lower_workers)
    l2_flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")     # 256 MB > 126 MB L2

    def sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def run_steps(dag, stream, first: int, n: int, e2e: bool, batch: int = 0) -> tuple:
        """Time n steps with CUDA events on the current stream; max over ranks."""
        batch = batch or args.batch
        progs = [[replay(dag, h) for h in step_slice(stream, first + s, batch, world)] for s in range(n)]
        results, records = [], []
        sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s, ps in enumerate(progs):
            l2_flush.zero_()                   # 256 MB write: no step starts with a warm L2
            if e2e:                            # inputs from pinned host memory, ground truth recomputed
                runner.refresh()
            # steps are pipelined: the next step's candidates are lowered and compiled
            # behind this one (never across the edge of the timed region)
            nxt = progs[s + 1] if (s + 1 < len(progs) and not args.no_stage) else None
            results.append(sharded_measure(ps, stage=nxt))   # NCCL all_gather of (status, cost) records
            records.append(list(runner.last_records))
        e1.record()
        sync()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, results, records

    def summarise(cfg, ms, results, records, steps) -> dict:
        n_total = sum(len(rs) for rs in results)
        costs = [r.cost for rs in results for r in rs if r.status == "valid"]
        best_us = min(costs) if costs else float("nan")
        best = min((r for rs in records for r in rs if r.status == "valid"), key=lambda r: r.cost_us, default=None)
        achieved = FLOPS[cfg] / (best_us * 1e-6) / 1e12 if math.isfinite(best_us) else None
        return {"value": n_total / (ms / 1000.0), "ms": ms, "ms_per_step": ms / steps, "measured": n_total,
                "valid": len(costs), "best_us": best_us, "achieved": achieved,
                "best_sha1": best.key if best else None, "best_kernels": best.info.get("kernels") if best else None}

    # ---- headline config --------------------------------------------------------------
    dag, stream = load_stream(args.config)
    args.batch = bounded_batch(args, len(stream), world)
    need = (args.warmup + args.steps) * args.batch * world
    runner.prepare(dag, 0)                                   # inputs + fp64 ground truth resident
    run_steps(dag, stream, 0, args.warmup, False)           # warm-up: compile workers, clocks, lowering pool
    for k in list(runner.stats):
        runner.stats[k] = 0 if isinstance(runner.stats[k], int) else 0.0
    io0 = dict(runner.io)
    with Clocks(local) as clk:
        ms, results, records = run_steps(dag, stream, args.warmup, args.steps, False)
    stats = dict(runner.stats)
    head = summarise(args.config, ms, results, records, args.steps)
    timed_records = [r for step in records for r in step]
    # our kernels launched in the timed region: per measured candidate, its kernels x
    # (warm-up + repeats), one NaN-poison and one verification launch per output, one
    # poison launch per intermediate buffer
    n_launch = sum(len(r.info.get("kernels", [])) * (1 + r.repeats) + 2 * r.n_outputs
                   for r in timed_records if r.n_outputs)
    io1 = dict(runner.io)

    # e2e: the timed steps' own States from scratch through the public API
    runner.close()
    runner = measure.configure(device=local, workers=workers, cache_dir=tempfile.mkdtemp(prefix="lt_cubin_e2e_"),
                               lower_workers=lower_workers)
    runner.prepare(dag, 0)
    run_steps(dag, stream, 0, args.warmup, True)            # warm-up: the same untimed steps as above
    io_e0 = dict(runner.io)
    e2e_ms, _, _ = run_steps(dag, stream, args.warmup, args.steps, True)
    io_e1 = dict(runner.io)
    h2d_step = (io_e1["h2d"] - io_e0["h2d"]) / args.steps
    d2h_step = (io_e1["d2h"] - io_e0["d2h"]) / args.steps
    e2e = args.steps * args.batch * world / (e2e_ms / 1000.0)

    # ---- sub-configs (north_star's named operators) ----------------------------------------
    subs = {}
    for cfg in [c for c in args.sub_configs.split(",") if c and c != args.config]:
        sdag, sstream = load_stream(cfg)
        runner.prepare(sdag, 0)
        sb = min(args.batch, len(sstream) // ((1 + args.sub_steps) * world))     # the stream bounds the batch
        run_steps(sdag, sstream, 0, 1, False, sb)
        sms, sres, srec = run_steps(sdag, sstream, 1, args.sub_steps, False, sb)
        subs[cfg] = summarise(cfg, sms, sres, srec, args.sub_steps)
        subs[cfg]["stream_states"] = [sb * world, (1 + args.sub_steps) * sb * world]
        subs[cfg]["batch"] = sb

    # ---- best-found program per operator (north_star: >= 60% of FP32 peak) -------------
    # measured live here, through the same runner: cost = mean of CUDA-event repeats
    # (>= 1 ms of back-to-back launches) after a verified warm-up run
    found = {}
    for cfg, (fdag, hist, src) in best_found_programs().items():
        (rec,) = runner.measure_programs([replay(fdag, hist)])
        if rec.status == "valid":
            found[cfg] = {"us": rec.cost_us, "achieved": FLOPS[cfg] / (rec.cost_us * 1e-6) / 1e12,
                          "best_sha1": rec.key, "kernels": rec.info.get("kernels"), "source": src,
                          "max_rel_err": rec.max_rel_err}
        else:
            found[cfg] = {"us": None, "achieved": None, "status": rec.status, "detail": rec.detail}

    if world > 1:
        t = torch.tensor([n_launch], device="cuda")
        dist.all_reduce(t)
        n_launch = int(t.item())

    if rank == 0:
        import ctypes
        lib = rt.load()
        tf, pms = ctypes.c_double(), ctypes.c_double()
        rt.check(lib.lt_ffma_peak(local, ctypes.byref(tf), ctypes.byref(pms)), "ffma peak")
        peak = tf.value
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except (OSError, ValueError):
            pass

        def roofline(s, what="best candidate of the timed steps (cost = mean of CUDA-event repeats on the "
                                  "candidate's stream)"):
            return {"bound": "fp32", "achieved": s["achieved"], "peak": peak, "unit": "TFLOP/s",
                    "frac": (s["achieved"] / peak) if s["achieved"] else None,
                    "traffic": traffic_of(s.get("best_sha1") or ""), "kernel": what,
                    "peak_source": "lt_ffma_peak: FFMA issue-bound microbenchmark on this GPU (148 SM x 128 lanes "
                                   "x 2 x clock)"}

        def found_roofline(cfg):
            f = found.get(cfg)
            if not f or f.get("achieved") is None:
                return None
            r = roofline(f, f"best-found {cfg} program ({f['source']}), measured in this run through the runner "
                            "(mean of CUDA-event repeats after a verified warm-up)")
            r["us"] = f["us"]
            r["kernels"] = f["kernels"]
            return r

        line = {
            "metric": metric(args.config), "value": head["value"], "unit": "cand/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": NAMES[args.config], "candidates_per_rank_per_step": args.batch,
                       "stream": f"tests/golden/streams/{args.config}.json.gz (reference sampler, legal launches)",
                       "timed_states": [args.warmup * args.batch * world, need],
                       "compile_workers_per_rank": workers, "cubin_cache": "empty at start", "rate": RATE_DEF,
                       "pipelined_steps": (not args.no_stage and
                                           "step s+1's candidates are lowered and compiled behind step s (compile "
                                           "pool priority: the older step's jobs first); nothing crosses the edges "
                                           "of the timed region"),
                       "l2": "flushed before every timed step (256 MB write); a candidate's cost is the mean of "
                             "back-to-back repeats after its verified warm-up run"},
            "valid": head["valid"], "measured": head["measured"],
            "best_program": {"us": head["best_us"], "tflops": head["achieved"], "flop": FLOPS[args.config],
                             "source_sha1": head["best_sha1"], "kernels": head["best_kernels"]},
            "compile": {"compiled": stats["compiled"], "cache_hits": stats["cache_hits"],
                        "recompiled_O1": stats.get("recompiled", 0),
                        "kernels_compiled": stats.get("kernels_compiled", 0),
                        "kernels_shared": stats.get("kernels_shared", 0),
                        "mean_s": stats["compile_s"] / max(1, stats["compiled"])},
            "pipeline_s": {k: round(stats[k], 3) for k in ("wall_s", "lower_s", "gpu_s", "load_s", "idle_s", "prep_s", "lt_measure_s") if k in stats},
            "roofline": found_roofline(args.config) or roofline(head),
            "roofline_stream_best": roofline(head),
            "e2e": {"value": e2e, "unit": "cand/s", "h2d_bytes_per_step": int(h2d_step),
                    "d2h_bytes_per_step": int(d2h_step), "ms_per_step": e2e_ms / args.steps,
                    "note": "measure_batch from a fresh measuring process (new CUDA context, empty cubin cache, "
                            "its own warm-up steps); every timed step re-uploads the DAG's inputs (fp32 + fp64) and "
                            "recomputes the fp64 ground truth; cubins and launch lists H2D; per-candidate error "
                            "words D2H"},
            "gpu_launches": n_launch,
            "clocks": clk.summary(),
            "faults": {"device_faults": stats.get("device_faults", 0), "restarts": stats.get("restarts", 0)},
        }
        line["configs"] = {c: {"metric": metric(c), "value": s["value"], "unit": "cand/s",
                               "steps": args.sub_steps, "candidates_per_rank_per_step": s["batch"],
                               "measured": s["measured"], "valid": s["valid"],
                               "best_program": {"us": s["best_us"], "tflops": s["achieved"], "flop": FLOPS[c],
                                                "source_sha1": s["best_sha1"]},
                               "roofline": found_roofline(c) or roofline(s),
                               "roofline_stream_best": roofline(s), "timed_states": s["stream_states"]}
                           for c, s in subs.items()}
        line["best_found"] = {c: found_roofline(c) for c in found}
        if not args.no_scoring:
            progs = [replay(dag, h) for h in stream[:256]]
            sb = scoring_bench(local, progs)
            rows_bytes = sb["n_stmt"] * 164 * 8
            fbytes = sb["words_bytes"] + rows_bytes
            tbytes = sb["n_stmt"] * sb["n_used"] * 8 + sb["n_stmt"] * 8
            hbm = peaks.get("hbm_gbs")

            def hbm_roof(nbytes, ms, what, kernel=""):
                ach = nbytes / (ms / 1000) / 1e9
                # DRAM bytes of this kernel on this same population from one ncu --set full
                # capture (tools/profile_scoring.py, profiles/traffic.json "scoring:<kernel>")
                tr = traffic_of(f"scoring:{kernel}") if kernel else None
                return {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                        "frac": ach / hbm if hbm else None, "traffic": tr, "algorithmic_bytes": nbytes,
                        "bytes_def": what, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
            line["scoring"] = {
                "programs": sb["n_prog"], "statements": sb["n_stmt"],
                "device_programs_per_s": sb["n_prog"] / ((sb["features_ms"] + sb["trees_ms"] + sb["segsum_ms"]) / 1000),
                "e2e_programs_per_s": sb["n_prog"] / sb["e2e_s"],
                "features_ms": sb["features_ms"], "trees_ms": sb["trees_ms"], "segsum_ms": sb["segsum_ms"],
                "roofline_features": hbm_roof(fbytes, sb["features_ms"], "encoded words read + rows x 164 x 8 B written",
                                              "features_kernel"),
                "roofline_trees": hbm_roof(tbytes, sb["trees_ms"],
                                           f"rows x {sb['n_used']} used feature columns x 8 B read + rows x 8 B "
                                           "written (the model is shared-memory resident)", "predict_perfect_kernel")}
            line["train"] = train_bench()
        if not args.no_cpu:
            pool = RefPool(cores)
            try:
                timed_h = [h for s in range(args.warmup, args.warmup + args.steps)
                           for h in step_slice(stream, s, args.batch, world)]
                sample = timed_h[:cores]
                cb = ref_measure_rate(pool, dag, sample, args.cpu_seconds)
                line["cpu_baseline"] = {
                    "value": cb["value"], "unit": "cand/s", "cores": cores, "kind": "reference",
                    "sample": f"the first {cb['candidates']} timed States through loomtune.machine.measure_batch, "
                              f"one per process; {cb['capped']} stopped at the {args.cpu_seconds:g} s cap and "
                              "counted as measured (optimistic)"}
                cf = ref_interpret_rate(pool, dag, sample, args.cpu_seconds)
                line["cpu_full_execution"] = {
                    "value": cf["value"], "unit": "cand/s", "cores": cores, "kind": "reference",
                    "sample": f"the same {cf['candidates']} States: full-size loomtune.interp.interpret (the "
                              f"reference's only real execution of a State); {cf['capped']} stopped at the "
                              f"{args.cpu_seconds:g} s cap and counted as done (an upper bound)"}
                model_json = json.load(open(os.path.join(ROOT, "tests", "golden", "model.json")))
                cp = ref_predict_rate(pool, dag, stream[:256] * max(1, 2 * cores // 16), model_json)
                line["cpu_predict"] = {
                    "value": cp["value"], "unit": "programs/s", "cores": cores, "kind": "reference",
                    "sample": f"{cp['programs']} stream programs through loomtune extract_features + "
                              "CostModel.predict (tests/golden/model.json, 30 trees), chunks of 16 per process"}
                for c in subs:
                    sdag, sstream = load_stream(c)
                    r = ref_measure_rate(pool, sdag, step_slice(sstream, 1, subs[c]["batch"], world)[:cores],
                                         args.cpu_seconds)
                    line["configs"][c]["cpu_baseline"] = {
                        "value": r["value"], "unit": "cand/s", "cores": cores, "kind": "reference",
                        "sample": f"the first {r['candidates']} timed States through loomtune.machine.measure_batch; "
                                  f"{r['capped']} capped at {args.cpu_seconds:g} s"}
            finally:
                pool.close()
        print(json.dumps(line))
    runner.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
