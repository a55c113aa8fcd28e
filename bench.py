"""Headline benchmark: measured candidates/sec of the B200 measurement pipeline.

A step = measuring one batch of fresh candidate States of the BASELINE config
(default RC = ResNet-50 conv2d N16 56x56x64->64 3x3, BASELINE.json configs[1])
through the drop-in `measure_batch`: validate -> lower -> NVRTC compile (empty
cubin cache, exact constants) -> run on the B200 -> verify every output vs the
fp64 ground truth on device -> time.  Candidates come from
tests/golden/streams/<CFG>.json.gz (the reference's own sampler, filtered to
legal launches); every timed step uses States never seen before in the run.
The end-to-end pass (`e2e`) re-measures the same States from scratch: compiled
modules dropped, compile pool restarted on an empty cubin cache, inputs and
packed constants re-uploaded and the fp64 ground truth recomputed every step.

Multi-GPU (torchrun): each rank measures its own disjoint slice of every step's
batch (measurement units are independent); only the measured
records are gathered (NCCL all_gather).  value = candidates of all ranks /
max-over-ranks time.

--impl reference times the reference's CPU runner (oracle/machine.py, a
restatement of src/machine.py:249-285: validate + shrunken-twin interpretation
+ analytical cost) on the same candidates with all host cores.
"""

from __future__ import annotations

import argparse
import gzip
import json
import math
import os
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


def load_stream(cfg: str):
    from paper_2006_06762_b200.state import ComputeDAG, history_from_json
    with gzip.open(os.path.join(ROOT, "tests", "golden", "streams", f"{cfg}.json.gz"), "rt") as fh:
        data = json.load(fh)
    return ComputeDAG.from_json(data["dag"]), [history_from_json(h) for h in data["histories"]]


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


def cpu_reference(histories, dag, seconds: float, cores: int, fn=None) -> dict:
    """The reference's CPU runner restated (oracle/machine.py) on a fixed sample
    of stream candidates, one per host core, all in flight at once.  Rate =
    cores x candidates / sum of their core-seconds.  A candidate still running
    after `seconds` (the reference's heavy tail: one twin interpretation can take
    minutes) is stopped and counted with the time it used, a lower bound on its
    cost, so the rate is an optimistic bound for the reference."""
    from concurrent.futures import ProcessPoolExecutor, wait
    from paper_2006_06762_b200.state import history_to_json
    items = [(json.dumps(dag.to_json()), history_to_json(h)) for h in histories[:cores]]
    ex = ProcessPoolExecutor(max_workers=cores)
    for f in [ex.submit(int, 0) for _ in range(cores)]:      # workers up before the clock
        f.result()
    t0 = time.perf_counter()
    futs = [ex.submit(fn or _cpu_one, it) for it in items]
    done, pending = wait(futs, timeout=seconds)
    now = time.perf_counter()
    core_s = sum(f.result()[1] for f in done) + (now - t0) * len(pending)
    procs = list(getattr(ex, "_processes", {}).values())
    ex.shutdown(wait=False, cancel_futures=True)
    for pr in procs:              # stopped stragglers must not slow the next sample
        if pr.is_alive():
            pr.terminate()
    n = len(futs)
    return {"value": cores * n / core_s if core_s > 0 else 0.0, "candidates": n, "seconds": now - t0,
            "core_seconds": core_s, "truncated": len(pending)}


def _cpu_one(item):
    sys.path.insert(0, ROOT)
    t0 = time.perf_counter()
    from oracle import machine as OM
    from paper_2006_06762_b200.state import ComputeDAG, history_from_json, replay
    dag_json, hist = item
    p = replay(ComputeDAG.from_json(json.loads(dag_json)), history_from_json(hist))
    return OM.measure_batch([p])[0].status, time.perf_counter() - t0


def _cpu_full(item):
    """The reference's only full-size execution of a State: `interpret` on the
    real inputs (oracle/interp.py, src/interp.py:318-352) — what the B200 runner
    does for every candidate (run + verify against the state-free result)."""
    sys.path.insert(0, ROOT)
    t0 = time.perf_counter()
    import numpy as np
    from oracle import interp as OI
    from paper_2006_06762_b200.state import ComputeDAG, history_from_json, replay
    dag_json, hist = item
    dag = ComputeDAG.from_json(json.loads(dag_json))
    p = replay(dag, history_from_json(hist))
    OI.interpret(p, OI.random_inputs(dag, np.random.default_rng(0)))
    return "valid", time.perf_counter() - t0


def scoring_bench(runner_dev: int, programs: list, reps: int = 20) -> dict:
    """Population scoring (features + trees) over a synthetic population of 2^16
    programs (replicated stream States): device-resident kernel times and the
    host e2e rate."""
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
    dev = torch.device("cuda", runner_dev)
    d_words = torch.from_numpy(words).to(dev)
    d_soff = torch.from_numpy(stmt_off).to(dev)
    d_poff = torch.from_numpy(prog_off).to(dev)
    d_rows = torch.empty((n_stmt, 164), dtype=torch.float64, device=dev)
    d_rs = torch.empty(n_stmt, dtype=torch.float64, device=dev)
    d_sc = torch.empty(n_prog, dtype=torch.float64, device=dev)
    d_err = torch.zeros(1, dtype=torch.int32, device=dev)
    h = model.handle()
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    def feats():
        rt.check(lib.lt_features_device_cm(d_words.data_ptr(), d_soff.data_ptr(), n_stmt, d_rows.data_ptr(),
                                        d_err.data_ptr(), sp), "features")

    def trees():
        rt.check(lib.lt_predict_cols_device(h, d_rows.data_ptr(), n_stmt, d_rs.data_ptr(), sp), "trees")
        rt.check(lib.lt_segment_sum_device(d_rs.data_ptr(), d_poff.data_ptr(), n_prog, d_sc.data_ptr(), sp), "sum")

    out = {}
    for name, fn in (("features", feats), ("trees", trees)):
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
    # host e2e: encode + H2D + fused scoring + D2H through the public API
    t0 = time.perf_counter()
    sc = model.predict_batch(programs * n_rep)
    out["e2e_s"] = time.perf_counter() - t0
    out.update(n_prog=n_prog, n_stmt=n_stmt, words_bytes=int(words.nbytes), scores_finite=bool(np.isfinite(sc).all()))
    return out


def traffic_of(sha1: str):
    """DRAM bytes per launch of a profiled candidate (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            hit = json.load(fh).get(sha1)
        return hit["dram_bytes_per_launch"] if hit else None
    except (OSError, ValueError, KeyError):
        return None


def train_bench(n_prog: int = 1500) -> dict:
    """GBDT training: `gbdt.train` (trees fitted on the
    B200) vs the CPU restatement of the reference's `train` (oracle/train.py,
    pinned to reference-trained golden models) on the same records: stream
    States of the four configs, labels U(0.05, 1), default hyper (30 trees,
    depth 6).  Models must be identical."""
    import numpy as np
    from oracle import train as OT
    from paper_2006_06762_b200 import gbdt
    from paper_2006_06762_b200.features import extract_features_batch
    from paper_2006_06762_b200.model import Hyper
    from paper_2006_06762_b200.state import replay

    class Rec:
        def __init__(self, f, y):
            self.feats, self.y, self.dag_id = f, float(y), "d"
    feats = []
    for cfg in ("RC", "G10", "CL", "TBG"):
        dag, stream = load_stream(cfg)
        feats += extract_features_batch([replay(dag, h) for h in stream[:n_prog // 4]])
    y = np.random.default_rng(0).uniform(0.05, 1.0, len(feats))
    gbdt.train([Rec(f, v) for f, v in zip(feats[:50], y[:50])], Hyper(trees=2))       # warm-up
    t0 = time.perf_counter()
    got = gbdt.train([Rec(f, v) for f, v in zip(feats, y)], Hyper()).to_json()
    gpu_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    want = OT.train(feats, y)
    cpu_s = time.perf_counter() - t0
    want.pop("train_losses")
    return {"programs": len(feats), "rows": int(sum(len(f) for f in feats)), "trees": 30, "depth": 6,
            "gpu_s": gpu_s, "cpu_s": cpu_s, "speedup": cpu_s / gpu_s, "identical": got == want,
            "cpu_kind": "port (oracle/train.py, 1 core)"}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="RC", choices=sorted(FLOPS))
    ap.add_argument("--batch", type=int, default=32, help="candidates per rank per step")
    ap.add_argument("--cpu-seconds", type=float, default=30.0,
                    help="per-sample cap on a reference candidate's CPU time (truncated ones count their time)")
    ap.add_argument("--no-scoring", action="store_true")
    ap.add_argument("--compile-workers", type=int, default=0, help="ptxas worker processes per rank (0: auto)")
    ap.add_argument("--lower-workers", type=int, default=0, help="lowering processes per rank (0: auto)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dag, stream = load_stream(args.config)
    cores = os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return
        per_step = []
        for s in range(args.warmup + args.steps):
            sample = stream[s * cores:(s + 1) * cores]
            r = cpu_reference(sample, dag, args.cpu_seconds, cores)
            if s >= args.warmup:
                per_step.append(r)
        tot_c = sum(r["candidates"] for r in per_step)
        tot_s = sum(r["seconds"] for r in per_step)
        v = cores * tot_c / sum(r["core_seconds"] for r in per_step)
        print(json.dumps({
            "impl": "reference", "metric": f"measured candidates/sec ({args.config}, SSSRRSRS)", "value": v,
            "unit": "cand/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * tot_s / len(per_step), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": NAMES[args.config], "stream": f"tests/golden/streams/{args.config}.json.gz"},
            "cpu_baseline": {"value": v, "unit": "cand/s", "cores": cores, "kind": "port",
                             "sample": f"{tot_c} stream States, one per core per step; oracle/machine.py "
                                       "measure_batch (validate + twin interpret + machine_cost); "
                                       f"{sum(r['truncated'] for r in per_step)} capped at "
                                       f"{args.cpu_seconds:g} s and counted with that time (optimistic)"},
            "e2e": {"value": v, "unit": "cand/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200 import runtime as rt
    from paper_2006_06762_b200.dist import measure_batch_sharded as sharded_measure
    from paper_2006_06762_b200.state import replay

    workers = max(1, cores // world - (1 if world == 1 else 0))
    cache = tempfile.mkdtemp(prefix="lt_cubin_")     # empty: every candidate really compiles
    if args.compile_workers:
        workers = args.compile_workers
    runner = measure.configure(device=local, workers=workers, cache_dir=cache,
                               lower_workers=args.lower_workers or max(1, min(8, cores // (2 * world))))
    runner.context(dag, 0)                             # inputs + fp64 ground truth resident

    B = args.batch
    need = (args.warmup + args.steps) * B * world
    if need > len(stream):
        raise SystemExit(f"stream has {len(stream)} States, run needs {need}")

    def batch(step: int):
        """The whole step's batch (B per rank); each rank measures its own shard."""
        lo = step * world * B
        return [replay(dag, h) for h in stream[lo:lo + world * B]]

    def sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    all_recs = []
    launch_log = []
    refresh_s = []

    l2_flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")     # 256 MB > 126 MB L2

    def run_steps(first: int, n: int, fresh_ctx: bool) -> float:
        """Time n steps with CUDA events on the current stream; max over ranks."""
        progs = [batch(first + s) for s in range(n)]
        sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for ps in progs:
            l2_flush.zero_()                   # 256 MB write: no step starts with a warm L2
            if fresh_ctx:   # e2e: inputs re-uploaded and ground truth recomputed inside the region
                t_r = time.perf_counter()
                for c in runner.ctx.values():
                    c.refresh()
                refresh_s.append(time.perf_counter() - t_r)
            res = sharded_measure(ps)          # NCCL all_gather of (status, cost) records
            all_recs.append(res)
            launch_log.append(list(runner.last_records))
        e1.record()
        sync()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    run_steps(0, args.warmup, False)                               # warm-up (NVRTC workers, clocks)
    runner.stats.update({k: 0 if isinstance(v, int) else 0.0 for k, v in runner.stats.items()})
    with Clocks(local) as clk:
        ms = run_steps(args.warmup, args.steps, False)
    stats = dict(runner.stats)
    timed = all_recs[-args.steps:]
    io0 = dict(runner.io)
    timed_records = [r for step in launch_log[-args.steps:] for r in step]
    # our kernels launched in the timed region: per measured candidate, its kernels x
    # (warm-up + repeats), plus one NaN-poison and one verification launch per output
    n_launch = sum(len(r.info.get("kernels", [])) * (1 + r.repeats) + 2 * r.n_outputs
                   for r in timed_records if r.n_outputs)
    io1 = dict(runner.io)
    # e2e re-measures the timed steps' own States from scratch (modules dropped,
    # compile pool restarted on an empty cubin cache), so value and e2e differ only
    # by the end-to-end work
    runner.forget_compiled(tempfile.mkdtemp(prefix="lt_cubin_e2e_"))
    e2e_ms = run_steps(args.warmup, args.steps, True)
    io2 = dict(runner.io)
    h2d_step = (io2["h2d"] - io1["h2d"]) / args.steps
    d2h_step = (io2["d2h"] - io1["d2h"]) / args.steps

    # every rank already holds the gathered, input-ordered results of each step
    n_total = sum(len(rs) for rs in timed)
    n_valid = sum(r.status == "valid" for rs in timed for r in rs)
    costs = [r.cost for rs in timed for r in rs if r.status == "valid"]
    best_us = min(costs) if costs else float("nan")
    best_rec = min((r for r in timed_records if r.status == "valid"), key=lambda r: r.cost_us, default=None)
    value = n_total / (ms / 1000.0)
    e2e = (args.steps * B * world) / (e2e_ms / 1000.0)
    if world > 1:   # launches of all ranks
        t = torch.tensor([n_launch], device="cuda")
        dist.all_reduce(t)
        n_launch = int(t.item())

    if rank == 0:
        lib = rt.load()
        import ctypes
        tf, pms = ctypes.c_double(), ctypes.c_double()
        rt.check(lib.lt_ffma_peak(local, ctypes.byref(tf), ctypes.byref(pms)), "ffma peak")
        peak = tf.value
        achieved = FLOPS[args.config] / (best_us * 1e-6) / 1e12 if math.isfinite(best_us) else None
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except (OSError, ValueError):
            pass
        line = {
            "metric": f"measured candidates/sec ({args.config}, SSSRRSRS, compile+run+verify)",
            "value": value, "unit": "cand/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": NAMES[args.config], "candidates_per_rank_per_step": B,
                       "stream": f"tests/golden/streams/{args.config}.json.gz (reference sampler, legal launches)",
                       "compile_workers_per_rank": workers, "cubin_cache": "empty at start",
                       "l2": "flushed before every timed step (256 MB write); a candidate's cost is the "
                             "mean of back-to-back repeats after its warm-up run (TVM time_evaluator semantics)"},
            "valid": n_valid, "measured": n_total,
            "best_program": {"us": best_us, "tflops": achieved, "flop": FLOPS[args.config],
                             "source_sha1": best_rec.key if best_rec else None,
                             "kernels": (best_rec.info.get("kernels") if best_rec else None)},
            "compile": {"compiled": stats["compiled"], "cache_hits": stats["cache_hits"],
                        "recompiled_O1": stats.get("recompiled", 0),
                        "kernels_compiled": stats.get("kernels_compiled", 0),
                        "kernels_shared": stats.get("kernels_shared", 0),
                        "mean_s": stats["compile_s"] / max(1, stats["compiled"])},
            "pipeline_s": {k: round(stats[k], 3) for k in ("wall_s", "lower_s", "gpu_s", "load_s", "idle_s")},
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": traffic_of(best_rec.key if best_rec else ""),
                         "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the best "
                                         "candidate (ncu --set full, profiles/traffic.json by source sha1; "
                                         "null when this run's best was not profiled)",
                         "kernel": "best candidate of the timed steps (cost = mean of CUDA-event repeats)",
                         "peak_source": "lt_ffma_peak: FFMA issue-bound microbenchmark on this GPU"},
            "e2e": {"value": e2e, "unit": "cand/s", "h2d_bytes_per_step": int(h2d_step),
                    "d2h_bytes_per_step": int(d2h_step),
                    "refresh_ms_per_step": 1e3 * sum(refresh_s) / max(1, len(refresh_s)),
                    "ms_per_step": e2e_ms / args.steps,
                    "note": "measure_batch on host Programs; every step re-uploads the DAG's input tensors "
                            "(fp32+fp64, pageable) and recomputes the fp64 ground truth on the device; cubins "
                            "H2D; per-candidate error words D2H"},
            "gpu_launches": n_launch,
        }
        line["clocks"] = clk.summary()
        if not args.no_scoring:
            line["train"] = train_bench()
            progs = [replay(dag, h) for h in stream[:256]]
            sb = scoring_bench(local, progs)
            rows_bytes = sb["n_stmt"] * 164 * 8
            fbytes = sb["words_bytes"] + rows_bytes
            hbm = peaks.get("hbm_gbs")
            line["scoring"] = {
                "programs": sb["n_prog"], "statements": sb["n_stmt"],
                "device_programs_per_s": sb["n_prog"] / ((sb["features_ms"] + sb["trees_ms"]) / 1000),
                "e2e_programs_per_s": sb["n_prog"] / sb["e2e_s"],
                "features_ms": sb["features_ms"], "trees_ms": sb["trees_ms"],
                "roofline_features": {"bound": "hbm", "achieved": fbytes / (sb["features_ms"] / 1000) / 1e9,
                                      "peak": hbm, "unit": "GB/s",
                                      "frac": (fbytes / (sb["features_ms"] / 1000) / 1e9) / hbm if hbm else None,
                                      "traffic": None, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}}
        # CPU baseline: the reference's runner restated, bounded sample, all host cores
        cb = cpu_reference(stream[-cores:], dag, args.cpu_seconds, cores)
        cf = cpu_reference(stream[-cores:], dag, args.cpu_seconds, cores, fn=_cpu_full)
        line["cpu_full_execution"] = {
            "value": cf["value"], "unit": "cand/s", "cores": cores, "kind": "port",
            "sample": f"{cf['candidates']} stream States (one per core): full-size `interpret` "
                      f"(oracle/interp.py), {cf['truncated']} capped at {args.cpu_seconds:g} s and counted with "
                      "that time (an upper bound on the reference's rate of really executing candidates)"}
        line["cpu_baseline"] = {"value": cb["value"], "unit": "cand/s", "cores": cores, "kind": "port",
                                "sample": f"{cb['candidates']} stream States (one per core) through "
                                          "oracle/machine.py measure_batch (validate + twin interpret + "
                                          f"machine_cost); {cb['truncated']} capped at {args.cpu_seconds:g} s "
                                          "and counted with that time (optimistic)"}
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
