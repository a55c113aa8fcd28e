"""Tuning-log replay with wall-clock costs.

The reference's `replay` command (`src/cli.py:258-281`) re-measures every
logged program and demands the exact logged cost: right for its deterministic
analytical machine, impossible for measured device time.  `replay_log` keeps
its contract where it still holds and relaxes it where it cannot:

* the log is read by the reference's own reader (`loomtune.logio.iter_records`,
  `src/logio.py:61-88`): NDJSON,
  every record stamped with schema version 1, a truncated or corrupt line or a
  foreign schema raises `LogError` naming the line; the header builds the DAGs
  (`src/cli.py:199-206`);
* every measurement record is replayed (`src/ir.py` histories) and re-measured on
  the B200 through `measure.measure_batch` (outputs verified on the device
  against the fp64 ground truth), grouped per task;
* status parity is exact; a logged cost is compared within `rtol` when the log
  was written by a B200 run (its header carries a `runner` block with
  `cost_unit` "us", see `runner_header`), and ignored for analytical-machine
  logs (different units);
* every replayed record reports the device and the measured µs.

`cmd_replay(args)` is the drop-in for `loomtune.cli.cmd_replay` (`args.log`,
optional `args.rtol`), printing the reference's summary lines.
"""

from __future__ import annotations

import json
import math

from .reference import loomtune  # noqa: F401

from loomtune.logio import SCHEMA_VERSION, LogError, iter_records  # noqa: E402,F401  (the reference's reader)


def load_log(path: str):
    """(header, records, {task name: DAG}) as `_load_log` (src/cli.py:199-206)."""
    from .state import build
    records = list(iter_records(path))
    if not records or records[0].get("kind") != "header":
        raise LogError("log has no header record")
    header = records[0]
    dags = {t["name"]: build(t["workload"], **t["params"]) for t in header["tasks"]}
    return header, records, dags


def runner_header() -> dict:
    """The `runner` block a B200 run adds to its log header."""
    from .measure import GPU_TOL, get_runner
    r = get_runner()
    name = "cuda:%d" % r.device
    try:
        import torch
        name = torch.cuda.get_device_name(r.device)
    except Exception:   # torch is plumbing only; the device index still identifies it
        pass
    return {"backend": r.backend, "device": name, "cost_unit": "us", "min_ms": r.min_ms,
            "check_tol": GPU_TOL}


def replay_log(path: str, rtol: float = 0.25, measure_batch=None) -> dict:
    """Re-measure every logged program; returns a summary with per-record rows."""
    from .measure import MeasureLimits
    from .measure import measure_batch as mb
    from .state import history_from_json, replay
    measure_batch = measure_batch or mb
    header, records, dags = load_log(path)
    runner = header.get("runner") or {}
    timed_log = runner.get("cost_unit") == "us"
    lim = header.get("limits") or {}
    limits = MeasureLimits(**{k: v for k, v in lim.items() if k in MeasureLimits.__dataclass_fields__})
    meas = [r for r in records if r.get("kind") == "measure"]
    by_task: dict = {}
    for i, rec in enumerate(meas):
        by_task.setdefault(rec["task"], []).append(i)
    results = [None] * len(meas)
    for task, idx in by_task.items():
        progs = [replay(dags[task], history_from_json(meas[i]["history"])) for i in idx]
        for i, res in zip(idx, measure_batch(progs, None, limits)):
            results[i] = res
    rows, status_bad, cost_bad = [], 0, 0
    for rec, res in zip(meas, results):
        logged = rec.get("cost")
        status_ok = res.status == rec["status"]
        cost_ok = True
        if timed_log and status_ok and res.status == "valid" and logged is not None:
            cost_ok = abs(res.cost - logged) <= rtol * logged
        status_bad += not status_ok
        cost_bad += status_ok and not cost_ok
        rows.append({"iteration": rec.get("iteration"), "task": rec["task"], "logged_status": rec["status"],
                     "status": res.status, "logged_cost": logged,
                     "cost_us": res.cost if math.isfinite(res.cost) else None,
                     "status_ok": status_ok, "cost_ok": cost_ok})
    return {"log": path, "checked": len(meas), "status_mismatches": status_bad, "cost_outliers": cost_bad,
            "timed_log": timed_log, "rtol": rtol, "device": runner_header()["device"], "records": rows}


def cmd_replay(args) -> int:
    """Drop-in for `cmd_replay` (src/cli.py:258-281)."""
    summary = replay_log(args.log, getattr(args, "rtol", 0.25) or 0.25)
    for row in summary["records"]:
        if not (row["status_ok"] and row["cost_ok"]):
            print(f"mismatch at iteration {row['iteration']} task {row['task']}: "
                  f"logged cost={row['logged_cost']} status={row['logged_status']}, "
                  f"measured cost={row['cost_us']} status={row['status']}")
    bad = summary["status_mismatches"] + summary["cost_outliers"]
    if bad:
        print(f"replayed {summary['checked']} measurements: {bad} mismatches")
        return 1
    print(f"replayed {summary['checked']} measurements on {summary['device']}: clean")
    return 0
