"""Tuning-log replay: the reference's log format and
damage checks (src/logio.py:60-86) on CPU; re-measurement on the B200 (gpu)."""

import json

import pytest


def _write(path, lines):
    with open(path, "w") as fh:
        for ln in lines:
            fh.write(ln + "\n")


def _header(tasks, runner=None):
    h = {"kind": "header", "schema": 1, "seed": 0, "objective": "total-latency", "budget": 1,
         "structure": "SSSRRSRS", "tasks": tasks, "machine": {}, "limits": {}, "training": {}, "params": {}}
    if runner:
        h["runner"] = runner
    return json.dumps(h, sort_keys=True)


TASK = {"name": "mm", "workload": "matmul", "params": {"n": 64, "m": 64, "k": 64}, "weight": 1, "dnn": "net"}


def test_log_damage_is_reported_with_line_numbers(tmp_path):
    from paper_2006_06762_b200.replay import LogError, iter_records, load_log
    p = tmp_path / "a.ndjson"
    _write(p, [_header([TASK]), "{not json"])
    with pytest.raises(LogError, match="line 2"):
        list(iter_records(str(p)))
    p.write_text(_header([TASK]) + "\n" + json.dumps({"kind": "measure", "schema": 1}))   # no trailing newline
    with pytest.raises(LogError, match="truncated"):
        list(iter_records(str(p)))
    _write(p, [json.dumps({"kind": "header", "schema": 2})])
    with pytest.raises(LogError, match="schema version 2"):
        list(iter_records(str(p)))
    _write(p, [json.dumps({"kind": "measure", "schema": 1})])
    with pytest.raises(LogError, match="no header"):
        load_log(str(p))
    _write(p, [_header([TASK])])
    header, records, dags = load_log(str(p))
    assert list(dags) == ["mm"] and dags["mm"].node("C").shape == (64, 64)


@pytest.mark.gpu
def test_replay_remeasures_on_the_b200(tmp_path):
    """A B200-timed log replays clean; a wrong status or a far-off cost is flagged."""
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200.replay import replay_log
    from paper_2006_06762_b200.state import Reorder, SetPragma, Split, apply_step, build, history_to_json, \
        naive_program
    measure.configure(device=0, cache_dir="")
    dag = build("matmul", n=64, m=64, k=64)
    naive = naive_program(dag)
    tiled = naive
    for st in (Split("C", "i", (2, 4, 2, 1)), Split("C", "j", (1, 8, 2, 2)), Split("C", "k", (4, 4)),
               Reorder("C", ("i.0", "j.0", "i.1", "j.1", "i.2", "j.2", "k.0", "k.1", "i.3", "j.3", "k.2",
                             "i.4", "j.4")), SetPragma("C", 512)):
        tiled = apply_step(tiled, st)
    res = measure.measure_batch([naive, tiled])
    rec = lambda p, r, it, **kw: json.dumps({"kind": "measure", "schema": 1, "seed": 0, "iteration": it,  # noqa
                                            "task": "mm", "history": history_to_json(p.history),
                                            "cost": r.cost, "status": r.status, **kw}, sort_keys=True)
    p = tmp_path / "b200.ndjson"
    runner = {"cost_unit": "us", "device": "B200", "backend": "ptx"}
    _write(p, [_header([TASK], runner), rec(naive, res[0], 0), rec(tiled, res[1], 1)])
    s = replay_log(str(p), rtol=0.5)
    assert s["checked"] == 2 and s["status_mismatches"] == 0 and s["cost_outliers"] == 0, s
    assert all(r["cost_us"] > 0 for r in s["records"])
    bad = json.loads(rec(tiled, res[1], 2))
    bad["cost"] = res[1].cost * 100
    _write(p, [_header([TASK], runner), json.dumps(bad, sort_keys=True)])
    assert replay_log(str(p), rtol=0.5)["cost_outliers"] == 1
    bad["status"] = "invalid"
    _write(p, [_header([TASK], runner), json.dumps(bad, sort_keys=True)])
    assert replay_log(str(p))["status_mismatches"] == 1
    measure._shutdown()
