"""§8(e) in the tune path: the reference's own `tune` with `integrate.install`
under a 2-rank gloo group shards every measurement batch and every evolution
population across the ranks (`dist.measure_batch_sharded`,
`dist.score_batch_sharded`) and gathers only records and fitness vectors.
With device-free stand-ins for the two device calls (the reference's
analytical `machine_cost` as the measured cost, the reference's
`CostModel.predict` as the score), the tune must be identical on both ranks
and identical to the single-process tune: same measured States in the same
order, same costs, same best program."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _stand_in():
    from loomtune.machine import machine_cost
    from loomtune.model import CostModel
    from paper_2006_06762_b200.measure import Record

    def measure_records(programs, seed):
        out = []
        for p in programs:
            r = Record(done=True)
            r.status, r.cost_us = "valid", float(machine_cost(p))
            out.append(r)
        return out

    def score(model, programs):
        ref = CostModel.from_json(model.to_json())
        return [ref.predict(p) for p in programs]
    return {"measure_records": measure_records, "score": score}


def _tune(sharded: bool):
    import loomtune as LT
    from loomtune.ir import history_to_json
    from paper_2006_06762_b200 import integrate
    dag = LT.build("matmul", n=32, m=32, k=16)
    task = LT.make_task("mm", dag)
    log = []

    def sink(rec):
        if rec.get("kind") == "measure":
            log.append((history_to_json(rec["history"]), rec["cost"], rec["status"]))
    orig = integrate.install(LT, gpu_train=False, sharded=sharded, stand_in=_stand_in())
    try:
        LT.tune([task], LT.Objective(), 3, LT.TuneSettings(batch_size=8), LT.SchedulerParams(), seed=0,
                log_sink=sink)
    finally:
        integrate.uninstall(LT, orig)
    return log, task.best_cost


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2006_06762_b200 import dist as D
        calls = {"measure": 0, "score": 0}
        m0, s0 = D.measure_batch_sharded, D.score_batch_sharded

        def m(*a, **k):
            calls["measure"] += 1
            return m0(*a, **k)

        def s(*a, **k):
            calls["score"] += 1
            return s0(*a, **k)
        D.measure_batch_sharded, D.score_batch_sharded = m, s
        log, best = _tune(sharded=True)
        q.put((rank, log, best, calls))
    finally:
        dist.destroy_process_group()


def test_sharded_tune_matches_single_process():
    from paper_2006_06762_b200.reference import loomtune  # noqa: F401
    want_log, want_best = _tune(sharded=False)
    assert len(want_log) > 16
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, log, best, calls in got:
        assert calls["measure"] > 0 and calls["score"] > 0, calls
        assert best == want_best
        assert log == want_log, rank
