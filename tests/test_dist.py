"""Multi-rank host logic of the sharded hot path, world_size 2 on gloo (CPU)."""

import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2006_06762_b200.dist import shard_bounds


def test_shard_bounds_cover_exactly():
    for n in range(0, 40):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _fake_records(programs, seed):
    """CPU stand-in for the GPU runner: deterministic cost per program id."""
    from paper_2006_06762_b200.measure import Record
    out = []
    for p in programs:
        r = Record()
        if p % 5 == 3:
            r.detail = f"gpu: illegal {p}"
        else:
            r.status, r.cost_us = "valid", 10.0 + (p * 7919 % 101)
        out.append(r)
    return out


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2006_06762_b200.dist import measure_batch_sharded, score_batch_sharded
        progs = list(range(n))
        res = measure_batch_sharded(progs, measure_records=_fake_records, best_cost=12.0)
        sc = score_batch_sharded(None, progs, score_fn=lambda ps: [float(p) * 0.5 for p in ps])
        q.put((rank, [(r.cost, r.throughput, r.status, r.detail) for r in res], list(sc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 16])
def test_sharded_measure_and_score_match_single_process(n):
    from paper_2006_06762_b200.measure import normalise
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    want = [(r.cost, r.throughput, r.status, r.detail)
            for r in normalise(_fake_records(list(range(n)), 0), best_cost=12.0)]
    for rank, res, sc in got:
        assert len(res) == n
        for a, b in zip(res, want):
            assert a[2] == b[2] and a[3] == b[3] and a[1] == b[1]
            assert (a[0] == b[0]) or (math.isinf(a[0]) and math.isinf(b[0]))
        assert sc == [p * 0.5 for p in range(n)]
