"""Multi-GPU sharding of the hot path.

Measurement units and population members are independent, so each rank works
on its own contiguous shard with its own device and compile pool; the only
exchange is a gather of fixed-size results over `torch.distributed` (NCCL on
the GPU box, gloo in the CPU tests):

* `measure_batch_sharded` — every rank measures `programs[shard]`; the
  (status, cost, detail) records are all-gathered and every rank returns the
  full, input-ordered `MeasureResult` list, normalised exactly like
  `measure_batch` (so the tuner above sees no difference).
* `score_batch_sharded` — every rank scores its shard of the population on its
  GPU; the fitness vector is all-gathered (the model is identical on all ranks:
  it is trained from the gathered records).

No reductions: results are bit-identical to the single-GPU path.
"""

from __future__ import annotations

import math

import numpy as np


def shard_bounds(n: int, rank: int, world: int) -> tuple:
    """Contiguous, balanced shard [lo, hi) of n items for `rank`."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _world(group=None):
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1, None
    return dist.get_rank(group), dist.get_world_size(group), dist


def _gather_array(local: np.ndarray, n_total: int, rank: int, world: int, dist, group, device):
    """All-gather per-rank float64 rows (shards may differ by one row)."""
    import torch
    width = local.shape[1]
    rows = max(shard_bounds(n_total, r, world)[1] - shard_bounds(n_total, r, world)[0] for r in range(world))
    pad = np.zeros((rows, width), np.float64)
    pad[: len(local)] = local
    t = torch.from_numpy(pad).to(device)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t, group=group)
    out = []
    for r, b in enumerate(bufs):
        lo, hi = shard_bounds(n_total, r, world)
        out.append(b.cpu().numpy()[: hi - lo])
    return np.concatenate(out, axis=0)


def measure_batch_sharded(programs, spec=None, limits=None, best_cost=None, measure_records=None,
                          group=None, device=None, stage=None):
    """`measure_batch` over all ranks; `measure_records(programs, seed)` -> Records
    (defaults to this rank's GPU runner).  `stage`: the next batch, whose shard
    this rank's runner lowers and compiles behind the current one."""
    from .measure import MeasureLimits, Record, get_runner, normalise
    limits = limits if limits is not None else MeasureLimits()
    programs = list(programs)
    rank, world, dist = _world(group)
    seed = getattr(limits, "check_seed", 0)
    if measure_records is None:
        nxt = None
        if stage:
            s_lo, s_hi = shard_bounds(len(stage), rank, world)
            nxt = list(stage)[s_lo:s_hi]
        measure_records = lambda ps, s: get_runner().measure_programs(ps, seed=s, stage=nxt)  # noqa: E731
    lo, hi = shard_bounds(len(programs), rank, world)
    recs = measure_records(programs[lo:hi], seed)
    if world == 1:
        return normalise(recs, best_cost, getattr(limits, "cost_ceiling", None))
    local = np.asarray([[1.0 if r.status == "valid" else 0.0, r.cost_us if math.isfinite(r.cost_us) else -1.0]
                        for r in recs], np.float64).reshape(-1, 2)
    if device is None:
        import torch
        device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    table = _gather_array(local, len(programs), rank, world, dist, group, device)
    details = [None] * world
    dist.all_gather_object(details, [r.detail for r in recs], group=group)
    flat_details = [d for part in details for d in part]
    full = []
    for (ok, cost), det in zip(table, flat_details):
        rr = Record()
        if ok > 0:
            rr.status, rr.cost_us = "valid", float(cost)
        rr.detail = det
        full.append(rr)
    return normalise(full, best_cost, getattr(limits, "cost_ceiling", None))


def score_batch_sharded(model, programs, group=None, device=None, score_fn=None):
    """Population fitness over all ranks (one fused device pass per rank)."""
    programs = list(programs)
    rank, world, dist = _world(group)
    score_fn = score_fn or (lambda ps: model.predict_batch(ps))
    lo, hi = shard_bounds(len(programs), rank, world)
    local = np.asarray(score_fn(programs[lo:hi]), np.float64).reshape(-1, 1)
    if world == 1:
        return local[:, 0]
    if device is None:
        device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    return _gather_array(local, len(programs), rank, world, dist, group, device)[:, 0]
