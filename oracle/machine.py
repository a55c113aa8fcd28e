"""ORACLE (test infrastructure only): CPU restatement of the reference's
measurement harness, `measure_batch` (`src/machine.py:249-285`) with its
analytical `machine_cost` (`src/machine.py:59-105`) and the shrunken-twin
`spot_check` (`shrink_dag`, `remap_history`, `_check_outputs`,
`src/machine.py:113-233`).

This is what `bench.py --impl reference` times as the reference's CPU runner,
and the State-exact checker of the GPU runner in tests.  State replay uses the
package's IR mirror (`paper_2006_06762_b200.state`), itself pinned to the
reference by tests/test_host.py; constant re-packing for the twin restates
`rewrite_constant_layout` (`src/annotate.py:227-300`).  Pinned against the
reference by `tests/golden/measure.json` (statuses, details, exact costs).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from oracle import features as OF
from oracle import interp as OI
from paper_2006_06762_b200 import state as IR
from paper_2006_06762_b200.state import ComputeDAG

VALID, INVALID, TIMEOUT = "valid", "invalid", "timeout"
FULL_CHECK_VOLUME = 1 << 25


@dataclass(frozen=True)
class MachineSpec:
    cores: int = 8
    vector_lanes: int = 8
    miss_penalty: float = 8.0
    loop_overhead: float = 0.5
    cache_bytes: int = 32 * 1024


@dataclass(frozen=True)
class MeasureResult:
    cost: float
    throughput: float
    status: str
    detail: str = ""


def statement_cost(st: dict, spec: MachineSpec) -> float:
    nest, own_start = st["nest"], st["own_start"]
    own = nest[own_start:]
    lanes = spec.vector_lanes if own and own[-1].annotation == "vectorize" and own[-1].lin_stride == 1 else 1
    threads = 1
    for l in nest:
        if l.annotation == "parallel":
            threads = min(l.extent, spec.cores)
            break
    compute = st["ops_total"] * st["total"] / (lanes * threads)
    missed = 0.0
    for a in st["accesses"]:
        lines = a["unique_lines"]
        for pos, l in enumerate(nest):
            if l.id in a["present"] or l.extent <= 1:
                continue
            if st["ws"][pos] > spec.cache_bytes:
                lines *= l.extent
        missed += lines
    memory = missed * spec.miss_penalty / threads
    boundary, prod = len(nest), 1
    for i in range(len(nest) - 1, own_start - 1, -1):
        if prod * nest[i].extent > st["unroll"]:
            break
        prod *= nest[i].extent
        boundary = i
    overhead, cum = 0.0, 1.0
    for i, l in enumerate(nest):
        cum *= l.extent
        if i < boundary:
            overhead += cum
    return compute + memory + overhead * spec.loop_overhead


def machine_cost(p, spec: MachineSpec = MachineSpec()) -> float:
    return sum(statement_cost(st, spec) for st in OF.analyze(p, with_present=True))


# ---- twin construction ---------------------------------------------------------

def prime_factors(n: int) -> list:
    out, d = [], 2
    while d * d <= n:
        while n % d == 0:
            out.append(d)
            n //= d
        d += 1 if d == 2 else 2
    if n > 1:
        out.append(n)
    return out


def shrink_dag(dag, cap: int = 8):
    need: dict = {}
    sized: dict = {}
    for name in OI._topo(dag):
        node = dag.node(name)
        if node.is_placeholder:
            req = need.get(name)
            sized[name] = replace(node, space=tuple((it, req[d] if req else min(e, cap))
                                                    for d, (it, e) in enumerate(node.space)))
            continue
        req = need.get(name, [1] * len(node.space))
        space = tuple((it, max(min(e, cap), req[d])) for d, (it, e) in enumerate(node.space))
        red = tuple((it, min(e, cap)) for it, e in node.reduce)
        sized[name] = replace(node, space=space, reduce=red)
        rng = {it: (0, e - 1) for it, e in (*space, *red)}
        for r in OI._reads(node.body):
            cur = need.setdefault(r.buffer, [1] * len(r.index))
            for d, lin in enumerate(r.index):
                cur[d] = max(cur[d], lin.interval(rng)[1] + 1)
    return ComputeDAG(tuple(sized[n.name] for n in dag.nodes))


def _packing_descriptor(s, buffer, dims):
    rs = [r for r in OI._reads(s.expr) if r.buffer == buffer]
    if len(rs) != 1:
        return None
    dmap = dict(s.index_map)
    fns = []
    for lin in rs[0].index:
        ast = IR.lin_to_decode(lin, dmap)
        vars_ = IR.d_vars(ast)

        def fn(lid, v, ast=ast, vars_=vars_):
            env = {x: 0 for x in vars_}
            if lid in env:
                env[lid] = v
            return IR.d_eval(ast, env)
        fns.append(fn)
    entries = []
    for l in s.loops:
        if l.extent is None:
            return None
        if l.extent <= 1:
            continue
        touch = None
        for d, fn in enumerate(fns):
            lo, hi, far = fn(l.id, 0), fn(l.id, 1), fn(l.id, l.extent - 1)
            if hi == lo and far == lo:
                continue
            stride = hi - lo
            if far - lo != stride * (l.extent - 1) or stride <= 0 or touch is not None:
                return None
            touch = (d, l.extent, stride)
        if touch is not None:
            entries.append(touch)
    per: dict = {}
    for d, e, st in entries:
        per.setdefault(d, []).append((e, st))
    for d, size in enumerate(dims):
        parts = per.get(d, [])
        tot = 1
        for e, _ in parts:
            tot *= e
        if tot != size:
            return None
        expect = size
        for e, st in parts:
            expect //= e
            if st != expect:
                return None
    return tuple((d, e) for d, e, _ in entries)


def rewrite_constant_layout(p):
    for node in p.dag.nodes:
        if not (node.is_placeholder and node.is_constant):
            continue
        readers = [s for s in p.stages if not s.inlined and s.expr is not None
                   and any(r.buffer == node.name for r in OI._reads(s.expr))]
        if len(readers) != 1:
            continue
        dims = node.shape
        desc = _packing_descriptor(readers[0], node.name, dims)
        if desc is None:
            continue
        if tuple(d for d, _ in desc) == tuple(range(len(dims))) and all(e == dims[d] for d, e in desc):
            continue
        p = IR.apply_step(p, IR.LayoutRewrite(node.name, desc))
    return p


def remap_history(history, dag):
    p = IR.naive_program(dag)
    done = False
    for st in history:
        k = type(st).__name__
        if k == "Split":
            ext = p.stage(st.stage).loop(st.loop).extent
            parts = [1] * (len(st.inner) + 1)
            for i, f in enumerate(prime_factors(ext)):
                parts[i % len(parts)] *= f
            st = IR.Split(st.stage, st.loop, tuple(parts[1:]))
        elif k == "Rfactor":
            ext = p.stage(st.stage).loop(st.loop).extent
            st = IR.Rfactor(st.stage, st.loop, math.gcd(st.factor or 1, ext))
        elif k == "LayoutRewrite":
            if not done:
                p = rewrite_constant_layout(p)
                done = True
            continue
        p = IR.apply_step(p, st)
    return p


def _volume(dag) -> int:
    tot = 0
    for n in dag.nodes:
        if n.is_placeholder:
            continue
        v = 1
        for _, e in (*n.space, *n.reduce):
            v *= e
        tot += v
    return tot


def check_outputs(p, dag, tol, seed):
    inputs = OI.random_inputs(dag, np.random.default_rng(seed))
    try:
        got = OI.interpret(p, inputs)
    except OI.InterpreterError as e:
        return str(e)
    for name, ref in OI.reference_outputs(dag, inputs).items():
        err = float(np.max(np.abs(got[name] - ref) / np.maximum(np.abs(ref), 1e-30)))
        if not np.isfinite(err) or err > tol:
            return f"output {name} differs from reference (max rel err {err:.3g})"
    return None


def spot_check(p, cap=8, tol=1e-5, seed=0):
    twin_dag = shrink_dag(p.dag, cap)
    try:
        twin = remap_history(p.history, twin_dag)
    except IR.IRError:
        if _volume(p.dag) <= FULL_CHECK_VOLUME:
            bad = IR.validate(p)
            if bad:
                return f"fails validation: {bad[0]}"
            return check_outputs(p, p.dag, tol, seed)
        return None
    bad = IR.validate(twin)
    if bad:
        return f"twin fails validation: {bad[0]}"
    return check_outputs(twin, twin_dag, tol, seed)


def measure_batch(programs, spec=MachineSpec(), cost_ceiling=None, check_cap=8, check_tol=1e-5,
                  check_seed=0, best_cost=None):
    results, costs = [], []
    for p in programs:
        bad = IR.validate(p)
        if bad:
            results.append(MeasureResult(math.inf, 0.0, INVALID, bad[0]))
            costs.append(None)
            continue
        err = spot_check(p, check_cap, check_tol, check_seed)
        if err is not None:
            results.append(MeasureResult(math.inf, 0.0, INVALID, err))
            costs.append(None)
            continue
        c = machine_cost(p, spec)
        if cost_ceiling is not None and c >= cost_ceiling:
            results.append(MeasureResult(c, 0.0, TIMEOUT))
            costs.append(None)
            continue
        results.append(MeasureResult(c, 0.0, VALID))
        costs.append(c)
    valid = [c for c in costs if c is not None] + ([best_cost] if best_cost is not None else [])
    if not valid:
        return results
    best = min(valid)
    return [replace(r, throughput=best / c) if c is not None else r for r, c in zip(results, costs)]
