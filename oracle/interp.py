"""ORACLE (test infrastructure only): CPU restatement of the reference's State
interpreter and ground truth, `interpret` / `reference_outputs` /
`random_inputs` (`src/interp.py:38-352`) and scalar `evaluate`
(`src/expr.py:342-396`).

It executes a State the way the reference does — attached stages run inside
their host loop iterations, cache/rfactor buffers are real, packed constants are
materialised, reductions initialise at the first interpreted reduction loop,
everything below the deepest attach point (or a 4 Mi-element grid) is evaluated
vectorised in float64 — so it is both the State-exact parity oracle for the GPU
runner and the timed CPU runner (`bench.py --impl reference`).

Pinned against the reference: `tests/golden/outputs.npz` holds the reference's
`reference_outputs`; `tests/test_oracle.py` checks `reference_outputs` here
against it and `interpret` against `reference_outputs` on corpus States.
"""

from __future__ import annotations

import numpy as np

GRID_LIMIT = 1 << 22
IDENTITY = {"sum": 0.0, "max": -np.inf}


class InterpreterError(RuntimeError):
    pass


def _k(x) -> str:
    return type(x).__name__


# ---- scalar expression semantics -------------------------------------------

def lin_eval(lin, env):
    out = lin.const
    for n, c in lin.terms:
        out = out + c * env[n]
    return out


def evaluate(e, env, read, mask):
    k = _k(e)
    if k == "Const":
        return np.asarray(e.value, dtype=np.float64)
    if k == "IterVal":
        return np.asarray(lin_eval(e.lin, env), dtype=np.float64)
    if k == "Read":
        return read(e.buffer, tuple(np.asarray(lin_eval(l, env)) for l in e.index), mask)
    if k == "Bin":
        a = evaluate(e.lhs, env, read, mask)
        b = evaluate(e.rhs, env, read, mask)
        op = e.op
        if op in ("lt", "le", "gt", "ge", "eq"):
            f = {"lt": np.less, "le": np.less_equal, "gt": np.greater, "ge": np.greater_equal,
                 "eq": np.equal}[op]
            return f(a, b).astype(np.float64)
        return {"add": np.add, "sub": np.subtract, "mul": np.multiply, "div": np.divide,
                "max": np.maximum, "min": np.minimum}[op](a, b)
    if k == "Call":
        return {"exp": np.exp, "sqrt": np.sqrt, "log": np.log, "abs": np.abs}[e.fn](
            evaluate(e.arg, env, read, mask))
    if k == "Select":
        c = evaluate(e.cond, env, read, mask)
        take = np.broadcast_to(c != 0.0, np.broadcast_shapes(np.shape(c), mask.shape))
        t = evaluate(e.then, env, read, mask & take)
        o = evaluate(e.other, env, read, mask & ~take)
        return np.where(take, t, o)
    raise InterpreterError(f"cannot evaluate {k}")


def d_eval(d, env):
    k = _k(d)
    if k == "DVar":
        return env[d.loop]
    if k == "DConst":
        return d.value
    if k == "DAdd":
        return d_eval(d.a, env) + d_eval(d.b, env)
    a = d_eval(d.a, env)
    return a * d.c if k == "DMul" else (a // d.c if k == "DDiv" else a % d.c)


def d_interval(d, ranges):
    k = _k(d)
    if k == "DVar":
        return ranges[d.loop]
    if k == "DConst":
        return d.value, d.value
    if k == "DAdd":
        a, b = d_interval(d.a, ranges), d_interval(d.b, ranges)
        return a[0] + b[0], a[1] + b[1]
    lo, hi = d_interval(d.a, ranges)
    if k == "DMul":
        return (lo * d.c, hi * d.c) if d.c >= 0 else (hi * d.c, lo * d.c)
    if k == "DDiv":
        return lo // d.c, hi // d.c
    return (lo % d.c, hi % d.c) if lo // d.c == hi // d.c else (0, d.c - 1)


def lin_decode_interval(lin, dmap, ranges):
    """Interval of `lin_to_decode(lin, dmap)` without building the AST."""
    lo = hi = lin.const
    for n, c in lin.terms:
        a, b = d_interval(dmap[n], ranges) if n in dmap else ranges[n]
        lo, hi = (lo + a * c, hi + b * c) if c >= 0 else (lo + b * c, hi + a * c)
    return lo, hi


def _reads(e):
    out = []
    stack = [e]
    while stack:
        n = stack.pop()
        k = _k(n)
        if k == "Read":
            out.append(n)
        kids = ((n.lhs, n.rhs) if k == "Bin" else (n.arg,) if k == "Call" else
                (n.cond, n.then, n.other) if k == "Select" else (n.body,) if k == "Reduce" else ())
        stack.extend(reversed(kids))
    return out


# ---- inputs and ground truth -------------------------------------------------

def random_inputs(dag, rng) -> dict:
    return {n.name: rng.uniform(0.25, 1.0, size=n.shape) for n in dag.nodes if n.is_placeholder}


def _gather(buf, name, idx, mask, where):
    if len(idx) != buf.ndim:
        raise InterpreterError(f"{where}: read of {name} has rank {len(idx)}, buffer rank {buf.ndim}")
    shape = np.broadcast_shapes(mask.shape, *[np.shape(i) for i in idx])
    m = np.broadcast_to(mask, shape)
    safe = []
    for d, i in enumerate(idx):
        a = np.broadcast_to(np.asarray(i), shape)
        if (m & ((a < 0) | (a >= buf.shape[d]))).any():
            raise InterpreterError(f"{where}: read of {name} out of bounds on dim {d}")
        safe.append(np.where(m, a, 0))
    return buf[tuple(safe)]


def _topo(dag):
    cons = {n.name: set(dag.consumers_of(n.name)) for n in dag.nodes}
    out, done = [], set()
    while len(out) < len(dag.nodes):
        nxt = sorted(n for n, c in cons.items() if n not in done and c <= done)[0]
        out.append(nxt)
        done.add(nxt)
    return out


def reference_outputs(dag, inputs: dict, chunk: int = 1 << 22) -> dict:
    """State-free evaluation, chunked over the space domain so full BASELINE
    shapes fit in memory (the reference builds one space x reduce grid)."""
    bufs = dict(inputs)
    for name in reversed(_topo(dag)):
        node = dag.node(name)
        if node.is_placeholder:
            continue
        space, red = list(node.space), list(node.reduce)
        rvol = 1
        for _, e in red:
            rvol *= e
        body = node.body.body if _k(node.body) == "Reduce" else node.body
        out = np.empty(tuple(e for _, e in space), dtype=np.float64)
        flat = out.reshape(-1)
        npts = flat.size
        step = max(1, chunk // max(rvol, 1))
        rgrid = np.meshgrid(*[np.arange(e) for _, e in red], indexing="ij") if red else []
        for s0 in range(0, npts, step):
            pts = np.arange(s0, min(npts, s0 + step))
            coords = np.unravel_index(pts, out.shape) if space else ()
            env = {}
            for (n, _), c in zip(space, coords):
                env[n] = c.reshape((-1,) + (1,) * len(red))
            for (n, _), g in zip(red, rgrid):
                env[n] = g.reshape((1,) + g.shape)
            shape = (len(pts),) + tuple(e for _, e in red)
            mask = np.ones(shape, dtype=bool)
            vals = np.broadcast_to(np.asarray(evaluate(
                body, env, lambda b, i, m: _gather(bufs[b], b, i, m, "reference"), mask), dtype=np.float64), shape)
            if red:
                axes = tuple(range(1, 1 + len(red)))
                vals = np.add.reduce(vals, axis=axes) if node.body.op == "sum" else np.maximum.reduce(vals, axis=axes)
            flat[s0:s0 + len(pts)] = vals
        bufs[name] = out
    return {o: bufs[o] for o in dag.outputs}


# ---- State interpreter -------------------------------------------------------

def _pack_strides(desc):
    out = []
    for j, (d, _) in enumerate(desc):
        s = 1
        for d2, e2 in desc[j + 1:]:
            if d2 == d:
                s *= e2
        out.append(s)
    return out


def pack_buffer(buf, desc):
    st = _pack_strides(desc)
    shape = tuple(e for _, e in desc)
    digits = np.indices(shape)
    logical = [np.zeros(shape, dtype=np.int64) for _ in range(buf.ndim)]
    for j, (d, _) in enumerate(desc):
        logical[d] = logical[d] + digits[j] * st[j]
    return buf[tuple(logical)]


def _attachment_case(stage, target):
    if any(r.buffer == stage.name for r in _reads(target.expr)):
        return "producer"
    if any(r.buffer == target.name for r in _reads(stage.expr)):
        return "consumer"
    raise InterpreterError(f"{stage.name} and {target.name} share no buffer edge")


class _Exec:
    def __init__(self, p, bufs, packed):
        self.p, self.bufs, self.packed = p, bufs, packed
        self.shapes = {s.name: tuple(e for _, e in s.space) for s in p.stages}

    def shape(self, name):
        return self.shapes.get(name) or self.p.dag.node(name).shape

    def reader(self, where):
        def read(b, idx, mask):
            if b in self.packed:
                phys, desc = self.packed[b]
                shape = np.broadcast_shapes(mask.shape, *[np.shape(i) for i in idx])
                m = np.broadcast_to(mask, shape)
                logical = self.shape(b)
                for d, i in enumerate(idx):
                    a = np.broadcast_to(np.asarray(i), shape)
                    if (m & ((a < 0) | (a >= logical[d]))).any():
                        raise InterpreterError(f"{where}: packed read of {b} out of bounds on dim {d}")
                st = _pack_strides(desc)
                pidx = [(np.where(m, np.broadcast_to(np.asarray(idx[d]), shape), 0) // st[j]) % e
                        for j, (d, e) in enumerate(desc)]
                return phys[tuple(pidx)]
            if b not in self.bufs:
                raise InterpreterError(f"{where}: read of unallocated buffer {b}")
            return _gather(self.bufs[b], b, idx, mask, where)
        return read

    def run_stage(self, s, offsets):
        children = {}
        for c in self.p.stages:
            if c.compute_at is not None and c.compute_at[0] == s.name:
                children.setdefault(c.compute_at[1], []).append(c)
        loops = s.loops
        deepest = max([i for i, l in enumerate(loops) if l.id in children], default=-1)
        vol = 1
        for l in loops:
            vol *= max(1, l.extent)
        prefix = deepest + 1
        while prefix < len(loops) and vol > GRID_LIMIT:
            vol //= max(1, loops[prefix].extent)
            prefix += 1
        init_at = None
        if any(l.kind == "reduce" for l in loops[:prefix]):
            init_at = next(i for i, l in enumerate(loops) if l.kind == "reduce")
        self._nest(s, offsets, children, prefix, init_at, 0, {})

    def _nest(self, s, offsets, children, prefix, init_at, i, env):
        if i == prefix:
            self._grid(s, offsets, s.loops[prefix:], env, init_at is not None)
            return
        if i == init_at:
            self._init(s, offsets, env)
        loop = s.loops[i]
        kids = children.get(loop.id, [])
        for v in range(loop.extent):
            env[loop.id] = v
            if kids:
                self._attach(kids, s, offsets, env, True)
            self._nest(s, offsets, children, prefix, init_at, i + 1, env)
            if kids:
                self._attach(kids, s, offsets, env, False)
        del env[loop.id]

    def _init(self, s, offsets, env):
        free = [l for l in s.loops if l.id not in env and l.kind != "reduce"]
        grids = np.meshgrid(*[np.arange(l.extent) for l in free], indexing="ij", sparse=True) if free else []
        genv = dict(env)
        genv.update({l.id: g for l, g in zip(free, grids)})
        dmap = dict(s.index_map)
        idx = tuple(np.asarray(d_eval(dmap[n], genv)) + offsets.get(n, 0) for n, _ in s.space)
        op = s.expr.op if _k(s.expr) == "Reduce" else "sum"
        self.bufs[s.name][idx] = IDENTITY[op]

    def _attach(self, kids, host, host_off, env, before):
        ranges = {l.id: ((env[l.id], env[l.id]) if l.id in env else (0, l.extent - 1)) for l in host.loops}
        hmap = dict(host.index_map)
        for c in kids:
            case = _attachment_case(c, host)
            if (case == "producer") != before:
                continue
            offs = {}
            if case == "producer":
                rds = [r for r in _reads(host.expr) if r.buffer == c.name]
                dims = self.shape(c.name)
                for d, (name, _) in enumerate(c.space):
                    lo = None
                    for r in rds:
                        a, _ = lin_decode_interval(r.index[d], hmap, ranges)
                        a += sum(co * host_off.get(it, 0) for it, co in r.index[d].terms)
                        lo = a if lo is None else min(lo, a)
                    w = next((l.extent for l in c.loops if l.id == name), 1)
                    offs[name] = max(0, min(lo or 0, dims[d] - w))
            else:
                dims = self.shape(host.name)
                for (name, _), (orig, _), dim in zip(c.space, host.space, dims):
                    a, _ = d_interval(hmap[orig], ranges) if orig in hmap else ranges[orig]
                    a += host_off.get(orig, 0)
                    w = next((l.extent for l in c.loops if l.id == name), 1)
                    offs[name] = max(0, min(a, dim - w))
            self.run_stage(c, offs)

    def _grid(self, s, offsets, tail, env, accumulate):
        grids = np.meshgrid(*[np.arange(l.extent) for l in tail], indexing="ij", sparse=True) if tail else []
        shape = tuple(l.extent for l in tail)
        genv = dict(env)
        genv.update({l.id: g for l, g in zip(tail, grids)})
        ienv = {}
        for n, d in s.index_map:
            v = d_eval(d, genv)
            o = offsets.get(n, 0)
            ienv[n] = v + o if o else v
        mask = np.ones(shape, dtype=bool)
        body = s.expr.body if _k(s.expr) == "Reduce" else s.expr
        vals = np.broadcast_to(np.asarray(evaluate(body, ienv, self.reader(f"stage {s.name}"), mask),
                                          dtype=np.float64), shape)
        red = tuple(i for i, l in enumerate(tail) if l.kind == "reduce")
        op = s.expr.op if _k(s.expr) == "Reduce" else None
        if red:
            vals = np.add.reduce(vals, axis=red) if op == "sum" else np.maximum.reduce(vals, axis=red)
        keep = tuple(0 if i in red else slice(None) for i in range(len(tail)))
        widx = tuple(np.broadcast_to(np.asarray(ienv[n]), shape)[keep] for n, _ in s.space)
        buf = self.bufs[s.name]
        if accumulate:
            buf[widx] = np.maximum(buf[widx], vals) if op == "max" else buf[widx] + vals
        else:
            buf[widx] = vals


def interpret(p, inputs: dict) -> dict:
    if not p.is_concrete():
        raise InterpreterError("program has unresolved symbolic extents")
    bufs = {}
    for n in p.dag.nodes:
        if n.is_placeholder:
            if n.name not in inputs:
                raise InterpreterError(f"missing input {n.name}")
            a = np.asarray(inputs[n.name], dtype=np.float64)
            if a.shape != n.shape:
                raise InterpreterError(f"input {n.name} has shape {a.shape}, expected {n.shape}")
            bufs[n.name] = a
    packed = {b: (pack_buffer(bufs[b], d), d) for b, d in p.layouts}
    for s in p.stages:
        if not s.inlined:
            bufs[s.name] = np.full(tuple(e for _, e in s.space), np.nan)
    ex = _Exec(p, bufs, packed)
    for s in p.stages:
        if not s.inlined and s.compute_at is None:
            ex.run_stage(s, {})
    out = {}
    for o in p.dag.outputs:
        if np.isnan(bufs[o]).any():
            raise InterpreterError(f"output {o} has unwritten cells")
        out[o] = bufs[o]
    return out
