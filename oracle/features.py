"""ORACLE (test infrastructure only): CPU restatement of per-statement feature
extraction, `extract_features` (`src/features.py:161-425`).

Only tests/, `__graft_entry__.smoke()` and bench.py's cpu_baseline leg may use
this module, and only as the checker.  It is pinned against the reference
itself: `tests/golden/features.npz` holds the reference's own
`extract_features` output for every corpus State (made by
`tools/make_golden.py` with the reference imported in the build container),
and `tests/test_oracle.py` requires this restatement to reproduce it exactly.

Works on any Program object with the reference's field names (the reference's
own, or the package mirror).  Pure Python + numpy, independent of the product
package.
"""

from __future__ import annotations

import math

import numpy as np

LINE_BYTES = 64
ELEM_BYTES = 4
N_FEATURES = 164
KINDS = ("add", "sub", "mul", "div", "minmax", "cmp", "math_call", "select", "other")
POS = ("none", "inner_spatial", "middle_spatial", "outer_spatial",
       "inner_reduce", "middle_reduce", "outer_reduce", "mixed")
ACC = ("read", "write", "read_write")
REUSE = ("loop_multiple_read", "serial_multiple_read", "no_reuse")


def _onehot_mask() -> np.ndarray:
    """Columns kept raw (`src/features.py:74-78`): the position one-hots of the
    three annotation blocks and the access / reuse one-hots of each buffer block."""
    m = np.zeros(N_FEATURES, dtype=bool)
    for blk in (18, 29, 40):                      # vectorize, unroll, parallel blocks
        m[blk + 1: blk + 9] = True
    for b in range(5):                            # buffer blocks start at column 69
        base = 69 + 18 * b
        m[base: base + 3] = True
        m[base + 7: base + 10] = True
    return m


ONEHOT = _onehot_mask()


# --- decode / expression helpers (duck-typed on class names) ---------------

def _k(x) -> str:
    return type(x).__name__


def interval(d, ranges):
    k = _k(d)
    if k == "DVar":
        return ranges[d.loop]
    if k == "DConst":
        return d.value, d.value
    if k == "DAdd":
        a, b = interval(d.a, ranges), interval(d.b, ranges)
        return a[0] + b[0], a[1] + b[1]
    lo, hi = interval(d.a, ranges)
    c = d.c
    if k == "DMul":
        return (lo * c, hi * c) if c >= 0 else (hi * c, lo * c)
    if k == "DDiv":
        return lo // c, hi // c
    if lo // c == hi // c:                        # DMod, same block
        return lo % c, hi % c
    return 0, c - 1


def evaluate(d, env):
    k = _k(d)
    if k == "DVar":
        return env[d.loop]
    if k == "DConst":
        return d.value
    if k == "DAdd":
        return evaluate(d.a, env) + evaluate(d.b, env)
    a = evaluate(d.a, env)
    return a * d.c if k == "DMul" else (a // d.c if k == "DDiv" else a % d.c)


def variables(d) -> set:
    k = _k(d)
    if k == "DVar":
        return {d.loop}
    if k == "DConst":
        return set()
    if k == "DAdd":
        return variables(d.a) | variables(d.b)
    return variables(d.a)


_TYPES: dict = {}


def _node(name, fields):
    cls = _TYPES.setdefault(name, type(name, (), {}))
    o = cls()
    o.__dict__.update(fields)
    return o


def compose(lin, dmap):
    """`lin_to_decode` (`src/ir.py:152-160`)."""
    out = _node("DConst", {"value": lin.const})
    for name, c in lin.terms:
        t = dmap.get(name) or _node("DVar", {"loop": name})
        if c != 1:
            t = _node("DMul", {"a": t, "c": c})
        out = t if (_k(out) == "DConst" and out.value == 0) else _node("DAdd", {"a": out, "b": t})
    return out


def _walk(e):
    yield e
    k = _k(e)
    kids = ((e.lhs, e.rhs) if k == "Bin" else (e.arg,) if k == "Call" else
            (e.cond, e.then, e.other) if k == "Select" else (e.body,) if k == "Reduce" else ())
    for c in kids:
        yield from _walk(c)


def op_counts(e) -> dict:
    table = {"add": "add", "sub": "sub", "mul": "mul", "div": "div", "max": "minmax",
             "min": "minmax", "lt": "cmp", "le": "cmp", "gt": "cmp", "ge": "cmp", "eq": "cmp"}
    out: dict = {}
    for n in _walk(e):
        k = _k(n)
        key = (table[n.op] if k == "Bin" else "math_call" if k == "Call" else "select"
               if k == "Select" else ("add" if n.op == "sum" else "minmax") if k == "Reduce" else None)
        if key:
            out[key] = out.get(key, 0) + 1
    return out


def _reads(e):
    return [n for n in _walk(e) if _k(n) == "Read"]


# --- analysis --------------------------------------------------------------

def _stage(p, name):
    return next(s for s in p.stages if s.name == name)


def _host_loops(p, s):
    """Loops of the attach chain above `s`, outermost first (`_nest_above`)."""
    if s.compute_at is None:
        return []
    tname, lid = s.compute_at
    t = _stage(p, tname)
    pos = [l.id for l in t.loops].index(lid)
    return _host_loops(p, t) + list(t.loops[: pos + 1])


def _packed(decs, desc):
    out = []
    for i, (d, ext) in enumerate(desc):
        st = 1
        for d2, e2 in desc[i + 1:]:
            if d2 == d:
                st *= e2
        dec = decs[d]
        if st > 1:
            dec = _node("DDiv", {"a": dec, "c": st})
        out.append((_node("DMod", {"a": dec, "c": ext}), ext))
    return out


def _widths(dims, ranges):
    w = []
    for dec, size in dims:
        lo, hi = interval(dec, ranges)
        w.append(max(min(hi, size - 1) - max(lo, 0) + 1, 1))
    return w


def _prod(xs) -> float:
    out = 1.0
    for x in xs:
        out *= x
    return out


def _buffer_shape(p, name):
    for s in p.stages:
        if s.name == name:
            return tuple(e for _, e in s.space)
    return p.dag.node(name).shape


def analyze(p, with_present: bool = True) -> list:
    """One dict per live statement, fields as `StatementAnalysis`."""
    layouts = dict(p.layouts)
    live = [s for s in p.stages if not s.inlined]
    stmts = []
    for s in live:
        nest = [l for l in _host_loops(p, s) if (l.extent or 1) > 1]
        own = [l for l in s.loops if (l.extent or 1) > 1]
        own_start = len(nest)
        nest += own
        total = _prod(l.extent for l in nest)
        ops = op_counts(s.expr) if s.expr is not None else {}
        dmap = dict(s.index_map)
        own_rng = {l.id: (0, (l.extent or 1) - 1) for l in s.loops}

        views: dict = {}
        accesses = [(r.buffer, r.index, "read") for r in _reads(s.expr)] if s.expr is not None else []
        accesses.append((s.name, [_node("Lin", {"terms": ((n, 1),), "const": 0}) for n, _ in s.space],
                         "write"))
        for buf, lins, mark in accesses:
            decs = [compose(l, dmap) for l in lins]
            dims = _packed(decs, layouts[buf]) if buf in layouts else list(zip(decs, _buffer_shape(p, buf)))
            views.setdefault(buf, (dims, []))[1].append(mark)

        red_prod = _prod(l.extent for l in own if l.kind == "reduce")
        acc_list = []
        for buf, (dims, marks) in views.items():
            n_acc = len(marks)
            has_w = "write" in marks
            has_r = "read" in marks or (has_w and red_prod > 1)
            acc = "read_write" if has_w and has_r else "write" if has_w else "read"
            present = set().union(*(variables(d) for d, _ in dims)) if dims else set()
            w = _widths(dims, own_rng)
            ub = _prod(w) * ELEM_BYTES if w else ELEM_BYTES
            ul = _prod(w[:-1]) * max(1.0, math.ceil((w[-1] if w else 1) * ELEM_BYTES / LINE_BYTES))
            touches = float(n_acc) * total
            tb = touches * ELEM_BYTES
            absent = [i for i, l in enumerate(nest) if l.id not in present and l.extent > 1]
            if has_w and s.reduce and red_prod > 1:
                rt, cnt, di, db = "serial_multiple_read", red_prod, 1.0, float(ELEM_BYTES * n_acc)
            elif absent:
                rt = "loop_multiple_read"
                cnt = _prod(nest[i].extent for i in absent)
                di = _prod(l.extent for l in nest[absent[-1] + 1:])
                db = di * ELEM_BYTES * n_acc
            else:
                rt, cnt, di, db = "no_reuse", 1.0, 0.0, 0.0
            stride = 0.0
            if own and own[-1].id in present:
                fs, a = [], 1
                for _, size in reversed(dims):
                    fs.append(a)
                    a *= size
                fs.reverse()
                e0 = {l.id: 0 for l in s.loops}
                e1 = dict(e0)
                e1[own[-1].id] = 1
                clip = lambda v, n: min(max(v, 0), n - 1)  # noqa: E731
                a0 = sum(clip(evaluate(d, e0), n) * f for (d, n), f in zip(dims, fs))
                a1 = sum(clip(evaluate(d, e1), n) * f for (d, n), f in zip(dims, fs))
                stride = abs(a1 - a0) * ELEM_BYTES
            acc_list.append(dict(buffer=buf, acc=acc, present=present, total_bytes=tb, unique_bytes=ub,
                                 lines=tb / LINE_BYTES, unique_lines=ul, reuse=rt, counter=cnt,
                                 dist_iters=di, dist_bytes=db, stride=stride))
        ws = []
        for pos in range(len(nest)):
            free = {l.id for l in nest[pos + 1:]}
            rng = {l.id: ((0, (l.extent or 1) - 1) if l.id in free else (0, 0)) for l in s.loops}
            ws.append(sum(_prod(_widths(dims, rng)) * ELEM_BYTES for dims, _ in views.values()))
        alloc = float(ELEM_BYTES) * _prod(l.extent for l in own if l.kind == "space")
        stmts.append(dict(nest=nest, own_start=own_start, total=total, ops=ops,
                          ops_total=sum(ops.values()), accesses=acc_list, ws=ws, alloc=alloc,
                          unroll=s.pragma_unroll, n_live=len(live)))
    return stmts


def _position(nest, i) -> str:
    same = [j for j, l in enumerate(nest) if l.kind == nest[i].kind]
    r = same.index(i)
    sfx = "spatial" if nest[i].kind == "space" else "reduce"
    return ("inner_" if r == len(same) - 1 else "outer_" if r == 0 and len(same) > 1 else "middle_") + sfx


def _block(hits, nest) -> list:
    b = [0.0] * 11
    if not hits:
        b[1] = 1.0
        return b
    tags = {_position(nest, i) for i in hits}
    b[0] = float(nest[hits[-1]].extent)
    b[1 + POS.index(tags.pop() if len(tags) == 1 else "mixed")] = 1.0
    b[9] = _prod(nest[i].extent for i in hits)
    b[10] = float(len(hits))
    return b


def row(st) -> np.ndarray:
    nest = st["nest"]
    v = [float(st["ops"].get(k, 0)) * st["total"] for k in KINDS] + [0.0] * 9
    v += _block([i for i, l in enumerate(nest) if l.annotation == "vectorize"], nest)
    covered, prod = [], 1
    if st["unroll"] > 0 and len(nest) > st["own_start"]:
        for i in range(len(nest) - 1, st["own_start"] - 1, -1):
            if prod * nest[i].extent > st["unroll"]:
                break
            prod *= nest[i].extent
            covered.append(i)
    ub = _block(covered, nest)
    if covered:
        ub[0], ub[9] = float(nest[covered[0]].extent), float(prod)
    v += ub
    v += _block([i for i, l in enumerate(nest) if l.annotation == "parallel"], nest)
    v += [0.0] * 8
    n = len(nest)
    if n == 0 or st["ops_total"] == 0:
        v += [0.0] * 10
    else:
        inside = [1.0] * (n + 1)
        for i in range(n - 1, -1, -1):
            inside[i] = inside[i + 1] * nest[i].extent
        for j in range(1, 11):
            pos = n - max(1, math.ceil(j / 10 * n))
            by = sum(a["unique_bytes"] for a in st["accesses"]) if pos == 0 else st["ws"][pos - 1]
            v.append(st["ops_total"] * inside[pos] / max(by, 1.0))
    ranked = sorted(st["accesses"], key=lambda a: (-a["total_bytes"], a["buffer"]))[:5]
    for a in ranked:
        oh = [0.0] * 3
        oh[ACC.index(a["acc"])] = 1.0
        rh = [0.0] * 3
        rh[REUSE.index(a["reuse"])] = 1.0
        c = max(a["counter"], 1.0)
        v += oh + [a["total_bytes"], a["unique_bytes"], a["lines"], a["unique_lines"]] + rh
        v += [a["dist_iters"], a["dist_bytes"], a["counter"], a["stride"],
              a["total_bytes"] / c, a["unique_bytes"] / c, a["lines"] / c, a["unique_lines"] / c]
    v += [0.0] * (18 * (5 - len(ranked)))
    v += [st["alloc"], float(st["n_live"]), float(n), st["total"], float(st["unroll"])]
    arr = np.asarray(v, dtype=np.float64)
    return np.where(ONEHOT, arr, np.log2(1.0 + np.maximum(arr, 0.0)))


def extract_features(p) -> np.ndarray:
    rows = [row(st) for st in analyze(p)]
    return np.vstack(rows) if rows else np.zeros((0, N_FEATURES))
