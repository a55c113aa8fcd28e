"""State encoder: Program objects -> flat int32 statement records for the
batched feature kernel (`csrc/features.cu`).

Everything the reference's `analyze_program` (`src/features.py:161-284`)
derives *structurally* is resolved here, once, on the host; everything it
derives *arithmetically* (decode-AST intervals and evaluations, hulls, reuse,
strides, working sets, the 164-wide row) is left to the GPU.  Host-side
resolutions, each cited:

* live statements in stage order, nest = attach-chain host loops + own loops
  with extent > 1 (`_nest_above`, `src/features.py:114-121,163-170`);
* loop identity is *by id string* (`src/features.py:224-225`): each nest
  position carries the index of the own loop with the same id (or -1), and each
  own loop carries the last nest position with its id (the `free` test of
  `ws_inside`, `src/features.py:266-274`);
* buffer views in first-access order, reads pre-order then the write
  (`src/features.py:183-200`); a view's dims come from its first access;
  packed constants add (stride, extent) per physical dim (`_phys_decodes`,
  `src/features.py:124-140`);
* buffer-name rank for the (-bytes, name) ordering (`src/features.py:398`);
* op counts of the stage expression (`src/expr.py:303-327`).

Record layout (int32 words, one record per statement, see include/loomtune_b200.h):

  header[HDR]  n_nest own_start n_loops n_iter n_views unroll n_live has_reduce
               ops[9]  n_nodes
  nest[n_nest]  x (extent, kind, annotation, own_index)
  loops[n_loops] x (extent, kind, last_nest_pos)
  iter[n_iter]  x (node_offset, node_count)          postfix decode ASTs per iterator
  nodes[n_nodes] x (op, arg)                          op: 0 var(own loop idx) 1 const
                                                         2 add 3 mul(c) 4 div(c) 5 mod(c)
  views[n_views]: n_marks has_write name_rank n_dims,
                  dims: (size, pack_stride, pack_ext, const, n_terms, (iter, coeff) x n_terms)
                  pack_ext == 0 means "not packed".
"""

from __future__ import annotations

import numpy as np

from .state import kind, op_counts, reads

HDR = 18
OP_VAR, OP_CONST, OP_ADD, OP_MUL, OP_DIV, OP_MOD = range(6)
ANN = {None: 0, "parallel": 1, "vectorize": 2}
KINDS = ("add", "sub", "mul", "div", "minmax", "cmp", "math_call", "select", "other")


class EncodeError(ValueError):
    pass


def _ops(expr, cache: dict) -> list:
    key = id(expr)
    hit = cache.get(key)
    if hit is None or hit[0] is not expr:
        c = op_counts(expr) if expr is not None else {}
        hit = (expr, [c.get(k, 0) for k in KINDS])
        cache[key] = hit
    return hit[1]


_DECODE_OP = {"DMul": OP_MUL, "DDiv": OP_DIV, "DMod": OP_MOD}


def _postfix(d, loop_idx: dict, out: list) -> None:
    """Postfix form of a decode AST (`src/ir.py:36-70`), iteratively: operands
    before operators, DAdd's left subtree first."""
    stack = [(d, False)]
    pop, push = stack.pop, stack.append
    while stack:
        node, done = pop()
        k = type(node).__name__
        if k == "DVar":
            j = loop_idx.get(node.loop)
            if j is None:
                raise EncodeError(f"decode references unknown loop {node.loop!r}")
            out += (OP_VAR, j)
        elif k == "DConst":
            out += (OP_CONST, int(node.value))
        elif k == "DAdd":
            if done:
                out += (OP_ADD, 0)
            else:
                push((node, True))
                push((node.b, False))
                push((node.a, False))
        else:
            if done:
                out += (_DECODE_OP[k], int(node.c))
            else:
                if node.c is None:
                    raise EncodeError("symbolic factor in decode")
                push((node, True))
                push((node.a, False))


def _stage_map(p) -> dict:
    return {s.name: s for s in p.stages}


def _nest_above(smap: dict, s) -> list:
    if s.compute_at is None:
        return []
    tname, lid = s.compute_at
    t = smap[tname]
    ids = [l.id for l in t.loops]
    return _nest_above(smap, t) + list(t.loops[: ids.index(lid) + 1])


def encode_program(p, out: list, ops_cache: dict, gpu_features: bool = False) -> int:
    """Append one record per live statement of `p` to `out` (a list of int
    lists); returns the number of statements.  gpu_features: flag the record
    (has_reduce bit 1) and append the statement's kernel binding (blockIdx.x,
    blockIdx.y, blockIdx.z, threadIdx.x, threadIdx.y, threadIdx.z, vthread,
    shared bytes) as 8 trailing words; the kernel fills the gpu_* slots from them."""
    smap = _stage_map(p)
    layouts = dict(p.layouts)
    live = [s for s in p.stages if not s.inlined]
    shapes = {s.name: tuple(e for _, e in s.space) for s in p.stages}
    for s in live:
        above = [l for l in _nest_above(smap, s) if (l.extent or 1) > 1]
        own = [l for l in s.loops if (l.extent or 1) > 1]
        nest = above + own
        loop_idx = {l.id: j for j, l in enumerate(s.loops)}
        last_pos = {}
        for q, l in enumerate(nest):
            last_pos[l.id] = q
        iters = [n for n, _ in s.index_map]
        iter_idx = {n: j for j, n in enumerate(iters)}
        dmap = dict(s.index_map)

        nodes: list = []
        iter_tab: list = []
        extra_iters: list = []          # iterators read but absent from the map -> DVar(name)
        for n in iters:
            start = len(nodes) // 2
            _postfix(dmap[n], loop_idx, nodes)
            iter_tab += (start, len(nodes) // 2 - start)

        def iter_slot(name: str) -> int:
            if name in iter_idx:
                return iter_idx[name]
            if name not in loop_idx:
                raise EncodeError(f"iterator {name!r} has no decode and no loop")
            iter_idx[name] = len(iters) + len(extra_iters)
            extra_iters.append(name)
            start = len(nodes) // 2
            nodes.extend((OP_VAR, loop_idx[name]))
            iter_tab.extend((start, 1))
            return iter_idx[name]

        views: dict = {}
        order: list = []
        accesses = [(r.buffer, r.index, 0) for r in reads(s.expr)] if s.expr is not None else []
        accesses.append((s.name, None, 1))
        for buf, idx, is_w in accesses:
            if buf not in views:
                if idx is None:
                    lins = [((n, 1),) for n, _ in s.space]
                    consts = [0] * len(s.space)
                else:
                    lins = [l.terms for l in idx]
                    consts = [l.const for l in idx]
                dims = []
                desc = layouts.get(buf)
                logical = [(consts[d], [(iter_slot(n), c) for n, c in lins[d]]) for d in range(len(lins))]
                if desc is not None:
                    for i, (d, ext) in enumerate(desc):
                        st = 1
                        for d2, e2 in desc[i + 1:]:
                            if d2 == d:
                                st *= e2
                        dims.append((ext, st, ext, logical[d]))
                else:
                    shape = shapes[buf] if buf in shapes else p.dag.node(buf).shape
                    dims = [(shape[d], 1, 0, logical[d]) for d in range(len(logical))]
                views[buf] = [0, 0, dims]
                order.append(buf)
            views[buf][0] += 1
            views[buf][1] |= is_w
        rank = {b: r for r, b in enumerate(sorted(order))}

        rec = [len(nest), len(above), len(s.loops), len(iter_tab) // 2, len(order),
               int(s.pragma_unroll), len(live), (1 if s.reduce else 0) | (2 if gpu_features else 0)]
        rec += _ops(s.expr, ops_cache)
        rec.append(len(nodes) // 2)
        for l in nest:
            rec += (int(l.extent), 0 if l.kind == "space" else 1, ANN.get(l.annotation, 0),
                    loop_idx.get(l.id, -1))
        for l in s.loops:
            rec += (int(l.extent or 1), 0 if l.kind == "space" else 1, last_pos.get(l.id, -1))
        rec += iter_tab
        rec += nodes
        for b in order:
            n_marks, has_w, dims = views[b]
            rec += (n_marks, has_w, rank[b], len(dims))
            for size, st, pext, (const, terms) in dims:
                rec += (int(size), st, pext, int(const), len(terms))
                for it, c in terms:
                    rec += (it, int(c))
        if gpu_features:
            from .lower import gpu_binding
            nb, nt, nv, smem = gpu_binding(p, s)
            rec += (min(nb, 2 ** 31 - 1), 1, 1, nt, 1, 1, nv, smem)
        out.append(rec)
    return len(live)


def _native():
    """The native encoder (`csrc/encode_ext.cpp`, built in-tree by build.py): the same
    records as `encode_program`, produced by C++ walking the reference's objects."""
    global _NATIVE
    if _NATIVE is None:
        import importlib.util
        import glob
        import os
        lib = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
        hits = glob.glob(os.path.join(lib, "_lt_encode*.so"))
        if not hits:
            raise ImportError(f"native encoder not built in {lib} (run python -m paper_2006_06762_b200.build)")
        spec = importlib.util.spec_from_file_location("_lt_encode", hits[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mod.set_error(EncodeError)
        _NATIVE = mod
    return _NATIVE


_NATIVE = None


def encode_batch(programs, gpu_features: bool = False, native: bool | None = None) -> tuple:
    """-> (words int32[], stmt_offsets int64[n_stmt+1], prog_row_offsets int64[n_prog+1]).
    The native encoder runs unless gpu_features is asked (its kernel-binding words come
    from the lowering, in Python) or native=False / LT_PY_ENCODER=1 (A/B and tests)."""
    if native is None:
        import os
        native = os.environ.get("LT_PY_ENCODER", "") != "1"
    if native and not gpu_features:
        w, so, po = _native().encode_batch(list(programs))
        return np.frombuffer(w, np.int32), np.frombuffer(so, np.int64), np.frombuffer(po, np.int64)
    recs: list = []
    prog_off = [0]
    cache: dict = {}
    for p in programs:
        prog_off.append(prog_off[-1] + encode_program(p, recs, cache, gpu_features))
    stmt_off = np.zeros(len(recs) + 1, dtype=np.int64)
    np.cumsum([len(r) for r in recs], out=stmt_off[1:])
    flat: list = []
    for r in recs:
        flat.extend(r)
    words = np.array(flat, dtype=np.int32)
    return words, stmt_off, np.asarray(prog_off, dtype=np.int64)
