"""Direct PTX backend for the candidate templates (no NVVM).

NVRTC spends 80-90% of a candidate's compile in NVVM (C++ -> PTX); ptxas alone
is 5-10x faster.  This module emits PTX for exactly the templates `lower.py`
defines in CUDA C (same binding, staging, loop order, unroll coverage,
epilogues, legality), so a candidate only pays for ptxas.  It performs the
optimisations NVVM would otherwise do for these kernels: affine address
arithmetic folded into `[reg + imm]` forms, value numbering of address and
shared-memory loads inside straight-line regions, magic-number division by
constants (ptxas emits a generic reciprocal sequence for `div.u32` by an
immediate), fused multiply-add for sum-of-products reductions, predicated loads
for `Select` branches.

Unsupported constructs (math calls whose PTX approximations would not meet the
1e-4 contract: exp/log) raise `Unsupported`; the runner then uses the NVRTC
path for that candidate.  `tests/test_ptx_gpu.py` checks both backends produce
identical verdicts and outputs.
"""

from __future__ import annotations

import itertools
import math
import os
import struct

import numpy as np

from .lower import (
    MAX_ACC, MAX_SMEM, MAX_THREADS, MAX_UNROLLED, MAX_VTHREAD, NAIVE_THREADS, Buffer, Kernel,
    Lowered, LoweringError, _attached, _binding, _must_materialize, _reads_buffer, _unroll_flags, promote_register_tile,
    _written, ident, tile_levels,
)
from .state import kind, reads


# statements between a shared-memory load and its first use (16-128 measured within 2%
# of each other on the template bench after the reduction-outer nest order)
LOOKAHEAD = int(os.environ.get("LT_LOOKAHEAD", "64"))
SPILL_MARGIN = 24    # registers beyond the accumulator tile a tiled kernel needs
ASYNC_MAX_TRIPS = 64  # cp.async staging: per-operand trips per thread (carry-free beyond 16)
# template switches (all on in production; LT_PTX_OFF=promote,plan,pad turns them off for A/B checks)
_OFF = set(os.environ.get("LT_PTX_OFF", "").split(","))
FETCH_CHUNK = 1 if "chunk" in _OFF else 8   # loads in flight per thread in a rolled cooperative fetch
HOIST_SPILL_UNROLLED = 64   # spilling register tiles: reduction-outer order only up to this unrolled body


class Unsupported(Exception):
    pass


# ---------------------------------------------------------------------------
# affine integer forms over registers
# ---------------------------------------------------------------------------


class Aff:
    __slots__ = ("terms", "const")

    def __init__(self, terms=None, const=0):
        self.terms = {r: c for r, c in terms.items() if c} if terms else {}
        self.const = int(const)

    @staticmethod
    def _raw(terms: dict, const: int) -> "Aff":
        """No copying or zero filtering: `terms` is already clean and is never
        mutated afterwards (Aff values are immutable; dicts may be shared)."""
        a = object.__new__(Aff)
        a.terms, a.const = terms, const
        return a

    @staticmethod
    def reg(r, c=1):
        return Aff._raw({r: c} if c else {}, 0)

    @staticmethod
    def k(c):
        return Aff._raw({}, int(c))

    def __add__(self, o):
        if isinstance(o, int):
            return Aff._raw(self.terms, self.const + o)
        if not o.terms:
            return Aff._raw(self.terms, self.const + o.const)
        if not self.terms:
            return Aff._raw(o.terms, self.const + o.const)
        t = dict(self.terms)
        for r, c in o.terms.items():
            v = t.get(r, 0) + c
            if v:
                t[r] = v
            else:
                del t[r]
        return Aff._raw(t, self.const + o.const)

    def scale(self, s):
        if not s:
            return Aff._raw({}, 0)
        return Aff._raw({r: c * s for r, c in self.terms.items()}, self.const * s)

    def runtime(self):
        return Aff._raw(self.terms, 0)

    def key(self):
        return tuple(sorted(self.terms.items()))


def _reg_order(item):
    reg = item[0]
    i = len(reg)
    while i and reg[i - 1].isdigit():
        i -= 1
    return (reg[:i], int(reg[i:]) if i < len(reg) else -1)


def _magic(d):
    L = (d - 1).bit_length()
    return -(-(1 << (31 + L)) // d), L - 1


def _f32(x) -> str:
    return "0f%08X" % struct.unpack("<I", struct.pack("<f", float(x)))[0]


def _f64(x) -> str:
    return "0d%016X" % struct.unpack("<Q", struct.pack("<d", float(x)))[0]


_MISSING = object()


class Ptx:
    """One kernel's instruction stream with scoped value numbering."""

    def __init__(self, dtype: str):
        self.ft = "f32" if dtype == "float" else "f64"
        self.fr = "%f" if self.ft == "f32" else "%fd"
        self.esz = 4 if self.ft == "f32" else 8
        self.n = {"%r": 0, "%rd": 0, "%p": 0, self.fr: 0}
        self.lines: list = []
        self.table: dict = {}           # key -> value, innermost scope wins
        self.undo: list = [[]]          # per scope: (key, shadowed value) to restore on pop
        self.labels = 0

    def new(self, cls: str) -> str:
        self.n[cls] += 1
        return f"{cls}{self.n[cls]}"

    def __call__(self, s: str) -> None:
        self.lines.append("  " + s)

    def label(self, name: str) -> None:
        self.lines.append(f"{name}:")

    def new_label(self) -> str:
        self.labels += 1
        return f"L{self.labels}"

    def fconst(self, x) -> str:
        return _f32(x) if self.ft == "f32" else _f64(x)

    # value numbering
    def cached(self, key):
        return self.table.get(key)

    def remember(self, key, val):
        self.undo[-1].append((key, self.table.get(key, _MISSING)))
        self.table[key] = val
        return val

    def push(self):
        self.undo.append([])

    def pop(self):
        for key, old in reversed(self.undo.pop()):
            if old is _MISSING:
                del self.table[key]
            else:
                self.table[key] = old

    # integer arithmetic
    def aff(self, a: Aff) -> str:
        key = ("aff", a.key(), a.const)
        hit = self.cached(key)
        if hit:
            return hit
        r = None
        # oldest registers first: the loop-invariant prefix of the chain is then
        # hoistable by ptxas out of rolled loops
        terms = sorted(a.terms.items(), key=_reg_order if "order" not in _OFF else None)
        start = 0
        if "prefix" not in _OFF:
            # every partial sum of two or more terms is value-numbered: chains that share
            # a prefix (each fetch trip's address = the same block / stage part + its own
            # digits) reuse it instead of re-emitting it (smaller PTX, less ptxas time)
            for j in range(len(terms), 1, -1):
                hit = self.cached(("affp", tuple(terms[:j])))
                if hit:
                    r, start = hit, j
                    break
        for j in range(start, len(terms)):
            reg, c = terms[j]
            if r is None:
                if c == 1:
                    r = reg
                else:
                    r = self.new("%r")
                    self(f"mul.lo.s32 {r}, {reg}, {c};")
            else:
                nr = self.new("%r")
                if c == 1:
                    self(f"add.s32 {nr}, {reg}, {r};")
                else:
                    self(f"mad.lo.s32 {nr}, {reg}, {c}, {r};")
                r = nr
                if "prefix" not in _OFF:
                    self.remember(("affp", tuple(terms[:j + 1])), r)
        if r is None:
            r = self.new("%r")
            self(f"mov.s32 {r}, {a.const};")
        elif a.const:
            nr = self.new("%r")
            self(f"add.s32 {nr}, {r}, {a.const};")
            r = nr
        return self.remember(key, r)

    def udiv(self, x: str, d: int) -> str:
        if d == 1:
            return x
        key = ("div", x, d)
        hit = self.cached(key)
        if hit:
            return hit
        r = self.new("%r")
        if d & (d - 1) == 0:
            self(f"shr.u32 {r}, {x}, {d.bit_length() - 1};")
        else:
            m, s = _magic(d)
            self(f"mul.hi.u32 {r}, {x}, {m};")
            if s:
                self(f"shr.u32 {r}, {r}, {s};")
        return self.remember(key, r)

    def urem(self, x: str, d: int) -> str:
        if d == 1:
            return self.aff(Aff.k(0))
        key = ("rem", x, d)
        hit = self.cached(key)
        if hit:
            return hit
        r = self.new("%r")
        if d & (d - 1) == 0:
            self(f"and.b32 {r}, {x}, {d - 1};")
        else:
            q = self.udiv(x, d)
            self(f"mad.lo.s32 {r}, {q}, {-d}, {x};")
        return self.remember(key, r)

    def decompose(self, x: str, radices: list) -> list:
        """Mixed-radix digits of x (last radix fastest)."""
        out = [None] * len(radices)
        cur = x
        for i in range(len(radices) - 1, -1, -1):
            d = radices[i]
            if i == 0:
                out[i] = cur
            else:
                out[i] = self.urem(cur, d)
                cur = self.udiv(cur, d)
        return out

    def gaddr(self, base: str, flat: Aff) -> tuple:
        """(64-bit base register, byte immediate) for element `flat` of a global buffer."""
        rt = flat.runtime()
        key = ("gaddr", base, rt.key())
        hit = self.cached(key)
        if hit is None:
            if rt.terms:
                off = self.aff(rt)
                w = self.new("%rd")
                self(f"mul.wide.s32 {w}, {off}, {self.esz};")
                hit = self.new("%rd")
                self(f"add.s64 {hit}, {base}, {w};")
            else:
                hit = base
            self.remember(key, hit)
        return hit, flat.const * self.esz


# ---------------------------------------------------------------------------
# expression emission
# ---------------------------------------------------------------------------


class Expr:
    """Emit a scalar expression; `read(buf, index_affs, guard)` yields a register."""

    def __init__(self, g: Ptx, iv, read):
        self.g, self.iv, self.read = g, iv, read
        self.guard = None           # predicate register: loads run only where it holds

    def lin(self, lin) -> Aff:
        a = Aff.k(lin.const)
        for n, c in lin.terms:
            a = a + self.iv(n).scale(c)
        return a

    def pred(self, e):
        """Predicate register of a condition built from comparisons of IterVal
        with constants, multiplied together (the padding stage's in-bounds test,
        `src/workloads.py:45-67`), in integer arithmetic: the same truth value as
        the float evaluation (0/1 products, != 0) without int->float conversions
        and float multiplies.  None when the condition has another shape."""
        g = self.g
        k = kind(e)
        if k != "Bin":
            return None
        if e.op == "mul":
            a = self.pred(e.lhs)
            b = self.pred(e.rhs) if a is not None else None
            if b is None:
                return None
            p = g.new("%p")
            g(f"and.pred {p}, {a}, {b};")
            return p
        if e.op not in ("ge", "gt", "le", "lt") or "ipred" in _OFF:
            return None
        lhs, rhs, op = e.lhs, e.rhs, e.op
        if kind(lhs) == "Const" and kind(rhs) == "IterVal":
            lhs, rhs, op = rhs, lhs, {"ge": "le", "le": "ge", "gt": "lt", "lt": "gt"}[op]
        if kind(lhs) != "IterVal" or kind(rhs) != "Const":
            return None
        c = float(rhs.value)
        if not math.isfinite(c) or abs(c) > 2 ** 30:
            return None
        ci = math.ceil(c) if op in ("ge", "lt") else math.floor(c)   # integer x vs real c
        a = self.lin(lhs.lin)
        if not a.terms:
            return None
        x = g.aff(Aff(a.terms))
        p = g.new("%p")
        g(f"setp.{op}.s32 {p}, {x}, {ci - a.const};")
        return p

    def __call__(self, e) -> str:
        g = self.g
        k = kind(e)
        if k == "Const":
            return g.fconst(e.value)
        if k == "IterVal":
            r = g.aff(self.lin(e.lin))
            f = g.new(g.fr)
            g(f"cvt.rn.{g.ft}.s32 {f}, {r};")
            return f
        if k == "Read":
            return self.read(e.buffer, [self.lin(l) for l in e.index], self.guard)
        if k == "Bin":
            a, b = self(e.lhs), self(e.rhs)
            f = g.new(g.fr)
            op = e.op
            if op in ("add", "sub", "mul"):
                g(f"{op}.rn.{g.ft} {f}, {a}, {b};" if op != "sub" else f"sub.rn.{g.ft} {f}, {a}, {b};")
            elif op == "div":
                g(f"div.rn.{g.ft} {f}, {a}, {b};")
            elif op in ("max", "min"):
                g(f"{op}.{g.ft} {f}, {a}, {b};")
            else:
                p = g.new("%p")
                g(f"setp.{op}.{g.ft} {p}, {a}, {b};")
                g(f"selp.{g.ft} {f}, {g.fconst(1.0)}, {g.fconst(0.0)}, {p};")
            return f
        if k == "Call":
            a = self(e.arg)
            f = g.new(g.fr)
            if e.fn == "sqrt":
                g(f"sqrt.rn.{g.ft} {f}, {a};")
            elif e.fn == "abs":
                g(f"abs.{g.ft} {f}, {a};")
            else:
                raise Unsupported(f"math call {e.fn}")
            return f
        if k == "Select":
            p = self.pred(e.cond)
            if p is None:
                c = self(e.cond)
                p = g.new("%p")
                g(f"setp.ne.{g.ft} {p}, {c}, {g.fconst(0.0)};")
            np_ = g.new("%p")
            g(f"not.pred {np_}, {p};")
            outer = self.guard
            pt, pf = p, np_
            if outer is not None:
                pt, pf = g.new("%p"), g.new("%p")
                g(f"and.pred {pt}, {p}, {outer};")
                g(f"and.pred {pf}, {np_}, {outer};")
            self.guard = pt
            t = self(e.then)
            self.guard = pf
            o = self(e.other)
            self.guard = outer
            f = g.new(g.fr)
            g(f"selp.{g.ft} {f}, {t}, {o}, {p};")
            return f
        raise Unsupported(f"expression node {k}")


# ---------------------------------------------------------------------------
# kernel emission
# ---------------------------------------------------------------------------


class _Mod:
    """Module-level state shared by the kernels of one candidate."""

    def __init__(self, p, dtype):
        self.p, self.dtype, self.dag = p, dtype, p.dag
        self.live = {s.name: s for s in p.stages if not s.inlined}
        self.layouts = dict(p.layouts)
        self.buffers: dict = {}
        self._att: dict = {}
        self._rd: dict = {}
        self._mm: dict = {}

    def attached(self, host: str) -> list:
        hit = self._att.get(host)
        if hit is None:
            hit = self._att[host] = _attached(self.p, host)
        return hit

    def reads(self, expr, name: str) -> bool:
        key = (id(expr), name)
        hit = self._rd.get(key)
        if hit is None:
            hit = self._rd[key] = _reads_buffer(expr, name)
        return hit

    def must_materialize(self, stage) -> bool:
        hit = self._mm.get(stage.name)
        if hit is None:
            hit = self._mm[stage.name] = _must_materialize(self, stage)
        return hit

    def shape(self, name):
        if name in self.live:
            return tuple(e for _, e in self.live[name].space)
        return self.dag.node(name).shape


class _Kern:
    def __init__(self, mod: _Mod, entry: str, threads: int):
        self.m = mod
        self.g = Ptx(mod.dtype)
        self.entry = entry
        self.threads = threads
        self.params: list = []          # buffer names in order
        self.ptr: dict = {}             # buffer -> 64-bit global pointer register
        self.writes: set = set()
        self.body: list = []
        self.vec_stores = False         # set for fully unrolled epilogues
        self.store_guard = None         # predicate on epilogue stores (naive multi-point steps)
        self.pending: list = []

    def param(self, name: str) -> str:
        if name not in self.ptr:
            self.params.append(name)
            self.ptr[name] = f"%ptr{len(self.params)}"
        return self.ptr[name]

    # -- global memory ----------------------------------------------------
    def gflat(self, name: str, idx: list) -> Aff:
        shape = self.m.shape(name)
        flat, mul = Aff.k(0), 1
        for d in range(len(shape) - 1, -1, -1):
            flat = flat + idx[d].scale(mul)
            mul *= shape[d]
        return flat

    def gload(self, name: str, idx: list, guard) -> str:
        g = self.g
        base, flat = self.gsource(name, idx)
        key = ("gld", base, flat.key(), flat.const, guard)
        hit = g.cached(key)
        if hit:
            return hit
        rb, imm = g.gaddr(base, flat)
        f = g.new(g.fr)
        pred = f"@{guard} " if guard else ""
        if guard:
            g(f"mov.b{32 if g.ft == 'f32' else 64} {f}, 0;")
        g(f"{pred}ld.global.nc.{g.ft} {f}, [{rb}+{imm}];")
        return g.remember(key, f)

    def gsource(self, name: str, idx: list) -> tuple:
        """(pointer register, flat element Aff) of element `idx` of a global input,
        through the packed physical layout when the State rewrote it."""
        g, m = self.g, self.m
        desc = m.layouts.get(name) if name not in m.live else None
        if desc is not None:
            key = f"{name}#packed"
            if key not in m.buffers:
                m.buffers[key] = Buffer(key, tuple(e for _, e in desc), "packed", tuple(desc), name)
            base = self.param(key)
            regs = {}
            flat, mul = Aff.k(0), 1
            for j in range(len(desc) - 1, -1, -1):
                d, e = desc[j]
                st = 1
                for d2, e2 in desc[j + 1:]:
                    if d2 == d:
                        st *= e2
                if d not in regs:
                    regs[d] = g.aff(idx[d])
                x = g.udiv(regs[d], st)
                if e < m.shape(name)[d] or st > 1:
                    x = g.urem(x, e)
                flat = flat + Aff.reg(x, mul)
                mul *= e
        else:
            if name not in m.live and name not in m.buffers:
                m.buffers[name] = Buffer(name, m.shape(name), "input")
            base = self.param(name)
            flat = self.gflat(name, idx)
        return base, flat

    def gbase(self, name: str) -> str:
        """Pointer register of an unpacked global buffer (registers it as a parameter)."""
        m = self.m
        if name not in m.live and name not in m.buffers:
            m.buffers[name] = Buffer(name, m.shape(name), "input")
        return self.param(name)

    def gload_at(self, ptr: str, off: Aff, const: int, guard) -> str:
        """Load element `ptr + off + const` (off: runtime element offset)."""
        g = self.g
        key = ("gld@", ptr, off.key(), const, guard)
        hit = g.cached(key)
        if hit:
            return hit
        if off.terms:
            k2 = ("gptr@", ptr, off.key())
            rb = g.cached(k2)
            if rb is None:
                o = g.aff(off.runtime())
                w = g.new("%rd")
                g(f"mul.wide.s32 {w}, {o}, {g.esz};")
                rb = g.new("%rd")
                g(f"add.s64 {rb}, {ptr}, {w};")
                g.remember(k2, rb)
        else:
            rb = ptr
        f = g.new(g.fr)
        pred = f"@{guard} " if guard else ""
        if guard:
            g(f"mov.b{32 if g.ft == 'f32' else 64} {f}, 0;")
        g(f"{pred}ld.global.nc.{g.ft} {f}, [{rb}+{const * g.esz}];")
        return g.remember(key, f)

    def gstore(self, name: str, idx: list, val: str) -> None:
        g = self.g
        base = self.param(name)
        self.writes.add(name)
        flat = self.gflat(name, idx)
        rb, imm = g.gaddr(base, flat)
        if not self.vec_stores or g.ft != "f32":
            pred = f"@{self.store_guard} " if self.store_guard else ""
            g(f"{pred}st.global.{g.ft} [{rb}+{imm}], {val};")
            return
        # 16-byte alignment of rb holds when every runtime coefficient is a
        # multiple of 4 elements (buffers are cudaMalloc'd, 256-byte aligned)
        aligned = all(c % 4 == 0 for c in flat.runtime().terms.values())
        self.pending.append((rb, imm, val, aligned))
        self.drain_stores(False)

    def drain_stores(self, final: bool) -> None:
        """Emit pending epilogue stores, four consecutive aligned words as one
        st.global.v4 (the register tile's innermost run along the output's
        contiguous dim)."""
        g, P = self.g, self.pending
        while P:
            rb, imm, val, al = P[0]
            run = al and imm % 16 == 0
            k = 1
            while run and k < len(P) and k < 4 and P[k][0] == rb and P[k][1] == imm + 4 * k:
                k += 1
            if run and k == 4:
                g(f"st.global.v4.f32 [{rb}+{imm}], {{{', '.join(x[2] for x in P[:4])}}};")
                del P[:4]
                continue
            if run and not final and k == len(P):
                return                  # the run may still complete
            g(f"st.global.f32 [{rb}+{imm}], {val};")
            del P[0]

    # -- inline producers and readers ---------------------------------------
    def reader(self, stage, iv, override=None):
        attached_prod = {s.name for s in self.m.attached(stage.name) if self.m.reads(stage.expr, s.name)}

        def read(buf, idx, guard):
            if override is not None:
                r = override(buf, idx, guard)
                if r is not None:
                    return r
            if buf in attached_prod:
                return self.producer(buf, idx, guard)
            return self.gload(buf, idx, guard)
        return read

    def zfill_producer(self, name: str) -> bool:
        """An attached producer of the form Select(cond, Read(buf, affine), 0) — the
        padding stage — which a zero-filling cp.async can stage directly."""
        s = self.m.live.get(name)
        if s is None or s.reduce or kind(s.expr) != "Select":
            return False
        e = s.expr
        return (kind(e.then) == "Read" and kind(e.other) == "Const" and float(e.other.value) == 0.0
                and not list(reads(e.cond)) and e.then.buffer not in self.m.live
                and self.m.layouts.get(e.then.buffer) is None)

    def zfill_source(self, name: str, idx: list) -> tuple:
        """(64-bit address register, byte immediate, predicate) of a zero-fill
        producer's element: the Read's element when the condition holds, else
        the buffer base (a valid address that is never read: src-size 0)."""
        g = self.g
        s = self.m.live[name]
        env = {n: a for (n, _), a in zip(s.space, idx)}
        ex = Expr(g, lambda n: env[n], None)
        p = ex.pred(s.expr.cond)
        if p is None:
            c = ex(s.expr.cond)
            p = g.new("%p")
            g(f"setp.ne.{g.ft} {p}, {c}, {g.fconst(0.0)};")
        rd = s.expr.then
        base, flat = self.gsource(rd.buffer, [ex.lin(l) for l in rd.index])
        rb, imm = g.gaddr(base, flat)
        a = g.new("%rd")
        g(f"add.s64 {a}, {rb}, {imm};")
        sel = g.new("%rd")
        g(f"selp.b64 {sel}, {a}, {base}, {p};")
        return sel, 0, p

    def producer(self, name: str, idx: list, guard) -> str:
        g = self.g
        s = self.m.live[name]
        env = {n: a for (n, _), a in zip(s.space, idx)}
        body = s.expr.body if kind(s.expr) == "Reduce" else s.expr
        if not s.reduce:
            ex = Expr(g, lambda n: env[n], self.reader(s, lambda n: env[n]))
            ex.guard = guard
            return ex(body)
        # reducing producer: serial loops, fully unrolled when small
        op = s.expr.op
        acc = g.new(g.fr)
        g(f"mov.{'b32' if g.ft == 'f32' else 'b64'} {acc}, {g.fconst(0.0 if op == 'sum' else -math.inf)};")
        red = list(s.reduce)

        def rec(i, env):
            nonlocal acc
            if i == len(red):
                ex = Expr(g, lambda n: env[n], self.reader(s, lambda n: env[n]))
                ex.guard = guard
                v = ex(body)
                na = g.new(g.fr)
                g(f"{'add.rn' if op == 'sum' else 'max'}.{g.ft} {na}, {acc}, {v};")
                g(f"mov.{'b32' if g.ft == 'f32' else 'b64'} {acc}, {na};")
                return
            n, e = red[i]
            self.loop(e, False, lambda r: rec(i + 1, {**env, n: r}))
        rec(0, env)
        return acc

    # -- loops ----------------------------------------------------------------
    def loop(self, extent: int, unroll: bool, body) -> None:
        """Counted loop: unrolled -> body(Aff.k(i)) per i; else a PTX loop."""
        g = self.g
        if extent == 1:
            body(Aff.k(0))
            return
        if unroll:
            for i in range(extent):
                body(Aff.k(i))
            return
        v = g.new("%r")
        lab = g.new_label()
        g(f"mov.s32 {v}, 0;")
        g.label(lab)
        g(".pragma \"nounroll\";")
        g.push()
        body(Aff.reg(v))
        g.pop()
        p = g.new("%p")
        g(f"add.s32 {v}, {v}, 1;")
        g(f"setp.lt.s32 {p}, {v}, {extent};")
        g(f"@{p} bra {lab};")

    # -- epilogue -------------------------------------------------------------
    def epilogue(self, host, idx_of: dict, value: str, materialize: bool) -> None:
        g = self.g
        space = [n for n, _ in host.space]
        if materialize:
            self.gstore(host.name, [idx_of[n] for n in space], value)
        for c in self.m.attached(host.name):
            if not self.m.reads(c.expr, host.name) or self.m.reads(host.expr, c.name):
                continue
            cspace = [n for n, _ in c.space]
            if len(cspace) != len(space) or c.reduce:
                raise LoweringError(f"consumer {c.name} cannot be fused")
            cenv = {cn: idx_of[hn] for cn, hn in zip(cspace, space)}

            def ov(buf, idx, guard, host=host, cspace=cspace):
                if buf == host.name:
                    want = [cenv[n] for n in cspace]
                    if all(a.key() == b.key() and a.const == b.const for a, b in zip(idx, want)):
                        return value
                    raise LoweringError(f"consumer {c.name} reads {host.name} at a non-identity index")
                return None
            ex = Expr(g, lambda n: cenv[n], self.reader(c, lambda n: cenv[n], override=ov))
            ex.guard = self.store_guard
            v = ex(c.expr)
            self.epilogue(c, {n: cenv[n] for n in cspace}, v, True)

    def text(self) -> str:
        g = self.g
        ps = ", ".join(f".param .u64 p{i}" for i in range(len(self.params)))
        head = [f".visible .entry {self.entry}({ps}) .maxntid {self.threads}, 1, 1", "{"]
        decl = [f"  .reg .b32 %r<{g.n['%r'] + 1}>;", f"  .reg .b64 %rd<{g.n['%rd'] + 1}>;",
                f"  .reg .pred %p<{g.n['%p'] + 1}>;",
                f"  .reg .{g.ft} {g.fr}<{g.n[g.fr] + 1}>;",
                f"  .reg .b64 %ptr<{len(self.params) + 1}>;"]
        loads = []
        for i, _ in enumerate(self.params):
            loads.append(f"  ld.param.u64 %ptr{i + 1}, [p{i}];")
            loads.append(f"  cvta.to.global.u64 %ptr{i + 1}, %ptr{i + 1};")
        return "\n".join(head + decl + self.body + loads + g.lines + ["  ret;", "}"]) + "\n"


# output points per thread per grid-stride step.  4 was measured on the golden
# streams (tools/template_bench.py) with no gain over 1 (naive kernels are not
# bound by loads in flight) and costs PTX size, i.e. compile time: 1.
NAIVE_POINTS = int(os.environ.get("LT_NAIVE_POINTS", "1"))


def _dec(g: Ptx, d, lv: dict) -> Aff:
    """A decode AST (src/ir.py:73-93) over loop values `lv` as an Aff."""
    kk = kind(d)
    if kk == "DVar":
        return lv[d.loop]
    if kk == "DConst":
        return Aff.k(d.value)
    if kk == "DAdd":
        return _dec(g, d.a, lv) + _dec(g, d.b, lv)
    a = _dec(g, d.a, lv)
    if kk == "DMul":
        return a.scale(d.c)
    r = g.aff(a)
    return Aff.reg(g.udiv(r, d.c) if kk == "DDiv" else g.urem(r, d.c))


def _quad_read(mod: _Mod, s):
    """The elementwise stages the naive template moves four points at a time
    (16-byte loads and stores): no reduction; the innermost loop is the output's
    innermost iterator itself (identity decode), its extent a multiple of 4; the
    body is `Read(buf, idx)` or `Select(cond, Read(buf, idx), 0)` — a copy, or
    the padding stage — where only idx's innermost dim uses that iterator
    (coefficient 1, constant a multiple of 4, an unpacked buffer whose innermost
    extent is a multiple of 4) and cond does not use it.  Returns (iterator,
    Read, Select or None) or None."""
    if s.reduce or mod.dtype != "float" or "nquad" in _OFF:
        return None
    sp = [l for l in s.loops if l.kind == "space"]
    if not sp or sp[-1].extent % 4:
        return None
    last = sp[-1]
    space = [n for n, _ in s.space]
    dmap = dict(s.index_map)
    n_last = space[-1]
    d = dmap.get(n_last)
    if d is None or kind(d) != "DVar" or d.loop != last.id or s.space[-1][1] % 4:
        return None

    def uses(d2):
        k2 = kind(d2)
        if k2 == "DVar":
            return d2.loop == last.id
        if k2 == "DConst":
            return False
        if k2 == "DAdd":
            return uses(d2.a) or uses(d2.b)
        return uses(d2.a)
    if any(uses(dmap[n]) for n in space[:-1] if n in dmap):
        return None
    e = s.expr
    sel = None
    if kind(e) == "Select":
        if kind(e.other) != "Const" or float(e.other.value) != 0.0:
            return None
        sel, e = e, e.then
        if any(n_last in lin_iters(x) for x in _itervals(sel.cond)) or list(reads(sel.cond)):
            return None
    if kind(e) != "Read":
        return None
    buf = e.buffer
    if buf in mod.layouts and buf not in mod.live:
        return None
    if any(c.name == buf for c in mod.attached(s.name)):       # an inline producer, not in memory
        return None
    shape = mod.shape(buf)
    if shape[-1] % 4:
        return None
    for j, lin in enumerate(e.index):
        c = dict(lin.terms).get(n_last, 0)
        if j < len(e.index) - 1:
            if c:
                return None
        elif c != 1 or lin.const % 4 or any(n != n_last and cc % 4 for n, cc in lin.terms):
            return None
    return n_last, e, sel


def _itervals(e):
    k = kind(e)
    if k == "IterVal":
        yield e.lin
    elif k == "Bin":
        yield from _itervals(e.lhs)
        yield from _itervals(e.rhs)
    elif k in ("Call",):
        yield from _itervals(e.arg)
    elif k == "Select":
        yield from _itervals(e.cond)
        yield from _itervals(e.then)
        yield from _itervals(e.other)


def lin_iters(lin) -> set:
    return {n for n, _ in lin.terms}


def _naive_quad(mod: _Mod, s, entry: str, plan) -> tuple:
    """`_naive` for the elementwise stages `_quad_read` accepts: a thread step
    covers four consecutive innermost points with one 16-byte load (predicated
    by the padding condition, zero-filled otherwise) and one 16-byte store."""
    n_last, rd, sel = plan
    k = _Kern(mod, entry, NAIVE_THREADS)
    g = k.g
    sp_loops = [l for l in s.loops if l.kind == "space"]
    exts = [l.extent for l in sp_loops[:-1]] + [sp_loops[-1].extent // 4]
    total = 1
    for x in exts:
        total *= x
    if 4 * total + 148 * 16 * NAIVE_THREADS >= (1 << 31):
        raise Unsupported("index space exceeds 2^31")
    grid = max(1, min((total + NAIVE_THREADS - 1) // NAIVE_THREADS, 148 * 16))
    step = grid * NAIVE_THREADS
    dmap = dict(s.index_map)
    space_names = [n for n, _ in s.space]
    tid, cta, pidx = g.new("%r"), g.new("%r"), g.new("%r")
    g(f"mov.u32 {tid}, %tid.x;")
    g(f"mov.u32 {cta}, %ctaid.x;")
    g(f"mad.lo.s32 {pidx}, {cta}, {NAIVE_THREADS}, {tid};")
    top, done = g.new_label(), g.new_label()
    pe = g.new("%p")
    g(f"setp.ge.s32 {pe}, {pidx}, {total};")
    g(f"@{pe} bra {done};")
    g.label(top)
    g.push()
    digits = g.decompose(pidx, exts)
    lv = {l.id: Aff.reg(dg) for l, dg in zip(sp_loops, digits)}
    lv[sp_loops[-1].id] = Aff.reg(digits[-1], 4)
    env = {n: _dec(g, dmap[n], lv) for n in space_names if n in dmap}
    ex = Expr(g, lambda n: env[n], None)
    pred = None
    if sel is not None:
        pred = ex.pred(sel.cond)
        if pred is None:
            c = ex(sel.cond)
            pred = g.new("%p")
            g(f"setp.ne.{g.ft} {pred}, {c}, {g.fconst(0.0)};")
    base, flat = k.gsource(rd.buffer, [ex.lin(l) for l in rd.index])
    rb, imm = g.gaddr(base, flat)
    vals = [g.new(g.fr) for _ in range(4)]
    if pred is not None:
        for v in vals:
            g(f"mov.b32 {v}, 0;")
    g(f"{'@' + pred + ' ' if pred else ''}ld.global.nc.v4.f32 {{{', '.join(vals)}}}, [{rb}+{imm}];")
    k.vec_stores = True
    for u, v in enumerate(vals):
        k.epilogue(s, {n: (env[n] + u if n == n_last else env[n]) for n in space_names}, v,
                   mod.must_materialize(s))
    k.drain_stores(True)
    k.vec_stores = False
    g.pop()
    g(f"add.s32 {pidx}, {pidx}, {step};")
    g(f"setp.lt.s32 {pe}, {pidx}, {total};")
    g(f"@{pe} bra {top};")
    g.label(done)
    args = _args(k, mod, s)
    return k, Kernel(entry, grid, NAIVE_THREADS, 0, args, {"template": "naive", "stage": s.name, "points": 4 * total,
                                                            "points_per_thread_step": 4, "vector": 4})


def _naive(mod: _Mod, s, entry: str) -> tuple:
    """One output point per thread-iteration (the State's own loops and decode
    maps, reductions serial), NAIVE_POINTS points per grid-stride step so each
    thread keeps several independent loads / accumulation chains in flight."""
    plan = _quad_read(mod, s) if NAIVE_POINTS == 1 else None
    if plan is not None:
        return _naive_quad(mod, s, entry, plan)
    k = _Kern(mod, entry, NAIVE_THREADS)
    g = k.g
    sp_loops = [l for l in s.loops if l.kind == "space"]
    rd_loops = [l for l in s.loops if l.kind != "space"]
    total = 1
    for l in sp_loops:
        total *= l.extent
    U = max(1, NAIVE_POINTS)
    if total + U * 148 * 16 * NAIVE_THREADS >= (1 << 31):
        raise Unsupported("index space exceeds 2^31")
    grid = max(1, min((total + NAIVE_THREADS * U - 1) // (NAIVE_THREADS * U), 148 * 16))
    step = grid * NAIVE_THREADS
    dmap = dict(s.index_map)
    space_names = [n for n, _ in s.space]
    tid, cta, pidx = g.new("%r"), g.new("%r"), g.new("%r")
    g(f"mov.u32 {tid}, %tid.x;")
    g(f"mov.u32 {cta}, %ctaid.x;")
    g(f"mad.lo.s32 {pidx}, {cta}, {NAIVE_THREADS}, {tid};")
    top, done = g.new_label(), g.new_label()
    pe = g.new("%p")
    g(f"setp.ge.s32 {pe}, {pidx}, {total};")
    g(f"@{pe} bra {done};")
    g.label(top)
    g.push()

    def dec(d, lv):
        return _dec(g, d, lv)

    # per point u: index, guard (u = 0 is in range inside the loop), decoded space env
    pts = []
    for u in range(U):
        if u == 0:
            pu, guard = pidx, None
        else:
            pu = g.new("%r")
            g(f"add.s32 {pu}, {pidx}, {u * step};")
            guard = g.new("%p")
            g(f"setp.lt.s32 {guard}, {pu}, {total};")
        lv = {}
        digits = g.decompose(pu, [l.extent for l in sp_loops]) if sp_loops else []
        for l, d in zip(sp_loops, digits):
            lv[l.id] = Aff.reg(d)
        pts.append((guard, lv, {n: dec(dmap[n], lv) for n in space_names if n in dmap}))

    values = []
    if rd_loops:
        op = s.expr.op
        flags = _unroll_flags([l.extent for l in rd_loops], s.pragma_unroll)
        mv = "b32" if g.ft == "f32" else "b64"
        accs = []
        for _ in range(U):
            acc = g.new(g.fr)
            g(f"mov.{mv} {acc}, {g.fconst(0.0 if op == 'sum' else -math.inf)};")
            accs.append(acc)
        body = s.expr.body

        def rec(i, rlv):
            if i == len(rd_loops):
                for (guard, lv, env), acc in zip(pts, accs):
                    env2 = dict(env)
                    for n, d in s.index_map:
                        if n not in space_names:
                            env2[n] = dec(d, {**lv, **rlv})
                    ex = Expr(g, lambda n, env2=env2: env2[n], k.reader(s, lambda n, env2=env2: env2[n]))
                    ex.guard = guard
                    if op == "sum" and kind(body) == "Bin" and body.op == "mul":
                        a_, b_ = ex(body.lhs), ex(body.rhs)
                        g(f"fma.rn.{g.ft} {acc}, {a_}, {b_}, {acc};")
                    else:
                        v = ex(body)
                        g(f"{'add.rn' if op == 'sum' else 'max'}.{g.ft} {acc}, {acc}, {v};")
                return
            l = rd_loops[i]
            k.loop(l.extent, flags[i], lambda r: rec(i + 1, {**rlv, l.id: r}))
        rec(0, {})
        values = accs
    else:
        expr = s.expr.body if kind(s.expr) == "Reduce" else s.expr
        for guard, lv, env in pts:
            ex = Expr(g, lambda n, env=env: env[n], k.reader(s, lambda n, env=env: env[n]))
            ex.guard = guard
            values.append(ex(expr))
    for (guard, lv, env), value in zip(pts, values):
        k.store_guard = guard
        k.epilogue(s, {n: env[n] for n in space_names}, value, mod.must_materialize(s))
    k.store_guard = None
    g.pop()
    g(f"add.s32 {pidx}, {pidx}, {U * step};")
    g(f"setp.lt.s32 {pe}, {pidx}, {total};")
    g(f"@{pe} bra {top};")
    g.label(done)
    args = _args(k, mod, s)
    return k, Kernel(entry, grid, NAIVE_THREADS, 0, args, {"template": "naive", "stage": s.name, "points": total,
                                                            "points_per_thread_step": U})


XREDUCE_MAX_THREADS = 1024


def _xreduce_pairs(mod: _Mod) -> dict:
    """{partial stage: final stage} for every rule-6 pair (ReductionFactorization,
    `src/sketch.py:307-329`; `_apply_rfactor` `src/ir.py:667-722`) that lowers as
    ONE cross-thread reduction kernel: the final stage reduces `X.rf` over `rf`
    exactly as `_apply_rfactor` builds it, the partial is read by nothing else,
    neither stage is attached, and the partial's space loops enumerate
    (rf, space...) in row-major order (checked on sample points, so a State
    whose loops were reordered keeps the two-kernel naive lowering)."""
    from .state import Lin
    from .state import d_eval, d_vars
    if "xreduce" in _OFF:
        return {}
    p, out = mod.p, {}
    for F in p.stages:
        P = mod.live.get(F.name + ".rf")
        if F.inlined or F.compute_at is not None or P is None or P.compute_at is not None:
            continue
        e, pe = F.expr, P.expr
        if kind(e) != "Reduce" or kind(pe) != "Reduce" or e.op not in ("sum", "max") or pe.op != e.op:
            continue
        if not P.space or len(F.reduce) != 1 or F.reduce[0] != P.space[0] or tuple(P.space[1:]) != tuple(F.space):
            continue
        rf = P.space[0][0]
        want = (Lin.var(rf),) + tuple(Lin.var(n) for n, _ in F.space)
        if kind(e.body) != "Read" or e.body.buffer != P.name or tuple(e.body.index) != want:
            continue
        if P.name in p.dag.outputs or any(st.name != F.name and mod.reads(st.expr, P.name)
                                          for st in mod.live.values()):
            continue
        if any(not mod.reads(P.expr, c.name) for c in mod.attached(P.name)):
            continue
        if any(not mod.reads(c.expr, F.name) for c in mod.attached(F.name)):
            continue
        sp = [l for l in P.loops if l.kind == "space"]
        ext = [l.extent for l in sp]
        total = int(np.prod(ext)) if ext else 1
        names = [n for n, _ in P.space]
        dims = [x for _, x in P.space]
        dmap = dict(P.index_map)
        sp_ids = {l.id for l in sp}
        if total != int(np.prod(dims)) or any(n not in dmap or not d_vars(dmap[n]) <= sp_ids for n in names):
            continue
        rng = np.random.default_rng(0)
        qs = set(range(min(total, 64))) | set(range(max(0, total - 64), total))
        qs |= set(int(x) for x in rng.integers(0, total, 128))
        ok = True
        for q in sorted(qs):
            env, r = {}, q
            for l in reversed(sp):
                env[l.id] = r % l.extent
                r //= l.extent
            r = q
            for n, x in zip(reversed(names), reversed(dims)):
                if d_eval(dmap[n], env) != r % x:
                    ok = False
                    break
                r //= x
            if not ok:
                break
        if ok:
            out[P.name] = F
    return out


def _xreduce(mod: _Mod, P, F, entry: str) -> tuple:
    """A rule-6 pair as one cross-thread reduction (the GPU lowering of rfactor:
    rf -> threadIdx.x).  One block per output point of the final stage
    (grid-stride), thread t owns rf = t, t+T, ... and runs the partial stage's
    own reduction loops serially over rk; the block then combines the partials
    with warp shuffles and one shared-memory round, and thread 0 writes the point
    (with the final stage's fused consumers).  The partial buffer never exists."""
    f = P.space[0][1]
    S = 1
    for _, x in F.space:
        S *= x
    if f * S >= (1 << 31):
        raise Unsupported("index space exceeds 2^31")
    T = min(XREDUCE_MAX_THREADS, -(-f // 32) * 32)
    n_it = -(-f // T)
    grid = max(1, min(S, 148 * 16))
    k = _Kern(mod, entry, T)
    g = k.g
    op = F.expr.op
    mv = "b32" if g.ft == "f32" else "b64"
    ident = g.fconst(0.0 if op == "sum" else -math.inf)
    comb = "add.rn" if op == "sum" else "max"
    sp_loops = [l for l in P.loops if l.kind == "space"]
    rd_loops = [l for l in P.loops if l.kind != "space"]
    dmap = dict(P.index_map)
    pnames = [n for n, _ in P.space]
    body = P.expr.body
    flags = _unroll_flags([l.extent for l in rd_loops], P.pragma_unroll)
    tid, sidx = g.new("%r"), g.new("%r")
    g(f"mov.u32 {tid}, %tid.x;")
    g(f"mov.u32 {sidx}, %ctaid.x;")
    n_warp = T // 32
    if n_warp > 1:
        lane, warp, sm = g.new("%r"), g.new("%r"), g.new("%r")
        g(f"and.b32 {lane}, {tid}, 31;")
        g(f"shr.u32 {warp}, {tid}, 5;")
        g(f"mov.u32 {sm}, smem_;")
        wa, ra = g.new("%r"), g.new("%r")
        g(f"mad.lo.s32 {wa}, {warp}, {g.esz}, {sm};")
        g(f"mad.lo.s32 {ra}, {tid}, {g.esz}, {sm};")
        pl0, pin = g.new("%p"), g.new("%p")
        g(f"setp.eq.s32 {pl0}, {lane}, 0;")
        g(f"setp.lt.s32 {pin}, {tid}, {n_warp};")
    p0 = g.new("%p")
    g(f"setp.eq.s32 {p0}, {tid}, 0;")
    top = g.new_label()
    g.label(top)
    g.push()
    acc = g.new(g.fr)
    g(f"mov.{mv} {acc}, {ident};")

    def one_rf(r: Aff) -> None:
        guard = None
        if f % T:
            rr = g.aff(r)
            guard = g.new("%p")
            g(f"setp.lt.s32 {guard}, {rr}, {f};")
        q = g.aff(r.scale(S) + Aff.reg(sidx))
        digits = g.decompose(q, [l.extent for l in sp_loops]) if sp_loops else []
        lv = {l.id: Aff.reg(d) for l, d in zip(sp_loops, digits)}
        env = {n: _dec(g, dmap[n], lv) for n in pnames}
        pacc = g.new(g.fr)
        g(f"mov.{mv} {pacc}, {ident};")

        def rec(i, rlv):
            if i == len(rd_loops):
                env2 = dict(env)
                for n, d in P.index_map:
                    if n not in pnames:
                        env2[n] = _dec(g, d, {**lv, **rlv})
                ex = Expr(g, lambda n: env2[n], k.reader(P, lambda n: env2[n]))
                ex.guard = guard
                if op == "sum" and kind(body) == "Bin" and body.op == "mul":
                    a_, b_ = ex(body.lhs), ex(body.rhs)
                    g(f"fma.rn.{g.ft} {pacc}, {a_}, {b_}, {pacc};")
                else:
                    g(f"{comb}.{g.ft} {pacc}, {pacc}, {ex(body)};")
                return
            l = rd_loops[i]
            k.loop(l.extent, flags[i], lambda v: rec(i + 1, {**rlv, l.id: v}))
        rec(0, {})
        if guard is not None:
            g(f"selp.{mv} {pacc}, {pacc}, {ident}, {guard};")
        g(f"{comb}.{g.ft} {acc}, {acc}, {pacc};")

    if n_it == 1:
        one_rf(Aff.reg(tid))
    else:
        k.loop(n_it, False, lambda i: one_rf(Aff.reg(tid) + i.scale(T)))

    def warp_reduce(v: str) -> None:
        for off in (16, 8, 4, 2, 1):
            t = g.new(g.fr)
            if g.ft == "f32":
                g(f"shfl.sync.bfly.b32 {t}, {v}, {off}, 31, -1;")
            else:
                lo, hi, lo2, hi2 = (g.new("%r") for _ in range(4))
                g(f"mov.b64 {{{lo}, {hi}}}, {v};")
                g(f"shfl.sync.bfly.b32 {lo2}, {lo}, {off}, 31, -1;")
                g(f"shfl.sync.bfly.b32 {hi2}, {hi}, {off}, 31, -1;")
                g(f"mov.b64 {t}, {{{lo2}, {hi2}}};")
            g(f"{comb}.{g.ft} {v}, {v}, {t};")

    warp_reduce(acc)
    if n_warp > 1:
        g(f"@{pl0} st.shared.{g.ft} [{wa}], {acc};")
        g("bar.sync 0;")
        g(f"mov.{mv} {acc}, {ident};")
        g(f"@{pin} ld.shared.{g.ft} {acc}, [{ra}];")
        warp_reduce(acc)
    k.store_guard = p0
    fdig = g.decompose(sidx, [x for _, x in F.space]) if F.space else []
    k.epilogue(F, {n: Aff.reg(d) for (n, _), d in zip(F.space, fdig)}, acc, mod.must_materialize(F))
    k.store_guard = None
    g.pop()
    if grid < S:
        if n_warp > 1:
            g("bar.sync 0;")                    # the next point reuses the shared slots
        pe = g.new("%p")
        g(f"add.s32 {sidx}, {sidx}, {grid};")
        g(f"setp.lt.s32 {pe}, {sidx}, {S};")
        g(f"@{pe} bra {top};")
    smem = n_warp * g.esz if n_warp > 1 else 0
    return k, Kernel(entry, grid, T, smem, _args(k, mod, F),
                     {"template": "xreduce", "stage": F.name, "partial": P.name, "points": S, "rf": f,
                      "threads": T, "rf_per_thread": n_it})


def _args(k: _Kern, mod: _Mod, s) -> list:
    return list(k.params)


def _bank_degree(coord_sets, st) -> int:
    """Worst number of distinct words one shared-memory bank serves for the
    warp's accesses (coordinates: one row per lane)."""
    if coord_sets is None or len(coord_sets) == 0:
        return 1
    addr = np.unique(np.asarray(coord_sets, np.int64) @ np.asarray(st, np.int64))
    return int(np.bincount(addr % 32, minlength=32).max())


def _smem_strides(hull: list, lane_coords, order=None, step: int = 1, store_coords=None) -> tuple:
    """Strides (indexed by hull dim) of a staged tile laid out in `order`
    (outer->inner), innermost dim padded by a multiple of `step` to minimise
    shared-memory bank conflicts of the warp's first compute-side access, then
    of the cooperative fetch's stores (`store_coords`: the tile coordinates the
    warp's lanes store in one fetch instruction)."""
    order = list(range(len(hull))) if order is None else order
    best = None
    for pad in range(0, 33, step):
        st = [0] * len(hull)
        m = 1
        for j, d in enumerate(reversed(order)):
            st[d] = m
            m *= hull[d] + (pad if j == 0 else 0)
        deg = _bank_degree(lane_coords, st)
        sdeg = _bank_degree(store_coords, st) if store_coords else 1
        cand = (deg, sdeg, m, pad)
        if best is None or cand < best[0]:
            best = (cand, st, m)
        if deg == 1 and sdeg == 1:
            break
    return best[1], best[2], best[0][0]


def _tiled(mod: _Mod, s, levels, entry: str) -> tuple:
    structure, factors = levels
    space = [n for n, _ in s.space]
    red = [n for n, _ in s.reduce]
    block, vthread, thread, stage_lv, inner = _binding(structure)
    if not stage_lv:
        raise LoweringError("tiled stage has no reduction level to stage")

    def f(a, lv):
        return factors[a][lv[1]]

    def axes_of(lv):
        return space if lv[0] == "S" else red

    n_threads = n_blocks = n_vt = 1
    for a in space:
        for lv in thread:
            n_threads *= f(a, lv)
        for lv in block:
            n_blocks *= f(a, lv)
        for lv in vthread:
            n_vt *= f(a, lv)
    if n_threads > MAX_THREADS:
        raise LoweringError(f"{n_threads} threads per block exceed {MAX_THREADS}")
    if n_vt > MAX_VTHREAD:
        raise LoweringError(f"{n_vt} virtual threads exceed {MAX_VTHREAD}")
    reg_levels = vthread + [lv for lv in inner if lv[0] == "S"]
    acc_dims = []
    for a in space:
        n = 1
        for lv in reg_levels:
            n *= f(a, lv)
        acc_dims.append(n)
    n_acc = 1
    for n in acc_dims:
        n_acc *= n
    if n_acc > MAX_ACC:
        raise LoweringError(f"register tile of {n_acc} accumulators per thread exceeds {MAX_ACC}")
    n_s, n_r = structure.count("S"), structure.count("R")
    T = {}
    for a in space:
        t = 1
        for k_ in range(1, n_s):
            t *= factors[a][k_]
        T[a] = t
    RT = {}
    for r in red:
        t = 1
        for k_ in range(1, n_r):
            t *= factors[r][k_]
        RT[r] = t

    k = _Kern(mod, entry, n_threads)
    g = k.g
    tid, cta = g.new("%r"), g.new("%r")
    g(f"mov.u32 {tid}, %tid.x;")
    g(f"mov.u32 {cta}, %ctaid.x;")
    dig: dict = {}                    # (axis, level tag) -> Aff
    blk = [(a, lv) for a in space for lv in block if f(a, lv) > 1]
    for (a, lv), d in zip(blk, g.decompose(cta, [f(a, lv) for a, lv in blk]) if blk else []):
        dig[(a, lv)] = Aff.reg(d)
    thr = [(a, lv) for a in space for lv in thread if f(a, lv) > 1]
    thr_regs = g.decompose(tid, [f(a, lv) for a, lv in thr]) if thr else []
    for (a, lv), d in zip(thr, thr_regs):
        dig[(a, lv)] = Aff.reg(d)

    def digit(a, lv):
        return dig.get((a, lv), Aff.k(0))

    def mixed(a, kind_, lo, dg):
        n_lv = n_s if kind_ == "S" else n_r
        e = Aff.k(0)
        for kk in range(lo, n_lv):
            e = e.scale(factors[a][kk]) + dg(a, (kind_, kk))
        return e

    # operands: distinct reads of the reduction body, staged per R0 step
    body = s.expr.body
    operands = []
    for r in reads(body):
        key = (r.buffer, tuple((l.terms, l.const) for l in r.index))
        if key not in [o["key"] for o in operands]:
            operands.append({"key": key, "read": r})
    attached_prod = {c.name for c in mod.attached(s.name) if mod.reads(s.expr, c.name)}
    span = {**T, **RT}
    for o in operands:
        hull, off = [], []
        for lin in o["read"].index:
            h, of = 1, 0
            for n, c in lin.terms:
                if n not in span:
                    raise LoweringError(f"read index uses iterator {n} outside the stage")
                h += abs(c) * (span[n] - 1)
                if c < 0:
                    of += -c * (span[n] - 1)
            hull.append(h)
            off.append(of)
        o["hull"], o["off"] = hull, off
        size = 1
        for h in hull:
            size *= h
        o["size"] = size

    # loop list of the per-thread nest
    loop_list = []
    for lv in vthread:
        for a in space:
            if f(a, lv) > 1:
                loop_list.append((a, lv, f(a, lv), True))
    for lv in inner:
        for a in axes_of(lv):
            if f(a, lv) > 1:
                loop_list.append((a, lv, f(a, lv), False))
    free = [x for x in loop_list if not x[3]]
    flags = _unroll_flags([x[2] for x in free], s.pragma_unroll)
    it = iter(flags)
    unroll = [True if x[3] else next(it) for x in loop_list]
    unrolled = 1
    for x, u in zip(loop_list, unroll):
        if u:
            unrolled *= x[2]
    if unrolled > MAX_UNROLLED:
        raise LoweringError(f"unrolled body of {unrolled} statements exceeds {MAX_UNROLLED}")
    if "promote" not in _OFF:
        unroll = promote_register_tile([x[2] for x in loop_list], unroll, [x[1][0] == "S" for x in loop_list],
                                       n_acc, n_threads)
    # the accumulator tile is indexed only by space-level digits: it stays in
    # registers whenever those loops are unrolled (rolled reduction loops are fine)
    acc_in_regs = all(u for x, u in zip(loop_list, unroll) if x[1][0] == "S")
    tile_spills = n_acc + SPILL_MARGIN > min(255, 65536 // n_threads)
    if acc_in_regs and "hoist" not in _OFF and (not tile_spills or unrolled <= HOIST_SPILL_UNROLLED):
        # register tile in registers: every space loop is unrolled, so the thread's
        # nest is issued reduction loops first (their relative order kept, hence
        # every accumulator's summation order is unchanged) and the whole tile
        # innermost — TVM's virtual-thread injection does the same for vthreads.
        # Each reduction step then loads its operands once for all accumulators
        # instead of once per vthread / S3 copy around a rolled reduction loop.
        # A tile that overflows the register file keeps the State's order unless
        # its reduction is mostly rolled: sweeping all accumulators every step
        # multiplies its spill traffic (template_bench A/B, 128 States per config).
        perm = ([i for i, x in enumerate(loop_list) if x[1][0] == "R"]
                + [i for i, x in enumerate(loop_list) if x[1][0] != "R"])
        loop_list = [loop_list[i] for i in perm]
        unroll = [unroll[i] for i in perm]

    # smem layout: pad each operand's innermost dim against the warp's bank pattern
    lanes = min(32, n_threads)
    lane_digits = []
    for ln in range(lanes):
        x, dd = ln, {}
        for (a, lv) in reversed(thr):
            dd[(a, lv)] = x % f(a, lv)
            x //= f(a, lv)
        lane_digits.append(dd)
    plain = sum(o["size"] for o in operands) * g.esz
    if plain > MAX_SMEM:
        raise LoweringError(f"shared memory {plain} bytes exceeds {MAX_SMEM}")
    # contiguous register runs: per space axis, the trailing inner register levels
    # (S3 S4 for SSSRRSRS) are adjacent digits of the axis's mixed radix, so a
    # thread's values along them are unit-stride when that dim is laid out
    # innermost -> vector shared loads of up to 4 words
    run_lvs = [lv for lv in inner if lv[0] == "S"]
    if "vrun" in _OFF:
        run_lvs = run_lvs[-1:]

    def run_len(n):
        r = 1
        for lv in run_lvs:
            r *= f(n, lv)
        return r
    def others_aligned(lin, n, w):
        """Every other iterator digit in this index dim moves by a multiple of w
        words when the dim is laid out innermost (else the runs would straddle
        vector boundaries and the layout change would buy nothing)."""
        for n2, c2 in lin.terms:
            if n2 == n:
                continue
            kind_ = "S" if n2 in T else "R"
            for kk in range(1, n_s if kind_ == "S" else n_r):
                if f(n2, (kind_, kk)) > 1:
                    m = 1
                    for k2 in range(kk + 1, n_s if kind_ == "S" else n_r):
                        m *= factors[n2][k2]
                    if (c2 * m) % w:
                        return False
        return True
    for o in operands:
        o["vec"], o["order"] = 1, list(range(len(o["hull"])))
        if not run_lvs:
            continue
        for di, lin in enumerate(o["read"].index):
            for n, cc in lin.terms:
                if n in T and cc == 1 and run_len(n) > 1 and o["off"][di] % 4 == 0 and \
                        sum(1 for l2 in o["read"].index for n2, _ in l2.terms if n2 == n) == 1:
                    w = 4 if run_len(n) % 4 == 0 else (2 if run_len(n) % 2 == 0 else 1)
                    if w > o["vec"] and others_aligned(lin, n, w):
                        o["vec"], o["vaxis"] = w, n
                        o["order"] = [d for d in range(len(o["hull"])) if d != di] + [di]
    total_words = 0
    for o in operands:
        coords = []
        for dd in lane_digits:
            c = []
            for di, lin in enumerate(o["read"].index):
                v = o["off"][di]
                for n, cc in lin.terms:
                    if n in T:
                        loc = 0
                        for kk in range(1, n_s):
                            loc = loc * factors[n][kk] + dd.get((n, ("S", kk)), 0)
                        v += cc * loc
                c.append(v)
            coords.append(c)
        scoords = []
        for ln in range(lanes):
            c, x = [], ln
            for h in reversed(o["hull"]):
                c.append(x % h)
                x //= h
            if x == 0:
                scoords.append(c[::-1])
        sc_ = None if "pad" in _OFF else scoords
        o["stride"], o["words"], deg = _smem_strides(o["hull"], coords, o["order"], o["vec"], sc_)
        if o["vec"] > 1:
            # a vector layout is kept only if its compute-side wavefronts per
            # element (conflict degree / vector width) beat the natural layout's
            st1, w1, deg1 = _smem_strides(o["hull"], coords, list(range(len(o["hull"]))), 1, sc_)
            if deg1 < deg / o["vec"] or (deg1 == deg / o["vec"] and w1 < o["words"]):
                o["stride"], o["words"], o["vec"] = st1, w1, 1
                o["order"] = list(range(len(o["hull"])))
        total_words = -(-total_words // 4) * 4          # 16-byte aligned operand bases
        o["base_word"] = total_words
        total_words += o["words"]
    if total_words * g.esz > MAX_SMEM:          # padding must not change legality: drop it
        total_words = 0
        for o in operands:
            st, m = [], 1
            for h in reversed(o["hull"]):
                st.append(m)
                m *= h
            o["stride"], o["words"], o["base_word"] = st[::-1], m, total_words
            o["vec"] = 1
            total_words += m
    total_words = -(-total_words // 4) * 4
    smem_bytes = total_words * g.esz
    sm = g.new("%r")
    g(f"mov.u32 {sm}, smem_;")

    # accumulators
    op = s.expr.op
    init = g.fconst(0.0 if op == "sum" else -math.inf)
    mv = "b32" if g.ft == "f32" else "b64"
    if acc_in_regs:
        acc = [g.new(g.fr) for _ in range(n_acc)]
        for r in acc:
            g(f"mov.{mv} {r}, {init};")
    else:
        k.body.append(f"  .local .align 8 .b8 accl[{n_acc * g.esz}];")
        ab = g.new("%rd")
        g(f"mov.u64 {ab}, accl;")
        iv0 = g.new("%r")
        g(f"mov.s32 {iv0}, 0;")
        lab = g.new_label()
        g.label(lab)
        w = g.new("%rd")
        g(f"mul.wide.s32 {w}, {iv0}, {g.esz};")
        a2 = g.new("%rd")
        g(f"add.s64 {a2}, {ab}, {w};")
        g(f"st.local.{g.ft} [{a2}], {init};")
        pz = g.new("%p")
        g(f"add.s32 {iv0}, {iv0}, 1;")
        g(f"setp.lt.s32 {pz}, {iv0}, {n_acc};")
        g(f"@{pz} bra {lab};")

    def acc_index(dg):
        idx = Aff.k(0)
        for ai, a in enumerate(space):
            e = Aff.k(0)
            for lv in reg_levels:
                if f(a, lv) > 1:
                    e = e.scale(f(a, lv)) + dg(a, lv)
            idx = idx.scale(acc_dims[ai]) + e
        return idx

    stage_axes = [(r, f(r, stage_lv[0])) for r in red if f(r, stage_lv[0]) > 1]

    def operand_base(o, sdig):
        base = []
        for lin in o["read"].index:
            b = Aff.k(lin.const)
            for n, c in lin.terms:
                if n in T:
                    mn = digit(n, ("S", 0)).scale(T[n])
                else:
                    mn = sdig(n).scale(RT[n])
                b = b + (mn.scale(c) if c >= 0 else (mn + (span[n] - 1)).scale(c))
            base.append(b)
        return base

    def carry_free_shifts(o, trips):
        """Per fetch trip t, the constant hull-coordinate shift with
        coords(tid + t*threads) == coords(tid) + shift for every live tid, or
        None when some tid carries across a hull digit."""
        hull = fhull(o)
        tids = np.arange(n_threads, dtype=np.int64)

        def digits(e):
            out, x = [], e.copy()
            for h in reversed(hull):
                out.append(x % h)
                x //= h
            out.append(x)             # overflow beyond the outermost dim
            return np.stack(out[::-1], axis=1)
        d0 = digits(tids)
        shifts = []
        for t in range(trips):
            e = tids + t * n_threads
            live = e < fsize(o)
            if not live.any():
                return None
            dd = digits(e)[live] - d0[live]
            if (dd != dd[0]).any() or dd[0][0] != 0:
                return None
            shifts.append([int(x) for x in dd[0][1:]])
        return shifts

    # vectorised fetch: an operand whose innermost (global-contiguous) dim is laid
    # out unit-stride with 16-byte aligned rows in shared memory and whose global
    # rows and block/stage offsets are multiples of 4 words moves as 16-byte
    # cp.async quads (o["fv"] = 4): a quarter of the copies and address math.
    # The layout is not changed to make rows 16-byte aligned: re-padding rows
    # for it measured slower (template_bench A/B: 7 of 30 such States regressed,
    # up to 3.7x), quads on already aligned layouts 17% faster (geomean, 36 States)
    def fhull_real(o):
        return o["hull"][:-1] + [o["hull"][-1] // o.get("fv", 1)]

    def fhull(o):
        """Fetch enumeration hull: the real one, or every dim rounded up to a power
        of two (o["p2"]) so that with a power-of-two block the per-trip coordinates
        are carry-free (one base register + immediates) instead of divided out per
        element; elements outside the real hull are predicated off."""
        h = fhull_real(o)
        return [1 << (x - 1).bit_length() for x in h] if o.get("p2") else h

    def fsize(o):
        return int(np.prod(fhull(o))) if o.get("p2") else o["size"] // o.get("fv", 1)

    def qcoords(o, cs):
        w = o.get("fv", 1)
        return cs if w == 1 else cs[:-1] + [cs[-1].scale(w)]

    def fetch_vec(o) -> int:
        name = o["read"].buffer
        d = len(o["hull"]) - 1
        if "fvec" in _OFF or g.ft != "f32" or name in attached_prod or d < 0:
            return 1
        if name not in mod.live and mod.layouts.get(name) is not None:
            return 1
        if o["order"][-1] != d or o["stride"][d] != 1 or o["hull"][d] % 4 or o["base_word"] % 4:
            return 1
        if any(o["stride"][j] % 4 for j in range(d)) or mod.shape(name)[-1] % 4:
            return 1
        last = operand_base(o, lambda n: Aff.reg(f"%stage_{n}"))[d]
        if last.const % 4 or any(c % 4 for c in last.terms.values()):
            return 1
        return 4

    # loop-invariant part of the cooperative fetch (coordinates, tail predicates,
    # shared-memory addresses, global pointers without the staging offset),
    # emitted once before the staging loop
    fetch_plan: dict = {}

    def plannable(o, trips, long_ok):
        """Hoisted per-trip addressing: always up to 16 trips; up to ASYNC_MAX_TRIPS
        when the trip decomposition is carry-free (one base register + immediates)."""
        if trips <= 16:
            return True
        return long_ok and trips <= ASYNC_MAX_TRIPS and carry_free_shifts(o, trips) is not None

    def prep_fetch(long_ok=False):
        zero = lambda r: Aff.k(0)  # noqa: E731
        for oi, o in enumerate(operands):
            trips = -(-fsize(o) // n_threads)
            if not plannable(o, trips, long_ok) or "plan" in _OFF:
                continue
            full = fsize(o) % n_threads == 0
            shifts = carry_free_shifts(o, trips)
            cs0 = g.decompose(tid, fhull(o)) if shifts is not None else None
            base0 = operand_base(o, zero)
            name = o["read"].buffer
            plain = name not in attached_prod and (name in mod.live or mod.layouts.get(name) is None)
            for t in range(trips):
                tail = None
                if not full and t == trips - 1:
                    tail = g.new("%p")
                    g(f"setp.lt.s32 {tail}, {tid}, {fsize(o) - t * n_threads};")
                if shifts is not None:
                    cs = [Aff.reg(c) + sh for c, sh in zip(cs0, shifts[t])]
                else:
                    cs = [Aff.reg(c) for c in g.decompose(g.aff(Aff.reg(tid) + t * n_threads), fhull(o))]
                if o.get("p2"):         # padded enumeration: predicate off coordinates beyond the hull
                    for c, hr, hp in zip(cs, fhull_real(o), fhull(o)):
                        if hr == hp:
                            continue
                        key = ("p2ok", c.key(), c.const, hr)
                        pv = g.cached(key)
                        if pv is None:
                            cr = g.aff(Aff(dict(c.terms)))
                            pv = g.new("%p")
                            g(f"setp.lt.s32 {pv}, {cr}, {hr - c.const};")
                            g.remember(key, pv)
                        if tail is None:
                            tail = pv
                        else:
                            t2 = g.new("%p")
                            g(f"and.pred {t2}, {tail}, {pv};")
                            tail = t2
                cs = qcoords(o, cs)
                saddr = Aff.k(o["base_word"])
                for c, st_ in zip(cs, o["stride"]):
                    saddr = saddr + c.scale(st_)
                srt = saddr.runtime()
                sreg = g.aff(srt) if srt.terms else None
                ptr = None
                if plain:
                    gb = k.gbase(name)
                    flat = k.gflat(name, [b_ + c for b_, c in zip(base0, cs)])
                    ptr, imm = g.gaddr(gb, flat)
                    ptr = (ptr, flat.const)
                fetch_plan[(oi, t)] = (cs, tail, (sreg, saddr.const), ptr)

    def fetch_load(sdig, pnext=None):
        """Issue the global loads (and inline producer math) of one staging step;
        returns (value, shared word address (register, const), predicate) per element."""
        items = []
        for oi, o in enumerate(operands):
            r = o["read"]
            hull = o["hull"]
            base = operand_base(o, sdig)
            trips = -(-o["size"] // n_threads)
            full = o["size"] % n_threads == 0

            def elem(e_aff, guard_tail, o=o, r=r, hull=hull, base=base):
                er = g.aff(e_aff)
                pt = pnext
                if guard_tail:
                    pt = g.new("%p")
                    g(f"setp.lt.s32 {pt}, {er}, {o['size']};")
                    if pnext is not None:
                        g(f"and.pred {pt}, {pt}, {pnext};")
                cs = g.decompose(er, hull)
                idx = [b_ + Aff.reg(c) for b_, c in zip(base, cs)]
                if r.buffer in attached_prod:
                    v = k.producer(r.buffer, idx, pt)
                else:
                    v = k.gload(r.buffer, idx, pt)
                saddr = Aff.k(o["base_word"])
                for c, st_ in zip(cs, o["stride"]):
                    saddr = saddr + Aff.reg(c, st_)
                items.append((v, (g.aff(saddr), 0), pt))

            def planned(t, o=o, oi=oi, r=r, base=base):
                cs, tail, sa, ptr = fetch_plan[(oi, t)]
                pt = pnext
                if tail is not None:
                    pt = tail
                    if pnext is not None:
                        pt = g.new("%p")
                        g(f"and.pred {pt}, {tail}, {pnext};")
                idx = [b_ + c for b_, c in zip(base, cs)]
                if ptr is None:
                    v = (k.producer(r.buffer, idx, pt) if r.buffer in attached_prod
                         else k.gload(r.buffer, idx, pt))
                else:
                    # global address = hoisted pointer + staging offset (shared by all trips)
                    flat = k.gflat(r.buffer, idx)
                    inv = k.gflat(r.buffer, [b_ + c for b_, c in zip(operand_base(o, lambda n: Aff.k(0)), cs)])
                    stage_part = flat + inv.scale(-1)
                    v = k.gload_at(ptr[0], stage_part, flat.const, pt)
                items.append((v, sa, pt))
            if trips <= 16:
                for t in range(trips):
                    if (oi, t) in fetch_plan:
                        planned(t)
                    else:
                        elem(Aff.reg(tid) + t * n_threads, not full and t == trips - 1)
            else:
                # long fetches: a rolled loop over chunks of FETCH_CHUNK trips, each
                # chunk issuing all its global loads before its shared stores
                n_ch = -(-trips // FETCH_CHUNK)

                def run(tv, o=o, elem=elem):
                    first = len(items)
                    for j in range(FETCH_CHUNK):
                        elem(Aff.reg(tid) + (tv.scale(FETCH_CHUNK) + j).scale(n_threads), True)
                    chunk = items[first:]
                    del items[first:]
                    fetch_store(chunk, sm)
                k.loop(n_ch, False, run)
        return items

    def fetch_store(items, buf):
        for v, (sa, sc), pt in items:
            key = ("sst", sa, buf)
            a = g.cached(key)
            if a is None:
                a = g.new("%r")
                if sa is None:
                    g(f"mov.u32 {a}, {buf};")
                else:
                    g(f"mad.lo.s32 {a}, {sa}, {g.esz}, {buf};")
                g.remember(key, a)
            pred = f"@{pt} " if pt else ""
            g(f"{pred}st.shared.{g.ft} [{a}+{sc * g.esz}], {v};")

    def fetch_async(sdig, buf, pnext):
        """One staging step as cp.async copies global -> shared (no register
        round trip): every element of every operand, predicated on its tail
        guard and on `pnext`; the caller commits the group."""
        for oi, o in enumerate(operands):
            r = o["read"]
            base = operand_base(o, sdig)
            zero_base = operand_base(o, lambda n: Aff.k(0))
            trips = -(-fsize(o) // n_threads)
            nb = g.esz * o.get("fv", 1)
            if (oi, 0) not in fetch_plan:
                # no hoistable addressing: a rolled loop over chunks of trips, every
                # element's coordinates decomposed in place (copies stay asynchronous)
                def chunk(tv, o=o, r=r, base=base):
                    for j in range(FETCH_CHUNK):
                        er = g.aff(Aff.reg(tid) + (tv.scale(FETCH_CHUNK) + j).scale(n_threads))
                        pt = g.new("%p")
                        g(f"setp.lt.s32 {pt}, {er}, {fsize(o)};")
                        if pnext is not None:
                            g(f"and.pred {pt}, {pt}, {pnext};")
                        cs = qcoords(o, [Aff.reg(c) for c in g.decompose(er, fhull(o))])
                        idx_ = [b_ + c for b_, c in zip(base, cs)]
                        zp = None
                        if r.buffer in attached_prod:
                            rb, imm, zp = k.zfill_source(r.buffer, idx_)
                        else:
                            gb, flat = k.gsource(r.buffer, idx_)
                            rb, imm = g.gaddr(gb, flat)
                        saddr = Aff.k(o["base_word"])
                        for c, st_ in zip(cs, o["stride"]):
                            saddr = saddr + c.scale(st_)
                        emit_cp(g.aff(saddr.runtime()) if saddr.runtime().terms else None, saddr.const, buf, pt,
                                rb, imm, zp, nb)
                k.loop(-(-trips // FETCH_CHUNK), False, chunk)
                continue
            for t in range(trips):
                cs, tail, (sa, sc), ptr = fetch_plan[(oi, t)]
                pt = pnext
                if tail is not None:
                    pt = tail
                    if pnext is not None:
                        pt = g.new("%p")
                        g(f"and.pred {pt}, {tail}, {pnext};")
                if r.buffer in attached_prod:           # zero-fill producer (padding)
                    rb, imm, zp = k.zfill_source(r.buffer, [b_ + c for b_, c in zip(base, cs)])
                    emit_cp(sa, sc, buf, pt, rb, imm, zp)
                    continue
                if ptr is None:             # packed layout: element address per stage
                    gb, flat = k.gsource(r.buffer, [b_ + c for b_, c in zip(base, cs)])
                    rb, imm = g.gaddr(gb, flat)
                    emit_cp(sa, sc, buf, pt, rb, imm, None, nb)
                    continue
                flat = k.gflat(r.buffer, [b_ + c for b_, c in zip(base, cs)])
                inv = k.gflat(r.buffer, [b_ + c for b_, c in zip(zero_base, cs)])
                off = flat + inv.scale(-1)
                if off.terms:
                    k2 = ("gptr@", ptr[0], off.key())
                    rb = g.cached(k2)
                    if rb is None:
                        o_ = g.aff(off.runtime())
                        w_ = g.new("%rd")
                        g(f"mul.wide.s32 {w_}, {o_}, {g.esz};")
                        rb = g.new("%rd")
                        g(f"add.s64 {rb}, {ptr[0]}, {w_};")
                        g.remember(k2, rb)
                else:
                    rb = ptr[0]
                emit_cp(sa, sc, buf, pt, rb, flat.const * g.esz, None, nb)

    def emit_cp(sa, sc, buf, pt, rb, imm, zpred=None, nbytes=None):
        key = ("sst", sa, buf)
        a = g.cached(key)
        if a is None:
            a = g.new("%r")
            if sa is None:
                g(f"mov.u32 {a}, {buf};")
            else:
                g(f"mad.lo.s32 {a}, {sa}, {g.esz}, {buf};")
            g.remember(key, a)
        pred = f"@{pt} " if pt else ""
        nbytes = nbytes or g.esz
        if zpred is None and nbytes == 16:           # 16-byte quads bypass L1 (.cg)
            g(f"{pred}cp.async.cg.shared.global [{a}+{sc * g.esz}], [{rb}+{imm}], 16;")
        elif zpred is None:
            g(f"{pred}cp.async.ca.shared.global [{a}+{sc * g.esz}], [{rb}+{imm}], {nbytes};")
        else:                   # zero-fill where the producer's condition fails
            n = g.new("%r")
            g(f"selp.u32 {n}, {g.esz}, 0, {zpred};")
            g(f"{pred}cp.async.ca.shared.global [{a}+{sc * g.esz}], [{rb}+{imm}], {g.esz}, {n};")

    # address coefficients: shared-memory word address of operand o as
    #   const0 + sum over local level digits (axis, level) of coef * digit
    def mult(n, lv):
        m = 1
        for kk in range(lv[1] + 1, n_s if lv[0] == "S" else n_r):
            m *= factors[n][kk]
        return m
    for o in operands:
        coef, c0 = {}, o["base_word"]
        for di, lin in enumerate(o["read"].index):
            c0 += o["stride"][di] * o["off"][di]
            for n, cc in lin.terms:
                kind_ = "S" if n in T else "R"
                for kk in range(1, n_s if kind_ == "S" else n_r):
                    lv = (kind_, kk)
                    if f(n, lv) > 1:
                        coef[(n, lv)] = coef.get((n, lv), 0) + o["stride"][di] * cc * mult(n, lv)
        o["coef"], o["c0"] = coef, c0
        w = o["vec"]
        if w > 1:   # every run must start on a w-word boundary, or fall back to scalar loads
            va = o["vaxis"]
            ok = c0 % w == 0 and run_len(va) % w == 0
            stride = 1
            for lv in reversed(run_lvs):       # run digits: unit-stride mixed radix
                if f(va, lv) > 1:
                    ok = ok and coef.get((va, lv)) == stride
                stride *= f(va, lv)
            ok = ok and all(c % w == 0 for kv, c in coef.items() if not (kv[0] == va and kv[1] in run_lvs))
            if not ok:
                o["vec"] = 1
    op_of = {o["key"]: o for o in operands}
    acc_coef = {}
    m_acc = 1
    for ai in range(len(space) - 1, -1, -1):
        a = space[ai]
        mm = m_acc
        for lv in reversed(reg_levels):
            if f(a, lv) > 1:
                acc_coef[(a, lv)] = mm
                mm *= f(a, lv)
        m_acc *= acc_dims[ai]
    thread_digits = {(a, lv): dig[(a, lv)] for (a, lv) in thr}

    def compute(sdig, smb):
        """Per-thread nest for one staging step; accumulates into acc."""
        g.push()
        fma_body = op == "sum" and kind(body) == "Bin" and body.op == "mul"

        def sbase(o, rt_items):
            key = ("sbase", smb, o["base_word"], rt_items)
            b = g.cached(key)
            if b is None:
                terms = {}
                for (n, lv), reg in rt_items:
                    c = o["coef"].get((n, lv), 0)
                    if c:
                        terms[reg] = terms.get(reg, 0) + c
                b = g.new("%r")
                if terms:
                    x = g.aff(Aff(terms))
                    g(f"mad.lo.s32 {b}, {x}, {g.esz}, {smb};")
                else:
                    g(f"mov.u32 {b}, {smb};")
                g.remember(key, b)
            return b

        state = {"cv": {}, "rv": {}, "rt": ()}
        thread_items = tuple(sorted((k_, next(iter(a_.terms))) for k_, a_ in thread_digits.items()))

        def smem_addr(buf, index, cv):
            o = op_of[(buf, tuple((l.terms, l.const) for l in index))]
            const = o["c0"]
            cf = o["coef"]
            for kv, val in cv.items():
                c = cf.get(kv)
                if c:
                    const += c * val
            return o, const

        def smem(buf, index):
            o, const = smem_addr(buf, index, state["cv"])
            return smem_load(o, const)

        def smem_load(o, const):
            b = sbase(o, state["rt"])
            ck = ("sld", b, const)
            hit = g.cached(ck)
            if hit:
                return hit
            w = o["vec"] if g.ft == "f32" else 1
            if w > 1:
                g0 = const - const % w
                regs = [g.new(g.fr) for _ in range(w)]
                g(f"ld.shared.v{w}.{g.ft} {{{', '.join(regs)}}}, [{b}+{g0 * g.esz}];")
                for j, rr in enumerate(regs):
                    g.remember(("sld", b, g0 + j), rr)
                return regs[const - g0]
            v = g.new(g.fr)
            g(f"ld.shared.{g.ft} {v}, [{b}+{const * g.esz}];")
            return g.remember(ck, v)

        def iv(n):      # global iterator value (only IterVal nodes need it)
            cv, rv = state["cv"], state["rv"]

            def dgf(a, lv):
                if (a, lv) in cv:
                    return Aff.k(cv[(a, lv)])
                if (a, lv) in rv:
                    return Aff.reg(rv[(a, lv)])
                if lv == stage_lv[0] and n in RT:
                    return sdig(a)
                return digit(a, lv)
            return mixed(n, "S" if n in T else "R", 0, dgf)

        class SE(Expr):
            def __call__(self2, e):
                if kind(e) == "Read":
                    return smem(e.buffer, e.index)
                return Expr.__call__(self2, e)
        ex = SE(g, iv, None)

        fma_reads = fma_body and kind(body.lhs) == "Read" and kind(body.rhs) == "Read"

        def region(i, cv):
            """Fully unrolled suffix of the nest: emit operand loads LOOKAHEAD
            statements ahead of their FMAs (software pipelining of the shared loads)."""
            # every statement's accumulator index and operand word offsets are the
            # fixed (outer) digits' part plus a mixed-radix sum over the enumerated
            # levels (innermost fastest): computed for all statements at once
            oa, ca = smem_addr(body.lhs.buffer, body.lhs.index, cv)
            ob, cb = smem_addr(body.rhs.buffer, body.rhs.index, cv)
            ai0 = sum(acc_coef.get(kv, 0) * val for kv, val in cv.items())
            ext = [x[2] for x in loop_list[i:]]
            keys = [(x[0], x[1]) for x in loop_list[i:]]
            grid = np.indices(ext).reshape(len(ext), -1) if ext else np.zeros((0, 1), np.int64)
            ais = ai0 + np.asarray([acc_coef.get(kv, 0) for kv in keys], np.int64) @ grid
            cas = ca + np.asarray([oa["coef"].get(kv, 0) for kv in keys], np.int64) @ grid
            cbs = cb + np.asarray([ob["coef"].get(kv, 0) for kv in keys], np.int64) @ grid
            plan = [(int(x), (oa, int(y)), (ob, int(z))) for x, y, z in zip(ais, cas, cbs)]
            nxt = 0
            for si, (ai, la, lb) in enumerate(plan):
                while nxt < len(plan) and nxt <= si + LOOKAHEAD:
                    smem_load(*plan[nxt][1])
                    smem_load(*plan[nxt][2])
                    nxt += 1
                ra, rb = smem_load(*la), smem_load(*lb)
                g(f"fma.rn.{g.ft} {acc[ai]}, {ra}, {rb}, {acc[ai]};")

        def pipelined(i, cv, rv):
            """A rolled reduction loop around a fully unrolled register tile,
            software-pipelined: the shared operands of step r+1 are loaded into a
            second register set while step r's FMAs issue, so the tile's FMAs do
            not wait for their own loads (with the one or two warps per scheduler
            the tuned tilings leave, nothing else hides shared-load latency).  The
            loop body covers two steps with the two sets alternating; every
            accumulator still sums the steps in loop order, so results are
            unchanged.  Returns False when the pattern or the register budget
            does not fit (the plain rolled loop is emitted instead)."""
            a, lv, ext, _ = loop_list[i]
            if ext < 2 or "pipe" in _OFF:
                return False
            oa, ca = smem_addr(body.lhs.buffer, body.lhs.index, cv)
            ob, cb = smem_addr(body.rhs.buffer, body.rhs.index, cv)
            ai0 = sum(acc_coef.get(kv, 0) * val for kv, val in cv.items())
            ext_in = [x[2] for x in loop_list[i + 1:]]
            keys = [(x[0], x[1]) for x in loop_list[i + 1:]]
            grid = np.indices(ext_in).reshape(len(ext_in), -1) if ext_in else np.zeros((0, 1), np.int64)
            ais = ai0 + np.asarray([acc_coef.get(kv, 0) for kv in keys], np.int64) @ grid
            cas = ca + np.asarray([oa["coef"].get(kv, 0) for kv in keys], np.int64) @ grid
            cbs = cb + np.asarray([ob["coef"].get(kv, 0) for kv in keys], np.int64) @ grid
            plan = [(int(x), int(y), int(z)) for x, y, z in zip(ais, cas, cbs)]
            step = {"a": oa["coef"].get((a, lv), 0), "b": ob["coef"].get((a, lv), 0)}
            ops_ = {"a": oa, "b": ob}
            width = {}
            for w_ in ("a", "b"):
                vw = ops_[w_]["vec"] if g.ft == "f32" else 1
                width[w_] = vw if vw > 1 and step[w_] % vw == 0 else 1
            groups = {"a": sorted({c - c % width["a"] for _, c, _ in plan}),
                      "b": sorted({c - c % width["b"] for _, _, c in plan})}
            n_regs = sum(len(groups[w_]) * width[w_] for w_ in ("a", "b"))
            if n_regs > 64 or n_acc + 2 * n_regs + SPILL_MARGIN > min(255, 65536 // n_threads):
                return False
            sets = []
            for _ in range(2):
                regs = {}
                for w_ in ("a", "b"):
                    for g0 in groups[w_]:
                        for j in range(width[w_]):
                            regs[(w_, g0 + j)] = g.new(g.fr)
                sets.append(regs)

            def load(regs, shift, pred):
                bases = {w_: sbase(ops_[w_], state["rt"]) for w_ in ("a", "b")}
                for w_ in ("a", "b"):
                    wd = width[w_]
                    for g0 in groups[w_]:
                        off = (g0 + shift * step[w_]) * g.esz
                        names = [regs[(w_, g0 + j)] for j in range(wd)]
                        if wd > 1:
                            g(f"{pred}ld.shared.v{wd}.{g.ft} {{{', '.join(names)}}}, [{bases[w_]}+{off}];")
                        else:
                            g(f"{pred}ld.shared.{g.ft} {names[0]}, [{bases[w_]}+{off}];")

            def fmas(regs):
                for ai, xa, xb in plan:
                    g(f"fma.rn.{g.ft} {acc[ai]}, {regs[('a', xa)]}, {regs[('b', xb)]}, {acc[ai]};")

            v = g.new("%r")
            g(f"mov.s32 {v}, 0;")
            rv2 = {**rv, (a, lv): v}
            saved = (state["rv"], state["rt"])
            state["rv"], state["rt"] = rv2, tuple(sorted(rv2.items())) + thread_items
            g.push()
            load(sets[0], 0, "")                           # step 0
            g.pop()
            lab = g.new_label()
            g.label(lab)
            g(".pragma \"nounroll\";")
            g.push()
            load(sets[1], 1, "")                           # step v + 1
            fmas(sets[0])                                  # step v
            p2 = g.new("%p")
            t2 = g.new("%r")
            g(f"add.s32 {t2}, {v}, 2;")
            g(f"setp.lt.s32 {p2}, {t2}, {ext};")
            load(sets[0], 2, f"@{p2} ")                    # step v + 2 (when it exists)
            fmas(sets[1])                                  # step v + 1
            g.pop()
            pq = g.new("%p")
            g(f"add.s32 {v}, {v}, 2;")
            g(f"setp.lt.s32 {pq}, {v}, {ext - 1};")
            g(f"@{pq} bra {lab};")
            if ext % 2:
                fmas(sets[0])                              # the last (odd) step
            state["rv"], state["rt"] = saved
            return True

        def rec(i, cv, rv):
            if acc_in_regs and fma_reads and all(unroll[i:]):
                region(i, cv)
                return
            if (acc_in_regs and fma_reads and i < len(loop_list) and not unroll[i] and all(unroll[i + 1:])
                    and loop_list[i][1][0] == "R" and pipelined(i, cv, rv)):
                return
            if i == len(loop_list):
                if acc_in_regs:
                    ai = 0
                    for kv, val in cv.items():
                        ai += acc_coef.get(kv, 0) * val
                    tgt = acc[ai]
                    if fma_body:
                        a_, b_ = ex(body.lhs), ex(body.rhs)
                        g(f"fma.rn.{g.ft} {tgt}, {a_}, {b_}, {tgt};")
                    else:
                        v = ex(body)
                        g(f"{'add.rn' if op == 'sum' else 'max'}.{g.ft} {tgt}, {tgt}, {v};")
                else:
                    ai = Aff.k(0)
                    for kv, val in cv.items():
                        ai = ai + acc_coef.get(kv, 0) * val
                    for kv, reg in rv.items():
                        if acc_coef.get(kv):
                            ai = ai + Aff.reg(reg, acc_coef[kv])
                    rb, imm = _local_addr(g, ab, ai)
                    cur = g.new(g.fr)
                    g(f"ld.local.{g.ft} {cur}, [{rb}+{imm}];")
                    if fma_body:
                        a_, b_ = ex(body.lhs), ex(body.rhs)
                        g(f"fma.rn.{g.ft} {cur}, {a_}, {b_}, {cur};")
                    else:
                        v = ex(body)
                        g(f"{'add.rn' if op == 'sum' else 'max'}.{g.ft} {cur}, {cur}, {v};")
                    g(f"st.local.{g.ft} [{rb}+{imm}], {cur};")
                return
            a, lv, ext, _ = loop_list[i]
            if unroll[i]:
                for val in range(ext):
                    cv[(a, lv)] = val
                    rec(i + 1, cv, rv)
                del cv[(a, lv)]
            else:
                def inner(r, i=i, a=a, lv=lv):
                    rv2 = {**rv, (a, lv): next(iter(r.terms))}
                    saved = (state["rv"], state["rt"])
                    state["rv"], state["rt"] = rv2, tuple(sorted(rv2.items())) + thread_items
                    rec(i + 1, cv, rv2)
                    state["rv"], state["rt"] = saved
                k.loop(ext, False, inner)
        state["cv"], state["rt"] = {}, thread_items
        rec(0, state["cv"], {})
        g.pop()

    n_stage = 1
    for _, e in stage_axes:
        n_stage *= e
    trips_all = [-(-o["size"] // n_threads) for o in operands]
    # asynchronous staging (cp.async, double-buffered): every operand a plain global
    # read (no inline producer, no packed layout) with hoistable addressing
    # ... and only where the second buffer keeps the SM busy: the same resident
    # blocks, or still >= 4 resident warps (measured on the golden streams: tilings
    # pushed below that lose more latency hiding than the overlap wins)
    occ1 = _blocks_per_sm(n_threads, n_acc, smem_bytes)
    occ2 = _blocks_per_sm(n_threads, n_acc, 2 * smem_bytes)
    spill_heavy = acc_in_regs and n_acc + SPILL_MARGIN > min(255, 65536 // n_threads) and "spillasync" not in _OFF
    async_ok = all(o["read"].buffer not in attached_prod or
                   ("zfill" not in _OFF and k.zfill_producer(o["read"].buffer)) for o in operands)
    use_async = (n_stage > 1 and 2 * smem_bytes <= MAX_SMEM and "async" not in _OFF and not spill_heavy and
                 async_ok and
                 (occ2 >= occ1 or occ2 * -(-n_threads // 32) >= 4))
    double = (not use_async and n_stage > 1 and 2 * smem_bytes <= MAX_SMEM and all(t <= 16 for t in trips_all)
              and sum(trips_all) <= 48)
    copy1 = not use_async and not double and not spill_heavy and "async1" not in _OFF and async_ok
    if use_async or copy1:
        for o in operands:
            o["fv"] = fetch_vec(o)
            if not use_async or "p2" in _OFF or n_threads & (n_threads - 1):
                continue
            # power-of-two fetch enumeration where it turns a per-element divided
            # (rolled) fetch into a carry-free hoisted one at <= 2x idle slots
            real = fhull_real(o)
            t1 = -(-fsize(o) // n_threads)
            if plannable(o, t1, True) or all(x & (x - 1) == 0 for x in real):
                continue
            o["p2"] = True
            t2 = -(-fsize(o) // n_threads)
            if fsize(o) > 2 * int(np.prod(real)) or not plannable(o, t2, True):
                o["p2"] = False
    prep_fetch(long_ok=use_async)
    if use_async:
        buf = total_words * g.esz
        radices = [e for _, e in stage_axes]

        def digits_of(treg):
            ds = g.decompose(treg, radices)
            m = {r: Aff.reg(d) for (r, _), d in zip(stage_axes, ds)}
            return lambda r: m.get(r, Aff.k(0))
        g.push()
        fetch_async(lambda r: Aff.k(0), sm, None)
        g.pop()
        g("cp.async.commit_group;")
        t = g.new("%r")
        lab = g.new_label()
        g(f"mov.s32 {t}, 0;")
        g.label(lab)
        g(".pragma \"nounroll\";")
        g.push()
        par, smb, nbuf, t1, pn = g.new("%r"), g.new("%r"), g.new("%r"), g.new("%r"), g.new("%p")
        g(f"and.b32 {par}, {t}, 1;")
        g(f"mad.lo.s32 {smb}, {par}, {buf}, {sm};")
        g(f"xor.b32 {nbuf}, {par}, 1;")
        g(f"mad.lo.s32 {nbuf}, {nbuf}, {buf}, {sm};")
        g(f"add.s32 {t1}, {t}, 1;")
        g(f"setp.lt.s32 {pn}, {t1}, {n_stage};")
        fetch_async(digits_of(t1), nbuf, pn)       # next step's copies fly during this step
        g("cp.async.commit_group;")
        g("cp.async.wait_group 1;")                # this step's group has landed
        g("bar.sync 0;")
        compute(digits_of(t), smb)
        g("bar.sync 0;")                           # the buffer is refilled next iteration
        g.pop()
        g(f"add.s32 {t}, {t}, 1;")
        pl = g.new("%p")
        g(f"setp.lt.s32 {pl}, {t}, {n_stage};")
        g(f"@{pl} bra {lab};")
        g("cp.async.wait_group 0;")
        smem_bytes = 2 * buf
    elif not double:
        # single-buffered: plain operands still move by cp.async (no register
        # round trip), others through registers
        def stage_rec(i, sd):
            if i == len(stage_axes):
                sdig = lambda r, sd=sd: sd.get(r, Aff.k(0))  # noqa: E731
                g.push()
                if copy1:
                    fetch_async(sdig, sm, None)
                    g("cp.async.commit_group;")
                    g("cp.async.wait_group 0;")
                else:
                    items = fetch_load(sdig)
                    fetch_store(items, sm)
                g.pop()
                g("bar.sync 0;")
                compute(sdig, sm)
                g("bar.sync 0;")
                return
            r, e = stage_axes[i]
            k.loop(e, False, lambda v: stage_rec(i + 1, {**sd, r: v}))
        stage_rec(0, {})
    else:
        # software pipeline: the next step's global loads are issued before this
        # step's FMAs and land in the other shared-memory buffer afterwards
        buf = total_words * g.esz
        radices = [e for _, e in stage_axes]

        def digits_of(treg):
            ds = g.decompose(treg, radices)
            m = {r: Aff.reg(d) for (r, _), d in zip(stage_axes, ds)}
            return lambda r: m.get(r, Aff.k(0))
        g.push()
        fetch_store(fetch_load(lambda r: Aff.k(0)), sm)
        g.pop()
        g("bar.sync 0;")
        t = g.new("%r")
        lab = g.new_label()
        g(f"mov.s32 {t}, 0;")
        g.label(lab)
        g(".pragma \"nounroll\";")
        g.push()
        par, smb, nbuf, t1, pn = g.new("%r"), g.new("%r"), g.new("%r"), g.new("%r"), g.new("%p")
        g(f"and.b32 {par}, {t}, 1;")
        g(f"mad.lo.s32 {smb}, {par}, {buf}, {sm};")
        g(f"xor.b32 {nbuf}, {par}, 1;")
        g(f"mad.lo.s32 {nbuf}, {nbuf}, {buf}, {sm};")
        g(f"add.s32 {t1}, {t}, 1;")
        g(f"setp.lt.s32 {pn}, {t1}, {n_stage};")
        items = fetch_load(digits_of(t1), pn)
        compute(digits_of(t), smb)
        fetch_store(items, nbuf)
        g("bar.sync 0;")
        g.pop()
        g(f"add.s32 {t}, {t}, 1;")
        pl = g.new("%p")
        g(f"setp.lt.s32 {pl}, {t}, {n_stage};")
        g(f"@{pl} bra {lab};")
        smem_bytes = 2 * buf

    # epilogue over the register tile
    reg_loops = [(a, lv, f(a, lv)) for lv in reg_levels for a in space if f(a, lv) > 1]

    mustm = mod.must_materialize(s)
    if acc_in_regs:
        # straight-line epilogue: every register-level digit is a constant, so each
        # element's index is a shared runtime base plus a compile-time offset
        reg_set = set(reg_levels)
        base_idx = {a: mixed(a, "S", 0, lambda a_, lv: Aff.k(0) if lv in reg_set else digit(a_, lv))
                    for a in space}
        k.vec_stores = "vst" not in _OFF
        for combo in itertools.product(*[range(ext) for _, _, ext in reg_loops]):
            off = dict.fromkeys(space, 0)
            ai = 0
            for (a, lv, _), val in zip(reg_loops, combo):
                off[a] += val * mult(a, lv)
                ai += acc_coef.get((a, lv), 0) * val
            k.epilogue(s, {a: base_idx[a] + off[a] for a in space}, acc[ai], mustm)
        k.drain_stores(True)
        k.vec_stores = False

    def ep(i, dg):
        if i == len(reg_loops):
            def dgf(a, lv):
                return dg.get((a, lv), digit(a, lv))
            idx_of = {a: mixed(a, "S", 0, dgf) for a in space}
            ai = acc_index(dgf)
            if acc_in_regs:
                val = acc[ai.const]
            else:
                rb, imm = _local_addr(g, ab, ai)
                val = g.new(g.fr)
                g(f"ld.local.{g.ft} {val}, [{rb}+{imm}];")
            g.push()
            k.epilogue(s, idx_of, val, mustm)
            g.pop()
            return
        a, lv, ext = reg_loops[i]
        k.loop(ext, False, lambda r: ep(i + 1, {**dg, (a, lv): r}))
    if not acc_in_regs:
        ep(0, {})

    info = {"template": "tiled", "stage": s.name, "structure": structure, "threads": n_threads,
            "blocks": n_blocks, "vthreads": n_vt, "acc": n_acc, "smem": smem_bytes, "unrolled": unrolled,
            "factors": {a: list(v) for a, v in factors.items()}, "backend": "ptx",
            "double_buffered": double or use_async, "async_copy": use_async, "acc_in_regs": acc_in_regs,
            "n_stage": n_stage, "fetch_vec": [o.get("fv", 1) for o in operands],
            "fetch_pow2": [bool(o.get("p2")) for o in operands]}
    return k, Kernel(entry, n_blocks, n_threads, smem_bytes, list(k.params), info)


def _blocks_per_sm(threads: int, n_acc: int, smem: int) -> int:
    """Resident blocks per SM (B200: 2048 threads, 64K registers, 228 KB shared
    memory with 1 KB reserved per block, 32 blocks), registers estimated as the
    accumulator tile plus SPILL_MARGIN."""
    regs = min(255, -(-(n_acc + SPILL_MARGIN) // 8) * 8)
    by_regs = 65536 // max(1, threads * regs)
    by_smem = (228 * 1024) // (smem + 1024) if smem else 32
    return max(0, min(32, 2048 // threads, by_regs, by_smem))


def _local_addr(g: Ptx, ab: str, ai: Aff) -> tuple:
    rt = ai.runtime()
    if not rt.terms:
        return ab, ai.const * g.esz
    key = ("laddr", rt.key())
    hit = g.cached(key)
    if hit is None:
        x = g.aff(rt)
        w = g.new("%rd")
        g(f"mul.wide.s32 {w}, {x}, {g.esz};")
        hit = g.new("%rd")
        g(f"add.s64 {hit}, {ab}, {w};")
        g.remember(key, hit)
    return hit, ai.const * g.esz


def lower_ptx(p, dtype: str = "float") -> Lowered:
    """Same contract as `lower.lower`, but `source` is a PTX module."""
    if not p.is_concrete():
        raise LoweringError("program has unresolved symbolic extents")
    mod = _Mod(p, dtype)
    kernels, texts = [], []
    pairs = _xreduce_pairs(mod)
    fused = {F.name for F in pairs.values()}
    for s in p.stages:
        if s.inlined or s.compute_at is not None or s.name in fused:
            continue
        for c in _attached(p, s.name):
            if _attached(p, c.name) and any(_reads_buffer(c.expr, gg.name) for gg in _attached(p, c.name)):
                raise LoweringError(f"nested producer attachment under {c.name} is not supported")
        entry = f"k{len(kernels)}_" + ident(s.name)
        levels = tile_levels(p, s) if s.name not in pairs else None
        if s.name in pairs:
            kk, kern = _xreduce(mod, s, pairs[s.name], entry)
        elif levels is not None:
            kk, kern = _tiled(mod, s, levels, entry)
        else:
            kk, kern = _naive(mod, s, entry)
        kern.info["backend"] = "ptx"
        kernels.append(kern)
        texts.append(kk.text())
    for name, st in mod.live.items():
        if name not in mod.buffers and name not in pairs:      # a fused partial never exists
            mod.buffers[name] = Buffer(name, tuple(e for _, e in st.space),
                                       "output" if name in p.dag.outputs else "temp")
    head = ".version 8.7\n.target sm_100a\n.address_size 64\n.extern .shared .align 16 .b8 smem_[];\n"
    info = {"kernels": [k.info for k in kernels], "backend": "ptx"}
    # ptxas -O3 has miscompiled kernels whose register tile overflows the register
    # file (wrong values, out-of-range shared addresses, kernel faults; correct at
    # -O1 and through NVRTC): such modules are assembled at -O1 up front
    for kk in kernels:
        ki = kk.info
        if "o1guard" not in _OFF and ki.get("template") == "tiled" and ki.get("acc_in_regs") and \
                ki["acc"] + SPILL_MARGIN > min(255, 65536 // ki["threads"]):
            info["ptxas_opt"] = "-O1"
            ki["ptxas"] = "-O1 (register tile exceeds the register file)"
    return Lowered(head + "\n".join(texts), kernels, mod.buffers, list(p.dag.outputs), info)
