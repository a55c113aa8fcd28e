"""State -> GPU kernel lowering and CUDA code generation.

Every live root stage of a State becomes one kernel; stages attached to it
(`compute_at`) are fused into it: attached producers are computed inline where
the host reads them (for a tiled host: inside the shared-memory operand fetch),
attached consumers become the host's epilogue.  Two templates:

* **tiled** — a stage multi-level tiled by the sketch rules (`_tile_plan`,
  `src/sketch.py:114-158`).  Level factors are read from the State's own
  `Split` steps (edited in place by `mutate_tile_size`) and the level order from
  its `Reorder` step, not from the fused/annotated loops.  For the GPU structure
  "SSSRRSRS" the binding is S0 -> blockIdx, S1 -> vthread (unrolled inside the
  thread, TVM semantics), S2 -> threadIdx, R0 -> the shared-memory staging step
  (each operand's interval hull over the block tile and one R0 step is fetched
  cooperatively), and R1 S3 R2 S4 -> the per-thread loop nest over a register
  accumulator tile.  Other structures bind generically: first leading S level
  -> blockIdx, last leading S level -> threadIdx, levels between -> vthread,
  first R level -> staging step.  The stage's `pragma_unroll`
  (auto_unroll_max_step) unrolls per-thread loops from the innermost outwards
  while the product of extents stays within the budget (`src/features.py:327-350`
  defines the same coverage); uncovered loops get `#pragma unroll 1`, except
  that the register tile's space loops are unrolled when the tile fits the
  register file (`promote_register_tile`: what NVCC does to TVM's output).
* **naive** — any other stage: one thread per output point (grid-stride),
  reductions serial per thread, unroll budget applied to the reduction loops.

CPU-only decisions (which loops are fused into the `parallel` band,
`vectorize` on a loop the GPU binds to lanes anyway) do not change the kernel;
two States that differ only there lower to the same source and share a cubin.

GPU legality (reported as INVALID with a detail string, the reference's
status for a program that cannot run): threads/block <= 1024 and shared memory
<= 227 KB (hardware); virtual threads <= 8 (TVM's CUDA `max_vthread_extent`,
the bound Ansor's GPU search and `verify_gpu_code` apply); accumulators/thread
<= 256 (the 255-register file: a larger tile cannot be register-resident);
unrolled statements <= 4096 (compile-time guard).  Values are computed in fp32 (FFMA), the paper's
search space having no tensor cores.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

from .state import kind, reads

MAX_THREADS = 1024
MAX_SMEM = 227 * 1024
MAX_ACC = 256
MAX_VTHREAD = 8
MAX_UNROLLED = 4096
NAIVE_THREADS = 256


class LoweringError(Exception):
    """The State cannot be expressed as a legal launch (-> INVALID)."""


@dataclass
class Buffer:
    name: str
    shape: tuple
    role: str                 # 'input' | 'packed' | 'temp' | 'output'
    desc: tuple = ()          # packing descriptor for 'packed'
    source: str = ""          # placeholder name for 'packed'

    @property
    def numel(self) -> int:
        n = 1
        for e in self.shape:
            n *= e
        return n


@dataclass
class Kernel:
    entry: str
    grid: int
    block: int
    smem: int
    args: list                # buffer names, in parameter order
    info: dict = field(default_factory=dict)


@dataclass
class Lowered:
    source: str
    kernels: list
    buffers: dict             # name -> Buffer
    outputs: list             # DAG output buffer names
    info: dict = field(default_factory=dict)


# ---------------------------------------------------------------------------
# State inspection
# ---------------------------------------------------------------------------


def tile_levels(p, stage):
    """(structure, {axis: factors outer->inner}) for a multi-level tiled stage,
    else None.  Reads the stage's Split/Reorder steps from the history."""
    space = [n for n, _ in stage.space]
    red = [n for n, _ in stage.reduce]
    ext = dict((*stage.space, *stage.reduce))
    splits, order = {}, None
    for st in p.history:
        k = kind(st)
        if getattr(st, "stage", None) != stage.name:
            continue
        if k == "Split" and st.loop in ext and st.loop not in splits:
            splits[st.loop] = tuple(st.inner)
        elif k == "Reorder" and order is None and any("." in x for x in st.order):
            order = tuple(st.order)
    if order is None or not red:
        return None
    levels = []
    for lid in order:
        base, _, lvl = lid.rpartition(".")
        if base not in ext or not lvl.isdigit():
            if lid in ext:          # axis left unsplit (one level of its kind)
                base, lvl = lid, "0"
            else:
                return None
        tag = ("S" if base in space else "R", int(lvl))
        if not levels or levels[-1] != tag:
            levels.append(tag)
    structure = "".join(t for t, _ in levels)
    n_s, n_r = structure.count("S"), structure.count("R")
    factors = {}
    for a in space + red:
        want = n_s if a in space else n_r
        inner = splits.get(a, ())
        if want == 1 and not inner:
            factors[a] = (ext[a],)
            continue
        if len(inner) != want - 1 or any(f is None for f in inner):
            return None
        prod = 1
        for f in inner:
            prod *= f
        if ext[a] % prod:
            return None
        factors[a] = (ext[a] // prod,) + tuple(inner)
    return structure, factors


def _attached(p, host_name):
    return [s for s in p.stages if not s.inlined and s.compute_at is not None and s.compute_at[0] == host_name]


def _reads_buffer(expr, name) -> bool:
    return expr is not None and any(r.buffer == name for r in reads(expr))


# ---------------------------------------------------------------------------
# C emission helpers
# ---------------------------------------------------------------------------


def _flt(x: float, dtype: str) -> str:
    """Exact constant: the reference's float64 literal, cast to the kernel type."""
    x = float(x)
    if math.isinf(x):
        v = "INFINITY" if x > 0 else "(-INFINITY)"
    elif math.isnan(x):
        v = "__int_as_float(0x7fc00000)"
    else:
        v = repr(x)
    return f"(({dtype}){v})"


def ident(name: str) -> str:
    """C identifier for a reference iterator / buffer name."""
    return "".join(ch if ch.isalnum() else "_" for ch in name)


def _lin(lin, iv) -> str:
    """C int expression of an affine form; `iv` maps iterator -> C expression."""
    parts = [str(lin.const)] if lin.const else []
    for n, c in lin.terms:
        t = f"({iv(n)})"
        parts.append(t if c == 1 else f"{c}*{t}")
    return " + ".join(parts) if parts else "0"


class Emitter:
    """Expression emitter over one stage's iterator space."""

    def __init__(self, dtype: str, iv, read):
        self.dtype, self.iv, self.read = dtype, iv, read
        self.guard = 0

    def __call__(self, e) -> str:
        k = kind(e)
        d = self.dtype
        if k == "Const":
            return _flt(e.value, d)
        if k == "IterVal":
            return f"(({d})({_lin(e.lin, self.iv)}))"
        if k == "Read":
            return self.read(e.buffer, e.index, self.guard > 0)
        if k == "Bin":
            a, b = self(e.lhs), self(e.rhs)
            f = "f" if d == "float" else ""
            one, zero = ("1.0f", "0.0f") if d == "float" else ("1.0", "0.0")
            return {"add": f"({a} + {b})", "sub": f"({a} - {b})", "mul": f"({a} * {b})",
                    "div": f"({a} / {b})", "max": f"fmax{f}({a}, {b})", "min": f"fmin{f}({a}, {b})",
                    "lt": f"(({a}) < ({b}) ? {one} : {zero})", "le": f"(({a}) <= ({b}) ? {one} : {zero})",
                    "gt": f"(({a}) > ({b}) ? {one} : {zero})", "ge": f"(({a}) >= ({b}) ? {one} : {zero})",
                    "eq": f"(({a}) == ({b}) ? {one} : {zero})"}[e.op]
        if k == "Call":
            f = "f" if d == "float" else ""
            return {"exp": f"exp{f}", "sqrt": f"sqrt{f}", "log": f"log{f}", "abs": f"fabs{f}"}[e.fn] + f"({self(e.arg)})"
        if k == "Select":
            # Branch reads are only performed where the condition holds
            # (src/expr.py:388-393); their indices may be negative elsewhere, which is
            # why every global address is formed from sign-extended 64-bit terms.
            zero = "0.0f" if d == "float" else "0.0"
            cond = self(e.cond)
            self.guard += 1
            try:
                a, b = self(e.then), self(e.other)
            finally:
                self.guard -= 1
            return f"(({cond}) != {zero} ? ({a}) : ({b}))"
        raise LoweringError(f"unsupported expression node {k}")


# ---------------------------------------------------------------------------
# Program lowering
# ---------------------------------------------------------------------------


class _Ctx:
    def __init__(self, p, dtype="float"):
        self.p = p
        self.dtype = dtype
        self.dag = p.dag
        self.live = {s.name: s for s in p.stages if not s.inlined}
        self.layouts = dict(p.layouts)
        self.buffers: dict = {}
        self.helpers: list = []      # device helper functions (inline producers)
        self.helper_deps: dict = {}  # helper name -> buffers it reads
        self.refs: list = []         # buffers read by the kernel being emitted

    def shape(self, name):
        if name in self.live:
            return tuple(e for _, e in self.live[name].space)
        return self.dag.node(name).shape

    def param(self, name) -> str:
        return "b_" + ident(name)

    def _ref(self, name):
        if name not in self.refs:
            self.refs.append(name)

    # global memory access (placeholders may be packed; stages are row-major)
    def global_load(self, name, idx_exprs) -> str:
        desc = self.layouts.get(name) if name not in self.live else None
        if desc is not None:
            key = f"{name}#packed"
            if key not in self.buffers:
                self.buffers[key] = Buffer(key, tuple(e for _, e in desc), "packed", tuple(desc), name)
            self._ref(key)
            phys = []
            for i, (d, e) in enumerate(desc):
                st = 1
                for d2, e2 in desc[i + 1:]:
                    if d2 == d:
                        st *= e2
                x = f"({idx_exprs[d]})"
                if st > 1:
                    x = f"({x} / {st})"
                phys.append(f"({x} % {e})" if e < self.shape(name)[d] or st > 1 else x)
            flat, mul = [], 1
            for i in range(len(desc) - 1, -1, -1):
                flat.append(f"(long long){phys[i]}" if mul == 1 else f"(long long){phys[i]}*{mul}")
                mul *= desc[i][1]
            return f"__ldg(&{self.param(key)}[{' + '.join(reversed(flat))}])"
        if name not in self.live and name not in self.buffers:
            self.buffers[name] = Buffer(name, self.shape(name), "input")
        self._ref(name)
        shape = self.shape(name)
        # 64-bit signed address arithmetic: unrolled loops share a base offset that
        # can be negative even when every access is in bounds
        flat, mul = [], 1
        for d in range(len(shape) - 1, -1, -1):
            flat.append(f"(long long)({idx_exprs[d]})" if mul == 1 else f"(long long)({idx_exprs[d]})*{mul}")
            mul *= shape[d]
        addr = " + ".join(reversed(flat)) if flat else "0"
        return f"__ldg(&{self.param(name)}[{addr}])"

    def store(self, name, idx_exprs, value) -> str:
        shape = self.shape(name)
        flat, mul = [], 1
        for d in range(len(shape) - 1, -1, -1):
            flat.append(f"(long long)({idx_exprs[d]})" if mul == 1 else f"(long long)({idx_exprs[d]})*{mul}")
            mul *= shape[d]
        return f"{self.param(name)}[{' + '.join(reversed(flat)) if flat else '0'}] = {value};"

    def producer_call(self, name, idx) -> str:
        """Inline value of attached producer stage `name` at a logical index."""
        fn = "prod_" + ident(name)
        if fn not in self.helper_deps:
            outer = self.refs
            self.refs = []
            s = self.live[name]
            space = [n for n, _ in s.space]
            red = [(n, e) for n, e in s.reduce]
            env = {n: "it_" + ident(n) for n, _ in (*s.space, *s.reduce)}
            em = Emitter(self.dtype, lambda n: env[n], self.reader(s, env))
            d = self.dtype
            body = s.expr.body if kind(s.expr) == "Reduce" else s.expr
            val = em(body)
            deps = list(self.refs)
            self.refs = outer
            params = [f"const {d}* __restrict__ {self.param(b)}" for b in deps] + \
                     [f"int {env[n]}" for n in space]
            lines = [f"__device__ __forceinline__ {d} {fn}({', '.join(params)}) {{"]
            if red:
                op = s.expr.op
                lines.append(f"  {d} acc = {_flt(0.0 if op == 'sum' else -math.inf, d)};")
                for n, e in red:
                    lines.append(f"  for (int {env[n]} = 0; {env[n]} < {e}; ++{env[n]})")
                f = "f" if d == "float" else ""
                lines.append(f"    acc = {'acc + ' + val if op == 'sum' else f'fmax{f}(acc, {val})'};")
                lines.append("  return acc;")
            else:
                lines.append(f"  return {val};")
            lines.append("}")
            self.helpers.append("\n".join(lines))
            self.helper_deps[fn] = deps
        for b in self.helper_deps[fn]:
            self._ref(b)
        args = [self.param(b) for b in self.helper_deps[fn]] + list(idx)
        return f"{fn}({', '.join(args)})"

    def reader(self, stage, env, override=None):
        """Read function for expressions of `stage`: attached producers inline,
        everything else from global memory."""
        attached_prod = {s.name for s in _attached(self.p, stage.name)
                         if _reads_buffer(stage.expr, s.name)}

        def read(buf, index, guarded=False):
            if override is not None:
                r = override(buf, index)
                if r is not None:
                    return r
            if buf in attached_prod:
                return self.producer_call(buf, [_lin(l, lambda n: env[n]) for l in index])
            # global addresses: iterator leaves widened to 64 bits before any
            # arithmetic, so a negative partial sum (padding reads under a Select)
            # can never be zero-extended by the compiler
            return self.global_load(buf, [_lin(l, lambda n: f"(long long){env[n]}") for l in index])
        return read


def _unroll_flags(extents: list, budget: int) -> list:
    """Innermost-outward coverage under the unroll budget (True = unrolled)."""
    flags = [False] * len(extents)
    prod = 1
    for i in range(len(extents) - 1, -1, -1):
        if budget <= 0 or prod * extents[i] > budget:
            break
        prod *= extents[i]
        flags[i] = True
    return flags


def promote_register_tile(extents: list, unroll: list, is_space: list, n_acc: int, n_threads: int) -> list:
    """Loops the unroll pragma leaves uncovered are left to the compiler, as TVM
    leaves them to NVCC (`auto_unroll_max_step` only forces unrolling).  NVCC
    fully unrolls constant-trip loops and promotes the local accumulator array to
    registers when every index becomes constant; we model that for the register
    tile: if some space-level loop is rolled, unroll all space-level loops as
    long as the unrolled body stays within MAX_UNROLLED.  Legality is decided on
    the pragma's own plan before this runs, so verdicts do not change.  Measured
    on the golden streams, a register tile that spills still beats explicit
    local-memory accumulators in ~95% of cases, so no register budget applies."""
    if all(u for u, sp in zip(unroll, is_space) if sp):
        return unroll
    trial = [u or sp for u, sp in zip(unroll, is_space)]
    prod = 1
    for e, u in zip(extents, trial):
        if u:
            prod *= e
    return trial if prod <= MAX_UNROLLED else unroll


def _pragma(flag: bool) -> str:
    return "#pragma unroll" if flag else "#pragma unroll 1"


def _epilogue(ctx: _Ctx, host, idx_of, value: str, indent: str, materialize: bool) -> list:
    """Store the host value and run attached consumers (recursively)."""
    out = []
    space = [n for n, _ in host.space]
    if materialize:
        out.append(indent + ctx.store(host.name, [idx_of[n] for n in space], value))
    for c in _attached(ctx.p, host.name):
        if not _reads_buffer(c.expr, host.name) or _reads_buffer(host.expr, c.name):
            continue
        cspace = [n for n, _ in c.space]
        if len(cspace) != len(space):
            raise LoweringError(f"consumer {c.name} rank differs from {host.name}")
        if c.reduce:
            raise LoweringError(f"attached consumer {c.name} reduces")
        cenv = {cn: idx_of[hn] for cn, hn in zip(cspace, space)}
        tmp = "v_" + ident(c.name)

        def ov(buf, index, host=host, cspace=cspace, value=value):
            if buf == host.name:
                if [l.terms for l in index] == [((n, 1),) for n in cspace] and all(l.const == 0 for l in index):
                    return f"({value})"
                raise LoweringError(f"consumer {c.name} reads {host.name} at a non-identity index")
            return None
        em = Emitter(ctx.dtype, lambda n: cenv[n], ctx.reader(c, cenv, override=ov))
        out.append(f"{indent}const {ctx.dtype} {tmp} = {em(c.expr)};")
        out += _epilogue(ctx, c, {n: cenv[n] for n in cspace}, tmp, indent, True)
    return out


def _must_materialize(ctx: _Ctx, stage) -> bool:
    if stage.name in ctx.dag.outputs:
        return True
    attached_cons = {c.name for c in _attached(ctx.p, stage.name) if _reads_buffer(c.expr, stage.name)}
    for s in ctx.live.values():
        if s.name != stage.name and _reads_buffer(s.expr, stage.name) and s.name not in attached_cons:
            return True
    return False


def _kernel_args(ctx: _Ctx, writes: list) -> list:
    """Parameters of the kernel being emitted: outputs first, then reads."""
    names = []
    for w in writes + ctx.refs:
        if w not in names:
            names.append(w)
    return names


def _signature(ctx: _Ctx, entry: str, args: list, writes: set, threads: int) -> str:
    ps = []
    for a in args:
        q = "" if a in writes else "const "
        ps.append(f"{q}{ctx.dtype}* __restrict__ {ctx.param(a)}")
    return f'extern "C" __global__ void __launch_bounds__({threads}) {entry}({", ".join(ps)})'


def _decode_c(d, lv) -> str:
    """C int expression of a decode AST over loop variables (`src/ir.py:73-93`)."""
    k = kind(d)
    if k == "DVar":
        return lv[d.loop]
    if k == "DConst":
        return str(d.value)
    if k == "DAdd":
        return f"({_decode_c(d.a, lv)} + {_decode_c(d.b, lv)})"
    op = {"DMul": "*", "DDiv": "/", "DMod": "%"}[k]
    return f"({_decode_c(d.a, lv)} {op} {d.c})"


def _naive_kernel(ctx: _Ctx, s, entry: str) -> tuple:
    """One thread per point of the stage's space loops; its reduction loops run
    serially in State order; iterators come from the stage's decode map, so split,
    fused and rfactor'd nests lower exactly as the State defines them."""
    d = ctx.dtype
    sp_loops = [l for l in s.loops if l.kind == "space"]
    rd_loops = [l for l in s.loops if l.kind != "space"]
    lv = {l.id: "l_" + ident(l.id) for l in s.loops}
    total = 1
    for l in sp_loops:
        total *= l.extent
    dmap = dict(s.index_map)
    env = {n: f"it_{ident(n)}" for n in dmap}
    em = Emitter(d, lambda n: env[n], ctx.reader(s, env))
    body = [f"  for (long long p_ = (long long)blockIdx.x * {NAIVE_THREADS} + threadIdx.x; p_ < {total}LL; "
            f"p_ += (long long)gridDim.x * {NAIVE_THREADS}) {{",
            "    long long q_ = p_;"]
    for l in reversed(sp_loops):
        body.append(f"    const int {lv[l.id]} = (int)(q_ % {l.extent}); q_ /= {l.extent};")
    space_names = {n for n, _ in s.space}
    for n, dec in s.index_map:
        if n in space_names:
            body.append(f"    const int {env[n]} = {_decode_c(dec, lv)};")
    if rd_loops:
        op = s.expr.op
        body.append(f"    {d} acc_ = {_flt(0.0 if op == 'sum' else -math.inf, d)};")
        flags = _unroll_flags([l.extent for l in rd_loops], s.pragma_unroll)
        ind = "    "
        for l, fl in zip(rd_loops, flags):
            body.append(f"{ind}{_pragma(fl)}")
            body.append(f"{ind}for (int {lv[l.id]} = 0; {lv[l.id]} < {l.extent}; ++{lv[l.id]}) {{")
            ind += "  "
        for n, dec in s.index_map:
            if n not in space_names:
                body.append(f"{ind}const int {env[n]} = {_decode_c(dec, lv)};")
        val = em(s.expr.body)
        f = "f" if d == "float" else ""
        body.append(f"{ind}acc_ = {'acc_ + ' + val if op == 'sum' else f'fmax{f}(acc_, {val})'};")
        for _ in rd_loops:
            ind = ind[:-2]
            body.append(f"{ind}}}")
        value = "acc_"
    else:
        expr = s.expr.body if kind(s.expr) == "Reduce" else s.expr
        value = "val_"
        body.append(f"    const {d} val_ = {em(expr)};")
    body += _epilogue(ctx, s, {n: env[n] for n, _ in s.space}, value, "    ", _must_materialize(ctx, s))
    body.append("  }")
    text = "\n".join(body)
    writes = _written(ctx, s)
    args = _kernel_args(ctx, writes)
    grid = max(1, min((total + NAIVE_THREADS - 1) // NAIVE_THREADS, 148 * 16))
    src = _signature(ctx, entry, args, set(writes), NAIVE_THREADS) + " {\n" + text + "\n}\n"
    return src, Kernel(entry, grid, NAIVE_THREADS, 0, args, {"template": "naive", "stage": s.name,
                                                               "points": total})


def _written(ctx: _Ctx, s) -> list:
    out = []
    if _must_materialize(ctx, s):
        out.append(s.name)
    for c in _attached(ctx.p, s.name):
        if _reads_buffer(c.expr, s.name) and not _reads_buffer(s.expr, c.name):
            out += _written_all(ctx, c)
    return out


def _written_all(ctx, c):
    out = [c.name]
    for cc in _attached(ctx.p, c.name):
        if _reads_buffer(cc.expr, c.name) and not _reads_buffer(c.expr, cc.name):
            out += _written_all(ctx, cc)
    return out


def _binding(structure: str):
    """Level roles: returns (block, vthread, thread, stage, inner) as lists of
    (kind, level) in structure order."""
    lv, cnt = [], {"S": 0, "R": 0}
    for ch in structure:
        lv.append((ch, cnt[ch]))
        cnt[ch] += 1
    m = 0
    while m < len(lv) and lv[m][0] == "S":
        m += 1
    lead = lv[:m]
    block = lead[:1]
    thread = lead[-1:] if m >= 2 else []
    vthread = lead[1:-1] if m >= 3 else []
    rest = lv[m:]
    stage = rest[:1] if rest and rest[0][0] == "R" else []
    inner = rest[1:] if stage else rest
    return block, vthread, thread, stage, inner


def gpu_binding(p, stage) -> tuple:
    """(blockIdx.x, threadIdx.x, vthread, shared bytes) of the kernel that runs
    `stage`'s root under this lowering, from the State's tile levels alone (no
    code generation): the values of the 8 `gpu_*` feature slots the reference
    leaves zero (src/features.py:63-65,395), for the opt-in GPU feature mode."""
    smap = {x.name: x for x in p.stages}
    root = stage
    while root.compute_at is not None:
        root = smap[root.compute_at[0]]
    levels = tile_levels(p, root)
    points = 1
    for _, e in root.space:
        points *= e
    if levels is None:
        grid = max(1, min((points + NAIVE_THREADS - 1) // NAIVE_THREADS, 148 * 16))
        return grid, NAIVE_THREADS, 1, 0
    structure, factors = levels
    block, vthread, thread, _, _ = _binding(structure)
    nb = nt = nv = 1
    for a, _ in root.space:
        for lv in block:
            nb *= factors[a][lv[1]]
        for lv in thread:
            nt *= factors[a][lv[1]]
        for lv in vthread:
            nv *= factors[a][lv[1]]
    n_s, n_r = structure.count("S"), structure.count("R")
    span = {}
    for a, _ in root.space:
        t = 1
        for k in range(1, n_s):
            t *= factors[a][k]
        span[a] = t
    for r, _ in root.reduce:
        t = 1
        for k in range(1, n_r):
            t *= factors[r][k]
        span[r] = t
    smem = 0
    seen = set()
    for rd in (reads(root.expr.body) if root.reduce else []):
        key = (rd.buffer, tuple((l.terms, l.const) for l in rd.index))
        if key in seen:
            continue
        seen.add(key)
        words = 1
        for lin in rd.index:
            words *= 1 + sum(abs(c) * (span.get(n, 1) - 1) for n, c in lin.terms)
        smem += words * 4
    return nb, nt, nv, smem


def _tiled_kernel(ctx: _Ctx, s, levels, entry: str) -> tuple:
    structure, factors = levels
    d = ctx.dtype
    space = [n for n, _ in s.space]
    red = [n for n, _ in s.reduce]
    block, vthread, thread, stage_lv, inner = _binding(structure)
    if not stage_lv:
        raise LoweringError("tiled stage has no reduction level to stage")
    lvl_index = {}
    for ch in "SR":
        k = 0
        for t in structure:
            if t == ch:
                lvl_index[(ch, k)] = k
                k += 1

    def f(axis, lv):           # factor of axis at level tag lv=(kind, k)
        return factors[axis][lv[1]]

    def axes_of(lv):
        return space if lv[0] == "S" else red

    n_threads = 1
    for lv in thread:
        for a in space:
            n_threads *= f(a, lv)
    n_blocks = 1
    for lv in block:
        for a in space:
            n_blocks *= f(a, lv)
    n_vthread = 1
    for lv in vthread:
        for a in space:
            n_vthread *= f(a, lv)
    if n_threads > MAX_THREADS:
        raise LoweringError(f"{n_threads} threads per block exceed {MAX_THREADS}")
    if n_vthread > MAX_VTHREAD:
        raise LoweringError(f"{n_vthread} virtual threads exceed {MAX_VTHREAD}")

    # per-thread register tile: vthread levels + inner space levels
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

    def digit(axis, lv):
        return f"{'s' if lv[0] == 'S' else 'r'}{(space if lv[0] == 'S' else red).index(axis)}_{lv[1]}"

    n_s = structure.count("S")
    n_r = structure.count("R")

    def mixed(axis, kind_, lo):
        """axis value from level `lo` inward (lo=0: global, lo=1: local)."""
        n_lv = n_s if kind_ == "S" else n_r
        expr = None
        for k in range(lo, n_lv):
            fac = factors[axis][k]
            if expr is None:
                expr = digit(axis, (kind_, k)) if fac > 1 else "0"
            elif fac > 1:
                expr = f"({expr})*{fac} + {digit(axis, (kind_, k))}"
        return expr or "0"

    def tile_span(axis, kind_):
        n_lv = n_s if kind_ == "S" else n_r
        t = 1
        for k in range(1, n_lv):
            t *= factors[axis][k]
        return t

    T = {a: tile_span(a, "S") for a in space}
    RT = {r: tile_span(r, "R") for r in red}

    # operands: distinct reads of the reduction body
    body = s.expr.body
    operands = []
    for r in reads(body):
        key = (r.buffer, tuple((l.terms, l.const) for l in r.index))
        if key not in [o["key"] for o in operands]:
            operands.append({"key": key, "read": r})
    attached_prod = {c.name for c in _attached(ctx.p, s.name) if _reads_buffer(s.expr, c.name)}

    smem_words = 0
    for oi, o in enumerate(operands):
        r = o["read"]
        hull, base_terms, off = [], [], []
        for lin in r.index:
            h = 1
            bt = [str(lin.const)] if lin.const else []
            of = 0
            for n, c in lin.terms:
                if n in T:
                    span, mn = T[n], f"{digit(n, ('S', 0))}*{T[n]}" if factors[n][0] > 1 else "0"
                elif n in RT:
                    span, mn = RT[n], f"{digit(n, ('R', 0))}*{RT[n]}" if factors[n][0] > 1 else "0"
                else:
                    raise LoweringError(f"read index uses iterator {n} outside the stage")
                h += abs(c) * (span - 1)
                if c >= 0:
                    bt.append(f"{c}*({mn})" if c != 1 else f"({mn})")
                else:
                    bt.append(f"{c}*({mn} + {span - 1})")
                    of += -c * (span - 1)
            hull.append(h)
            base_terms.append(" + ".join(bt) if bt else "0")
            off.append(of)
        size = 1
        for h in hull:
            size *= h
        o.update(hull=hull, base=base_terms, off=off, size=size, name=f"sm{oi}")
        smem_words += size
    smem_bytes = smem_words * 4 if d == "float" else smem_words * 8
    if smem_bytes > MAX_SMEM:
        raise LoweringError(f"shared memory {smem_bytes} bytes exceeds {MAX_SMEM}")

    # per-thread loop nest: vthread levels (always unrolled), then inner levels
    loop_list = []     # (digit var, extent, level, forced_unroll)
    for lv in vthread:
        for a in space:
            if f(a, lv) > 1:
                loop_list.append((digit(a, lv), f(a, lv), lv, True))
    for lv in inner:
        for a in axes_of(lv):
            if f(a, lv) > 1:
                loop_list.append((digit(a, lv), f(a, lv), lv, False))
    free = [x for x in loop_list if not x[3]]
    flags = _unroll_flags([x[1] for x in free], s.pragma_unroll)
    fl_iter = iter(flags)
    unroll = [True if x[3] else next(fl_iter) for x in loop_list]
    unrolled_stmts = 1
    for x, u in zip(loop_list, unroll):
        if u:
            unrolled_stmts *= x[1]
    if unrolled_stmts > MAX_UNROLLED:
        raise LoweringError(f"unrolled body of {unrolled_stmts} statements exceeds {MAX_UNROLLED}")
    unroll = promote_register_tile([x[1] for x in loop_list], unroll, [x[2][0] == "S" for x in loop_list],
                                   n_acc, n_threads)

    # accumulator index: per space axis, mixed radix over reg levels
    acc_idx_axis = []
    for a in space:
        e = None
        for lv in reg_levels:
            fac = f(a, lv)
            if fac == 1:
                continue
            dg = digit(a, lv)
            e = dg if e is None else f"({e})*{fac} + {dg}"
        acc_idx_axis.append(e or "0")
    acc_flat, mul = [], 1
    for a_i in range(len(space) - 1, -1, -1):
        acc_flat.append(f"({acc_idx_axis[a_i]})" if mul == 1 else f"({acc_idx_axis[a_i]})*{mul}")
        mul *= acc_dims[a_i]
    acc_index = " + ".join(reversed(acc_flat))

    glob = {a: mixed(a, "S", 0) for a in space}
    glob.update({r: mixed(r, "R", 0) for r in red})
    loc = {a: mixed(a, "S", 1) for a in space}
    loc.update({r: mixed(r, "R", 1) for r in red})

    def smem_read(buf, index, guarded=False):
        key = (buf, tuple((l.terms, l.const) for l in index))
        o = next(o for o in operands if o["key"] == key)
        coords = []
        for dd, lin in enumerate(index):
            parts = [str(o["off"][dd])] if o["off"][dd] else []
            for n, c in lin.terms:
                parts.append(f"({loc[n]})" if c == 1 else f"{c}*({loc[n]})")
            coords.append(" + ".join(parts) if parts else "0")
        flat, m = [], 1
        for dd in range(len(coords) - 1, -1, -1):
            flat.append(f"({coords[dd]})" if m == 1 else f"({coords[dd]})*{m}")
            m *= o["hull"][dd]
        return f"{o['name']}[{' + '.join(reversed(flat))}]"

    em = Emitter(d, lambda n: glob[n], smem_read)
    val = em(body)
    op = s.expr.op
    fsuf = "f" if d == "float" else ""
    init = _flt(0.0 if op == "sum" else -math.inf, d)

    L = []
    # digits from blockIdx / threadIdx (last axis fastest)
    L.append("  int bq_ = blockIdx.x;")
    for a in reversed(space):
        for lv in block:
            fac = f(a, lv)
            if fac > 1:
                L.append(f"  const int {digit(a, lv)} = bq_ % {fac}; bq_ /= {fac};")
    L.append("  int tq_ = threadIdx.x;")
    for a in reversed(space):
        for lv in thread:
            fac = f(a, lv)
            if fac > 1:
                L.append(f"  const int {digit(a, lv)} = tq_ % {fac}; tq_ /= {fac};")
    for o in operands:
        L.append(f"  {d}* {o['name']} = smem_ + {sum(p['size'] for p in operands[:operands.index(o)])};")
    L.append(f"  {d} acc_[{n_acc}];")
    L.append("  #pragma unroll")
    L.append(f"  for (int i_ = 0; i_ < {n_acc}; ++i_) acc_[i_] = {init};")
    ind = "  "
    stage_axes = [(r, f(r, stage_lv[0])) for r in red if f(r, stage_lv[0]) > 1]
    for r, e in stage_axes:
        L.append(f"{ind}#pragma unroll 1")
        L.append(f"{ind}for (int {digit(r, stage_lv[0])} = 0; {digit(r, stage_lv[0])} < {e}; ++{digit(r, stage_lv[0])}) {{")
        ind += "  "
    # cooperative fetch
    for o in operands:
        r = o["read"]
        hull = o["hull"]
        L.append(f"{ind}for (int e_ = threadIdx.x; e_ < {o['size']}; e_ += {n_threads}) {{")
        L.append(f"{ind}  int c_ = e_;")
        for dd in range(len(hull) - 1, -1, -1):
            L.append(f"{ind}  const int c{dd}_ = c_ % {hull[dd]}; c_ /= {hull[dd]};")
        idx = [f"({o['base'][dd]}) + c{dd}_" for dd in range(len(hull))]
        idx64 = [f"(long long)({o['base'][dd]}) + c{dd}_" for dd in range(len(hull))]
        if r.buffer in attached_prod:
            v = ctx.producer_call(r.buffer, idx)
        else:
            v = ctx.global_load(r.buffer, idx64)
        L.append(f"{ind}  {o['name']}[e_] = {v};")
        L.append(f"{ind}}}")
    L.append(f"{ind}__syncthreads();")
    cind = ind
    for (dg, e, lv, _), u in zip(loop_list, unroll):
        L.append(f"{cind}{_pragma(u)}")
        L.append(f"{cind}for (int {dg} = 0; {dg} < {e}; ++{dg}) {{")
        cind += "  "
    if op == "sum":
        L.append(f"{cind}acc_[{acc_index}] = acc_[{acc_index}] + {val};")
    else:
        L.append(f"{cind}acc_[{acc_index}] = fmax{fsuf}(acc_[{acc_index}], {val});")
    for _ in loop_list:
        cind = cind[:-2]
        L.append(f"{cind}}}")
    L.append(f"{ind}__syncthreads();")
    for _ in stage_axes:
        ind = ind[:-2]
        L.append(f"{ind}}}")
    # epilogue over the register tile
    reg_loops = []
    for lv in reg_levels:
        for a in space:
            if f(a, lv) > 1:
                reg_loops.append((digit(a, lv), f(a, lv)))
    eind = "  "
    ep_unroll = n_acc <= 256
    for dg, e in reg_loops:
        L.append(f"{eind}{_pragma(ep_unroll)}")
        L.append(f"{eind}for (int {dg} = 0; {dg} < {e}; ++{dg}) {{")
        eind += "  "
    # global coordinates need every digit: inner R digits are not involved
    idx_of = {a: f"gi{space.index(a)}_" for a in space}
    for a in space:
        L.append(f"{eind}const int {idx_of[a]} = {glob[a]};")
    L += _epilogue(ctx, s, idx_of, f"acc_[{acc_index}]", eind, _must_materialize(ctx, s))
    for _ in reg_loops:
        eind = eind[:-2]
        L.append(f"{eind}}}")

    # digits of inner space levels not in reg loops (factor 1) are folded to 0 by mixed()
    text = "\n".join(L)
    writes = _written(ctx, s)
    args = _kernel_args(ctx, writes)
    sig = _signature(ctx, entry, args, set(writes), n_threads)
    src = sig + " {\n" + f"  extern __shared__ {'float' if d == 'float' else 'double'} smem_[];\n" + text + "\n}\n"
    info = {"template": "tiled", "stage": s.name, "structure": structure, "threads": n_threads,
            "blocks": n_blocks, "vthreads": n_vthread, "acc": n_acc, "smem": smem_bytes,
            "unrolled": unrolled_stmts, "factors": {k: list(v) for k, v in factors.items()}}
    return src, Kernel(entry, n_blocks, n_threads, smem_bytes, args, info)


PRELUDE = """// generated by paper_2006_06762_b200.lower
#define INFINITY __int_as_float(0x7f800000)
"""


def lower(p, dtype: str = "float") -> Lowered:
    """Lower a concrete, validated State.  Raises LoweringError when the
    State has no legal GPU launch."""
    if not p.is_concrete():
        raise LoweringError("program has unresolved symbolic extents")
    ctx = _Ctx(p, dtype)
    sources, kernels = [], []
    for s in p.stages:
        if s.inlined or s.compute_at is not None:
            continue
        # attached chains must hang off this root: producers inline, consumers epilogue
        for c in _attached(p, s.name):
            if _attached(p, c.name) and any(_reads_buffer(c.expr, g.name) for g in _attached(p, c.name)):
                raise LoweringError(f"nested producer attachment under {c.name} is not supported")
        entry = f"k{len(kernels)}_" + ident(s.name)
        ctx.refs = []
        levels = tile_levels(p, s)
        if levels is not None:
            src, k = _tiled_kernel(ctx, s, levels, entry)
        else:
            src, k = _naive_kernel(ctx, s, entry)
        sources.append(src)
        kernels.append(k)
    for name, st in ctx.live.items():
        if name not in ctx.buffers:
            role = "output" if name in p.dag.outputs else "temp"
            ctx.buffers[name] = Buffer(name, tuple(e for _, e in st.space), role)
    source = PRELUDE + "\n".join(ctx.helpers) + "\n" + "\n".join(sources)
    info = {"kernels": [k.info for k in kernels]}
    return Lowered(source, kernels, ctx.buffers, list(p.dag.outputs), info)


def reference_lowering(dag) -> Lowered:
    """State-free fp64 ground truth of a DAG: one naive fp64 kernel per computed
    node in dependency order (the device analogue of `reference_outputs`,
    `src/interp.py:46-74`)."""
    from .state import naive_program
    return lower(naive_program(dag), dtype="double")
