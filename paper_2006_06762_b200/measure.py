"""GPU measurement: drop-in for the reference's `measure_batch`
(`src/machine.py:249-285`) with the same signature, result type and status
semantics.

Per candidate: `validate` (host, reference messages) -> lower to CUDA
(`lower.py`) -> compile with exact constants in the multi-process NVRTC pool
(cached on disk) -> run on the B200, verify every output against an fp64
ground truth on the device (max relative error <= `GPU_TOL`, the north star's
1e-4 for fp32) -> time with CUDA events.  `cost` is device microseconds.

Timing: one warm-up run (also verified), then, if it was shorter than
`min_ms` (1 ms), timed repeats until the timed region spans `min_ms`; a run of
at least `min_ms` is its own measurement unless a kernel of the candidate uses
local memory (spilling kernels pay for growing the local-memory pool on their
first launch, so they always get a timed run).  CUDA events on the task stream.

Statuses: INVALID (validation failure, no legal launch, compile/launch
failure, or wrong output — detail says which), TIMEOUT (cost >=
`limits.cost_ceiling`, read in microseconds), VALID.  Throughput is
`min(valid costs, best_cost) / cost` exactly as the reference normalises
(`src/machine.py:276-285`).  `spec` (the CPU machine model) is accepted and
ignored.  Inputs are `random_inputs(dag, default_rng(limits.check_seed))`
(`src/interp.py:38-43`), generated once per DAG and kept resident in HBM.
"""

from __future__ import annotations

import atexit
import ctypes
# imported before `atexit.register(_shutdown)` below: multiprocessing registers its
# own exit hook (joining non-daemon children) at import, and atexit runs hooks in
# reverse order, so the measuring process is told to close before it is joined
import multiprocessing.util  # noqa: F401
import hashlib
import queue
import threading
import json
import math
import os
import pickle
import sys
import time
from collections import OrderedDict
from dataclasses import dataclass, field, replace

import numpy as np

from . import runtime as rt
from .lower import Lowered, LoweringError, lower, reference_lowering
from .ptxgen import Unsupported, lower_ptx
from .state import history_to_json, validate

VALID, INVALID, TIMEOUT = "valid", "invalid", "timeout"
GPU_TOL = 1e-4
NVRTC_OPTS = "--gpu-architecture=sm_100a\n-default-device\n-lineinfo"
# --allow-expensive-optimizations=false: 12% less ptxas time (the bound on
# candidates/sec), identical kernel times on the golden streams (template_bench A/B)
PTX_OPTS = "--ptx\n--gpu-name=sm_100a\n" + os.environ.get("LT_PTXAS_OPT",
                                                          "-O3\n--allow-expensive-optimizations=false")
# ptxas has been seen to miscompile heavily spilling kernels (wrong values /
# out-of-range shared loads, valid at -O1 and through NVRTC): a PTX candidate
# whose output fails verification is recompiled once at -O1 and re-measured.
PTX_SAFE_OPTS = "--ptx\n--gpu-name=sm_100a\n-O1"
_TRACE = bool(os.environ.get("LT_TRACE"))


@dataclass(frozen=True)
class MeasureResult:
    """Same fields as `src/machine.py:51-56`."""
    cost: float
    throughput: float
    status: str
    detail: str = ""


@dataclass(frozen=True)
class MeasureLimits:
    """Same fields as `src/machine.py:241-246`; cost_ceiling is in microseconds here."""
    cost_ceiling: float | None = None
    check_cap: int = 8
    check_tol: float = 1e-5
    check_seed: int = 0


@dataclass
class Record:
    """Per-candidate telemetry (logged beside MeasureResult)."""
    status: str = INVALID
    detail: str = ""
    cost_us: float = math.inf
    first_us: float = 0.0
    max_rel_err: float = math.nan
    repeats: int = 0
    compile_s: float = 0.0
    cache_hit: bool = False
    lower_s: float = 0.0
    n_outputs: int = 0
    info: dict = field(default_factory=dict)
    key: str = ""             # sha1 of the candidate's generated source
    done: bool = False        # final (False: not reached before a fault ended the batch)
    t: dict = field(default_factory=dict)   # batch timeline (s from the batch start): lowered, start, end


def random_inputs(dag, seed: int) -> dict:
    """`random_inputs` (`src/interp.py:38-43`): U(0.25, 1) per placeholder in node order."""
    rng = np.random.default_rng(seed)
    return {n.name: rng.uniform(0.25, 1.0, size=n.shape) for n in dag.nodes if n.is_placeholder}


def pack_strides(shape, desc) -> tuple:
    """Device packing parameters of a packed constant (`lt_task_pack`): the physical
    extents (outer to inner) and, per physical dim, the step it makes in the flat
    row-major offset of the logical array -- the same index map as `pack`."""
    shape = tuple(int(x) for x in shape)
    lst = [1] * len(shape)
    for d in range(len(shape) - 2, -1, -1):
        lst[d] = lst[d + 1] * shape[d + 1]
    ext, mult = [], []
    for j, (d, e) in enumerate(desc):
        st = 1
        for d2, e2 in desc[j + 1:]:
            if d2 == d:
                st *= e2
        ext.append(int(e))
        mult.append(st * lst[d])
    for d in range(len(shape)):
        tot = 1
        for d2, e2 in desc:
            if d2 == d:
                tot *= e2
        if tot != shape[d]:
            raise ValueError(f"packed layout {desc} does not tile dim {d} of {shape}")
    return np.asarray(ext, np.int64), np.asarray(mult, np.int64)


def pack(arr: np.ndarray, desc) -> np.ndarray:
    """Physical layout of a packed constant (LayoutRewrite, `src/ir.py:747-760`):
    one physical dim per descriptor entry, outer to inner."""
    phys_shape = tuple(e for _, e in desc)
    grids = np.indices(phys_shape)
    idx = [np.zeros(phys_shape, dtype=np.int64) for _ in range(arr.ndim)]
    for j, (d, e) in enumerate(desc):
        st = 1
        for d2, e2 in desc[j + 1:]:
            if d2 == d:
                st *= e2
        idx[d] = idx[d] + grids[j] * st
    return arr[tuple(idx)]


def _dag_key(dag, seed: int) -> str:
    return hashlib.sha1((json.dumps(dag.to_json(), sort_keys=True) + f"#{seed}").encode()).hexdigest()


class _DagContext:
    """Device-resident state for one DAG: inputs (fp32 + fp64), fp64 ground truth,
    packed constants, candidate scratch buffers."""

    def __init__(self, runner: "Runner", dag, seed: int):
        self.r = runner
        self.dag = dag
        lib = runner.lib
        self.task = lib.lt_task_create(runner.device)
        if not self.task:
            raise rt.NativeError(lib.lt_last_error().decode())
        self.slots: dict = {}
        self.sizes: dict = {}
        self.pinned: list = []
        self.packed: dict = {}          # slot key -> (source, descriptor) its device copy currently holds
        self.inputs = random_inputs(dag, seed)
        self.h2d_bytes = 0
        # host copies of the inputs, page-locked once: every upload (the first and
        # each end-to-end refresh) is a DMA from pinned memory
        self.host: dict = {}
        for name, arr in self.inputs.items():
            for key, dt in ((f"in:{name}", np.float32), (f"in64:{name}", np.float64)):
                h = np.ascontiguousarray(arr, dtype=dt)
                self._pin(h)
                self.host[key] = h
                self._upload(key, h)
        # fp64 ground truth, computed once on the device from the fp64 inputs
        ref = reference_lowering(dag)
        funcs = runner.compile_and_load([ref.source], [[k.entry for k in ref.kernels]])[0]
        runner.pinned.add(hashlib.sha1(ref.source.encode()).hexdigest())
        if isinstance(funcs, str):
            raise rt.NativeError(f"ground-truth kernel failed to compile: {funcs}")
        for name, b in ref.buffers.items():
            if b.role in ("temp", "output"):
                self.slot(f"ref:{name}", b.numel * 8)
        self._ref = (ref, funcs)
        launches = self._launches(ref, funcs, fp64=True)
        rt.check(lib.lt_task_run(self.task, ctypes.addressof(launches), len(ref.kernels)), "ground truth")
        self.outputs = list(ref.outputs)

    def refresh(self) -> None:
        """Re-upload every input (fp32 + fp64) and packed constant (packed once,
        as Ansor's layout rewrite packs constants offline) into its existing
        slot and recompute the fp64 ground truth: the per-step host->device work
        of an end-to-end run."""
        for key, h in self.host.items():
            self._upload(key, h)
        self.packed.clear()                             # re-packed on the device at next use
        ref, funcs = self._ref
        launches = self._launches(ref, funcs, fp64=True)
        rt.check(self.r.lib.lt_task_run(self.task, ctypes.addressof(launches), len(ref.kernels)), "ground truth")

    def _pin(self, arr: np.ndarray) -> None:
        if arr.nbytes:
            rt.check(self.r.lib.lt_host_register(arr.ctypes.data, arr.nbytes), "pin input")
            self.pinned.append(arr)

    def release(self) -> None:
        """Destroy the device task and unpin the host copies."""
        self.r.lib.lt_task_destroy(self.task)
        for arr in self.pinned:
            self.r.lib.lt_host_unregister(arr.ctypes.data)
        self.pinned.clear()

    def slot(self, key: str, nbytes: int) -> int:
        if key not in self.slots:
            self.slots[key] = len(self.slots)
        if self.sizes.get(key, -1) < nbytes:
            rt.check(self.r.lib.lt_task_slot(self.task, self.slots[key], nbytes), f"alloc {key}")
            self.sizes[key] = nbytes
        return self.slots[key]

    def _upload(self, key: str, arr: np.ndarray) -> int:
        sid = self.slot(key, arr.nbytes)
        rt.check(self.r.lib.lt_task_upload(self.task, sid, arr.ctypes.data, arr.nbytes), f"upload {key}")
        self.h2d_bytes += arr.nbytes
        self.r.io["h2d"] += arr.nbytes
        return sid

    def buffer_slot(self, b, fp64: bool) -> int:
        if b.role == "input":
            return self.slots[f"in64:{b.name}" if fp64 else f"in:{b.name}"]
        if b.role == "packed":
            # one slot per packed buffer name, re-laid out on the device (a stream-ordered
            # gather, microseconds) whenever a candidate asks for another descriptor: no
            # host packing, no pinning, no allocation per layout
            key = f"pk:{b.name}"
            sid = self.slot(key, b.numel * 4)
            if self.packed.get(key) != (b.source, b.desc):
                ext, mult = pack_strides(self.inputs[b.source].shape, b.desc)
                rt.check(self.r.lib.lt_task_pack(self.task, sid, self.slots[f"in:{b.source}"], len(ext),
                                                 rt.ptr(ext, rt.c_i64p), rt.ptr(mult, rt.c_i64p)),
                         "pack constant")
                self.packed[key] = (b.source, b.desc)
            return sid
        if fp64:
            return self.slots[f"ref:{b.name}"]
        return self.slot(f"buf:{b.name}", b.numel * 4)

    def _launches(self, lo: Lowered, funcs: list, fp64: bool = False):
        arr = (rt.Launch * len(lo.kernels))()
        for i, (k, fn) in enumerate(zip(lo.kernels, funcs)):
            L = arr[i]
            L.func = fn
            L.grid[:] = (k.grid, 1, 1)
            L.block[:] = (k.block, 1, 1)
            L.smem = k.smem
            L.n_args = len(k.args)
            for a, name in enumerate(k.args):
                L.arg_slot[a] = self.buffer_slot(lo.buffers[name], fp64)
        return arr

    def measure(self, lo: Lowered, funcs: list, min_ms: float, max_repeat: int,
                min_repeat: int = 1) -> rt.MeasureRecord:
        t0 = time.perf_counter()
        launches = self._launches(lo, funcs)
        pairs, numel = [], []
        for name in lo.outputs:
            b = lo.buffers[name]
            pairs += [self.buffer_slot(b, False), self.slots[f"ref:{name}"]]
            numel.append(b.numel)
        # intermediate buffers are shared by every candidate of the DAG: NaN-poison
        # them too, so a candidate cannot pass on values an earlier one left there
        for b in lo.buffers.values():
            if b.role == "temp" and b.name not in lo.outputs:
                rt.check(self.r.lib.lt_task_fill(self.task, self.buffer_slot(b, False), b.numel, 0x7FC00000),
                         "poison temp")
        pairs_a = np.asarray(pairs, np.int32)
        numel_a = np.asarray(numel, np.int64)
        rec = rt.MeasureRecord()
        t1 = time.perf_counter()
        rt.check(self.r.lib.lt_measure(self.task, ctypes.addressof(launches), len(lo.kernels),
                                       rt.ptr(pairs_a, rt.c_i32p), rt.ptr(numel_a, rt.c_i64p), len(numel),
                                       min_repeat, max_repeat, min_ms, ctypes.addressof(rec)), "lt_measure")
        st = self.r.stats
        st["prep_s"] += t1 - t0
        st["lt_measure_s"] += time.perf_counter() - t1
        return rec

    def download(self, name: str, numel: int, fp64: bool = False) -> np.ndarray:
        out = np.empty(numel, np.float64 if fp64 else np.float32)
        key = f"ref:{name}" if fp64 else f"buf:{name}"
        rt.check(self.r.lib.lt_task_download(self.task, self.slots[key], out.ctypes.data, out.nbytes), "download")
        return out


def _modules_of(lo: Lowered) -> list:
    """[(entries, module source, compile options)]: PTX candidates compile one
    module per kernel, so a kernel shared by many candidates (a materialised
    padding stage, an unchanged consumer) is assembled once; CUDA C candidates
    stay one NVRTC module."""
    if not lo.source.startswith(".version"):
        return [([k.entry for k in lo.kernels], lo.source, None)]
    head, _, rest = lo.source.partition(".visible .entry ")
    bodies = [".visible .entry " + b for b in rest.split(".visible .entry ")]
    out = []
    for k, body in zip(lo.kernels, bodies):
        if not body.startswith(f".visible .entry {k.entry}("):
            raise LoweringError(f"module split mismatch at {k.entry}")
        out.append(([k.entry], head + body, PTX_SAFE_OPTS if k.info.get("ptxas") else None))
    return out


def _lower_one(p, backend: str):
    """validate + lower one State (runs in a lowering worker process).
    Returns (kind, payload, seconds): ("bad", detail) | ("err", detail) | ("ok", Lowered)."""
    t0 = time.perf_counter()
    bad = validate(p)
    if bad:
        return "bad", bad[0], 0.0
    try:
        lo = None
        if backend == "ptx":
            try:
                lo = lower_ptx(p)
            except Unsupported:
                pass
        if lo is None:
            lo = lower(p)
    except LoweringError as e:
        return "err", f"gpu: {e}", time.perf_counter() - t0
    return "ok", lo, time.perf_counter() - t0


class RunnerCore:
    """The GPU runner proper (lives in the measuring process, see `Runner`): one
    device, one compile pool, DAG contexts, module cache.

    Host work per candidate (validate + lowering, pure Python) runs in a pool of
    lowering processes so it neither serialises the batch nor holds the GIL the
    measurement thread needs between device calls."""

    def __init__(self, device: int = 0, workers: int | None = None, cache_dir: str | None = None,
                 min_ms: float = 1.0, max_repeat: int = 50, compile_timeout: float = 120.0,
                 min_repeat: int = 0, backend: str = "ptx", lower_workers: int | None = None,
                 first_run_timing: bool = True):
        self.lib = rt.load()
        self.device = device
        rt.check(self.lib.lt_set_device(device), "set device")
        self.workers = workers or max(1, (os.cpu_count() or 2) - 1)
        self.cache_dir = cache_dir if cache_dir is not None else os.environ.get(
            "LT_CUBIN_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "loomtune_b200", "cubin"))
        self.compile_timeout = compile_timeout
        rt.check(self.lib.lt_pool_start(self.workers, self.cache_dir.encode() if self.cache_dir else None,
                                        compile_timeout), "compile pool")
        self.min_ms, self.max_repeat, self.min_repeat = min_ms, max_repeat, min_repeat
        self.first_run_timing = first_run_timing
        self._local_bytes: dict = {}       # function handle -> local memory bytes per thread
        self.backend = backend
        self.ctx: dict = {}
        self._dag_keys: dict = {}          # (id(dag), seed) -> (dag, content key)
        self.modules: OrderedDict = OrderedDict()   # source hash -> (module, funcs)
        self.pinned: set = set()                      # ground-truth modules (held by DAG contexts)
        self.images: OrderedDict = OrderedDict()      # module key -> cubin (reload after a reset)
        self.mod_lock = threading.Lock()
        self.failed_keys: dict = {}
        self._drain_error = None
        self.stats = {"compiled": 0, "recompiled": 0, "cache_hits": 0, "compile_s": 0.0, "measured": 0,
                      "kernels_compiled": 0, "kernels_shared": 0,
                      "lower_s": 0.0, "gpu_s": 0.0, "load_s": 0.0, "idle_s": 0.0, "wall_s": 0.0,
                      "prep_s": 0.0, "lt_measure_s": 0.0}
        self.io = {"h2d": 0, "d2h": 0}      # host<->device bytes (inputs, cubins, launch lists / errors)
        self.last_records: list = []
        self.max_modules = 512          # loaded candidate modules kept (LRU)
        self.lower_workers = (lower_workers if lower_workers is not None
                              else int(os.environ.get("LT_LOWER_WORKERS", max(1, min(8, (os.cpu_count() or 2) // 2)))))
        self._lpool = None
        self.faulted = False            # a candidate faulted: this process's CUDA state is lost
        self._batch_seq = 0             # compile-pool priority of the batch being measured
        self._stage_thread = None       # lowering + compiling the next batch (see stage)
        self._staged: dict = {}
        self._staged_for = -1
        self.force_recompile = False    # test hook: treat every first verification as failed

    def _lower_pool(self):
        main = sys.modules.get("__main__")
        main_file = getattr(main, "__file__", None)
        if main_file is not None and not os.path.exists(main_file):
            return None             # spawn cannot re-import a stdin/REPL __main__: lower in-process
        if self._lpool is None and self.lower_workers > 1:
            import multiprocessing as mp
            from concurrent.futures import ProcessPoolExecutor
            self._lpool = ProcessPoolExecutor(self.lower_workers, mp_context=mp.get_context("spawn"))
        return self._lpool

    def forget_compiled(self, cache_dir: str) -> None:
        """Drop every compiled module and restart the compile pool on `cache_dir`
        (benchmarks re-measuring the same States from scratch)."""
        with self.mod_lock:
            for k in [k for k in self.modules if k not in self.pinned]:
                self.lib.lt_module_unload(self.modules.pop(k)[0])
            self._local_bytes.clear()
            self.failed_keys.clear()
        self.lib.lt_pool_stop()
        self.cache_dir = cache_dir
        rt.check(self.lib.lt_pool_start(self.workers, cache_dir.encode() if cache_dir else None,
                                        self.compile_timeout), "compile pool")

    def abandon(self):
        """After a fault: stop the host-side pools (no CUDA calls: the context is dead)."""
        if self._lpool is not None:
            self._lpool.shutdown(wait=False, cancel_futures=True)
            self._lpool = None
        self.lib.lt_pool_stop()

    def close(self):
        if self._lpool is not None:
            self._lpool.shutdown(wait=False, cancel_futures=True)
            self._lpool = None
        for m, _ in self.modules.values():
            self.lib.lt_module_unload(m)
        self.modules.clear()
        for c in self.ctx.values():
            c.release()
        self.ctx.clear()
        self.lib.lt_pool_stop()

    def context(self, dag, seed: int) -> _DagContext:
        hit = self._dag_keys.get((id(dag), seed))
        if hit is None or hit[0] is not dag:
            hit = (dag, _dag_key(dag, seed))
            self._dag_keys[(id(dag), seed)] = hit
        key = hit[1]
        if key not in self.ctx:
            self.ctx[key] = _DagContext(self, dag, seed)
        return self.ctx[key]

    # -- compile + load ------------------------------------------------------
    def submit(self, source: str, opts: str | None = None, prio: int = 0) -> int:
        b = source.encode()
        if opts is None:
            opts = PTX_OPTS if source.startswith(".version") else NVRTC_OPTS
        return self.lib.lt_compile_submit_prio(b, len(b), opts.encode(), prio)

    def lower(self, p) -> Lowered:
        """PTX backend by default; NVRTC (CUDA C) for what PTX does not express."""
        if self.backend == "ptx":
            try:
                return lower_ptx(p)
            except Unsupported:
                pass
        return lower(p)

    def collect(self, job: int):
        st, secs, hit, n = ctypes.c_int(), ctypes.c_double(), ctypes.c_int(), ctypes.c_int64()
        rt.check(self.lib.lt_compile_wait(job, ctypes.byref(st), ctypes.byref(secs), ctypes.byref(hit),
                                          ctypes.byref(n)), "compile wait")
        buf = ctypes.create_string_buffer(max(1, n.value))
        rt.check(self.lib.lt_compile_fetch(job, buf, n.value), "compile fetch")
        return st.value, secs.value, bool(hit.value), buf.raw[:n.value]

    def load(self, key: str, image: bytes, entries: list) -> list:
        with self.mod_lock:
            if key in self.modules:
                self.modules.move_to_end(key)
                return self.modules[key][1]
            if image:
                self.images[key] = image        # kept to reload after a device reset
                while len(self.images) > 1024:
                    self.images.pop(next(iter(self.images)))
            else:
                image = self.images.get(key, b"")
        m = self.lib.lt_module_load(self.device, image, len(image))
        self.io["h2d"] += len(image)
        if not m:
            raise rt.NativeError(f"module load: {self.lib.lt_last_error().decode()}")
        funcs = []
        for e in entries:
            f = self.lib.lt_module_function(m, e.encode())
            if not f:
                raise rt.NativeError(f"function {e}: {self.lib.lt_last_error().decode()}")
            funcs.append(f)
        with self.mod_lock:
            self.modules[key] = (m, funcs)
            while len(self.modules) > self.max_modules:     # LRU, never the ground-truth modules
                victim = next((k for k in self.modules if k not in self.pinned), None)
                if victim is None:
                    break
                old, _ = self.modules.pop(victim)
                self.lib.lt_module_unload(old)
                self._local_bytes.clear()       # a handle value may be handed out again
        return funcs

    def compile_and_load(self, sources: list, entries: list) -> list:
        jobs = [self.submit(s) for s in sources]
        out = []
        for s, j, e in zip(sources, jobs, entries):
            st, secs, hit, data = self.collect(j)
            if st != 0:
                out.append(data.decode(errors="replace"))
            else:
                out.append(self.load(hashlib.sha1(s.encode()).hexdigest(), data, e))
        return out

    # -- measurement ---------------------------------------------------------
    def _parts(self, lo: Lowered, batch_keys: dict, prio: int) -> list:
        """[(entries, kernel key, job | None | ("dup", key))] for one lowered
        candidate: loaded kernels are reused, a kernel already submitted for this
        batch is shared, every other kernel module is submitted (priority `prio`)."""
        parts = []
        for ents, text, opts in _modules_of(lo):
            kkey = hashlib.sha1((opts or "").encode() + text.encode()).hexdigest()
            with self.mod_lock:
                loaded = kkey in self.modules
            if loaded:
                parts.append((ents, kkey, None))
            elif kkey in batch_keys:                 # same kernel in another candidate
                parts.append((ents, kkey, ("dup", kkey)))
                self.stats["kernels_shared"] += 1
            else:
                job = self.submit(text, opts, prio)
                batch_keys[kkey] = job
                parts.append((ents, kkey, job))
        return parts

    @staticmethod
    def _program_key(p, dag_json: dict) -> str:
        d = dag_json.get(id(p.dag))
        if d is None:
            d = dag_json[id(p.dag)] = json.dumps(p.dag.to_json(), sort_keys=True)
        return hashlib.sha1((d + json.dumps(history_to_json(p.history))).encode()).hexdigest()

    def stage(self, programs: list) -> None:
        """Start lowering and compiling a LATER batch now, in the background: its
        compile jobs queue behind every job of the batch being measured (pool
        priority), so they only fill cores that batch leaves idle (its tail).
        The next `measure_programs` call picks up whatever is staged for its
        programs; nothing is measured here."""
        prio = self._batch_seq + 1
        staged: dict = {}
        self._staged_for, self._staged = prio, staged

        def work():
            dag_json: dict = {}
            batch_keys: dict = {}
            for i, p, res in self._lowered(programs):
                parts = self._parts(res[1], batch_keys, prio) if res[0] == "ok" else None
                staged[self._program_key(p, dag_json)] = (res, parts)
        self._stage_thread = threading.Thread(target=work, daemon=True)
        self._stage_thread.start()

    def measure_programs(self, programs: list, seed: int = 0, stage: list | None = None) -> list:
        """Validate + lower on this thread while a measurement thread drains
        finished compiles onto the GPU (ctypes drops the GIL inside lt_measure).
        `stage`: the programs of the next batch, lowered and compiled behind this
        one (see `stage`)."""
        t_start = time.perf_counter()
        self._t_batch = t_start
        self._batch_seq += 1
        prio = self._batch_seq
        staged: dict = {}
        if self._stage_thread is not None:
            self._stage_thread.join()
            self._stage_thread = None
            if self._staged_for == prio:
                staged = self._staged
            self._staged = {}
        recs = [Record() for _ in programs]
        for p in programs:                       # device contexts are created up front
            self.context(p.dag, seed)
        dag_json: dict = {}
        ready, fresh = [], []
        for i, p in enumerate(programs):
            hit = staged.pop(self._program_key(p, dag_json), None) if staged else None
            (ready if hit is not None else fresh).append((i, p, hit))
        self.stats["staged"] = self.stats.get("staged", 0) + len(ready)
        if stage:
            self.stage(list(stage))
        q: queue.Queue = queue.Queue()
        worker = threading.Thread(target=self._drain, args=(q, recs, seed), daemon=True)
        worker.start()
        batch_keys: dict = {}
        try:
            # compile jobs are submitted as lowerings finish; the pool hands the
            # largest pending source to each free worker (longest-processing-time
            # first), which shortens the batch's tail
            def results():
                for i, p, (res, parts) in ready:
                    yield i, p, res, parts
                for i, p, res in self._lowered([p for _, p, _ in fresh]):
                    yield fresh[i][0], p, res, None
            for i, p, (kind_, payload, secs), parts in results():
                recs[i].lower_s = secs
                recs[i].t["lowered"] = time.perf_counter() - t_start
                self.stats["lower_s"] += secs
                if kind_ != "ok":
                    recs[i].detail = payload
                    recs[i].done = True
                    continue
                lo = payload
                recs[i].info = lo.info
                key = hashlib.sha1(lo.source.encode()).hexdigest()
                recs[i].key = key
                if parts is None:
                    parts = self._parts(lo, batch_keys, prio)
                q.put((i, p, lo, key, parts))
        finally:
            q.put(None)
            worker.join()
        if self._drain_error is not None:
            err, self._drain_error = self._drain_error, None
            raise err
        self.last_records = recs
        self.stats["wall_s"] += time.perf_counter() - t_start
        return recs

    def _lowered(self, programs: list):
        """(index, program, lowering result) in completion order."""
        pool = self._lower_pool() if len(programs) > 1 else None
        done: set = set()
        if pool is not None:
            from concurrent.futures import as_completed
            from concurrent.futures.process import BrokenProcessPool
            try:
                futs = {pool.submit(_lower_one, p, self.backend): i for i, p in enumerate(programs)}
                for f in as_completed(futs):
                    i = futs[f]
                    res = f.result()
                    done.add(i)
                    yield i, programs[i], res
                return
            except (BrokenProcessPool, OSError, pickle.PicklingError) as e:    # host-side only: lower here
                self._lpool = None
                self.stats["lower_pool_error"] = repr(e)
        for i, p in enumerate(programs):
            if i not in done:
                yield i, p, _lower_one(p, self.backend)

    def _ready(self, item) -> bool:
        for _, kkey, job in item[4]:
            if job is None:
                continue
            if isinstance(job, tuple):
                # the other candidate's compile has landed: loaded, failed, or
                # loaded and already evicted by the LRU (reloaded from its image)
                with self.mod_lock:
                    if not (kkey in self.modules or kkey in self.failed_keys or kkey in self.images):
                        return False
            elif self.lib.lt_compile_ready(job) == 0:
                return False
        return True

    def _drain(self, q, recs, seed) -> None:
        waiting, closed = [], False
        try:
            while True:
                while True:
                    try:
                        item = q.get_nowait() if (waiting or closed) else q.get(timeout=0.05)
                    except queue.Empty:
                        break
                    if item is None:
                        closed = True
                    else:
                        waiting.append(item)
                if self.faulted:                # the rest of the batch goes to a fresh process
                    waiting.clear()
                    if closed:
                        return
                    time.sleep(0.0005)
                    continue
                idx = next((k for k, x in enumerate(waiting) if self._ready(x)), None)
                if idx is None:
                    if closed and not waiting:
                        return
                    t0 = time.perf_counter()
                    jobs = [job for x in waiting for _, _, job in x[4]
                            if isinstance(job, int) and self.lib.lt_compile_ready(job) == 0]
                    if jobs:        # sleep in the pool until a compile lands (GIL released)
                        arr = np.asarray(jobs, np.int64)
                        self.lib.lt_compile_wait_any(rt.ptr(arr, rt.c_i64p), len(jobs), 0.002)
                    else:
                        time.sleep(0.0005)
                    self.stats["idle_s"] += time.perf_counter() - t0
                    continue
                self._measure_one(waiting.pop(idx), recs, seed)
        except BaseException as e:          # surfaced on the calling thread
            self._drain_error = e
            while not closed:
                if q.get() is None:
                    closed = True

    def _measure_one(self, item, recs, seed) -> None:
        i, p, lo, key, parts = item
        rec = recs[i]
        rec.done = True
        entries = [k.entry for k in lo.kernels]
        funcs, compiled, rec.cache_hit = [], False, True
        for ents, kkey, job in parts:
            if job is None or isinstance(job, tuple):
                with self.mod_lock:
                    if kkey in self.failed_keys:
                        rec.detail = self.failed_keys[kkey]
                        return
                funcs += self.load(kkey, b"", ents)
                continue
            st, secs, hit, data = self.collect(job)
            rec.compile_s += secs
            rec.cache_hit = rec.cache_hit and hit
            compiled = compiled or not hit
            self.stats["compile_s"] += secs
            self.stats["kernels_compiled"] += 0 if hit else 1
            if st != 0:
                rec.detail = "gpu: compile failed: " + data.decode(errors="replace").strip()[:300]
                with self.mod_lock:
                    self.failed_keys[kkey] = rec.detail
                return
            t0 = time.perf_counter()
            funcs += self.load(kkey, data, ents)
            self.stats["load_s"] += time.perf_counter() - t0
        self.stats["compiled" if compiled else "cache_hits"] += 1
        ctx = self.context(p.dag, seed)
        if _TRACE:
            print(f"[lt trace] measuring #{i} {key[:12]} {[k.info.get('template') for k in lo.kernels]}",
                  file=sys.stderr, flush=True)
        t0 = time.perf_counter()
        rec.t["start"] = t0 - self._t_batch
        m = ctx.measure(lo, funcs, self.min_ms, self.max_repeat, self._min_repeat(funcs))
        rec.t["end"] = time.perf_counter() - self._t_batch
        if m.status == 2:
            # a faulting candidate is INVALID like any other failure (SPEC.md:522:
            # measure_batch never raises); the process's CUDA state is gone, so the
            # batch stops here and the parent carries on in a fresh measuring process
            rec.detail = "gpu: " + m.detail.decode(errors="replace")
            self.faulted = True
            return
        self.stats["gpu_s"] += time.perf_counter() - t0
        self.stats["measured"] += 1
        self.io["d2h"] += 4                                 # the max-relative-error word
        rec.first_us, rec.repeats = m.first_us, m.repeats
        rec.n_outputs = len(lo.outputs)
        rec.max_rel_err = float(m.max_rel_err)
        if m.status != 0:
            rec.detail = "gpu: " + m.detail.decode(errors="replace")
            return
        if self.force_recompile and lo.source.startswith(".version"):
            rec.max_rel_err = math.inf                      # test hook: exercise the recompile path
        if not (rec.max_rel_err <= GPU_TOL) and lo.source.startswith(".version") and m.status == 0:
            o1 = lo.info.get("ptxas_opt") == "-O1"
            m2 = self._remeasure_safe(lo, key, entries, ctx, PTX_OPTS if o1 else PTX_SAFE_OPTS)
            if self.faulted:
                rec.detail = "gpu: kernel fault (recompiled after failing verification)"
                return
            if m2 is not None and m2.status == 0:
                m = m2
                rec.first_us, rec.repeats = m.first_us, m.repeats
                rec.max_rel_err = float(m.max_rel_err)
                rec.info = {**rec.info, "ptxas": ("-O3 (the -O1 build failed verification)" if o1 else
                                                  "-O1 (the -O3 build failed verification)")}
        if (not (rec.max_rel_err <= GPU_TOL) and lo.source.startswith(".version") and m.status == 0
                and not self.faulted and os.environ.get("LT_NVRTC_FALLBACK", "1") != "0"):
            # both ptxas levels produced wrong values (seen on register-overflowing
            # tiles): the same State through the CUDA C lowering and NVRTC, verified again
            m3 = self._remeasure_nvrtc(p, key, ctx)
            if self.faulted:
                rec.detail = "gpu: kernel fault (NVRTC build after failing verification)"
                return
            if m3 is not None and m3.status == 0 and m3.max_rel_err <= GPU_TOL:
                m = m3
                rec.first_us, rec.repeats = m.first_us, m.repeats
                rec.max_rel_err = float(m.max_rel_err)
                rec.info = {**rec.info, "ptxas": "NVRTC (both PTX builds failed verification)"}
        if not (rec.max_rel_err <= GPU_TOL):
            names = ",".join(lo.outputs)
            rec.detail = f"output {names} differs from reference (max rel err {rec.max_rel_err:.3g})"
            return
        rec.status = VALID
        rec.cost_us = m.cost_us

    def _min_repeat(self, funcs: list) -> int:
        """Timed runs after the verified warm-up: a candidate whose kernels use no
        local memory and whose warm-up run already spans `min_ms` is timed by that
        run (0); kernels that spill keep >= 1 timed run, because their first launch
        also pays for growing the local-memory pool (measured up to 300x)."""
        if self.min_repeat > 0 or not self.first_run_timing:
            return max(1, self.min_repeat)
        for f in funcs:
            if f not in self._local_bytes:
                regs, local, mt, sm = (ctypes.c_int() for _ in range(4))
                rt.check(self.lib.lt_function_info(f, ctypes.byref(regs), ctypes.byref(local), ctypes.byref(mt),
                                                   ctypes.byref(sm)), "function info")
                self._local_bytes[f] = local.value
            if self._local_bytes[f]:
                return 1
        return 0

    def _remeasure_nvrtc(self, p, key, ctx):
        """Lower the State to CUDA C (`lower.lower`), compile it with NVRTC and measure it
        (None when it does not lower or compile)."""
        try:
            lo2 = lower(p)
        except (LoweringError, Unsupported):
            return None
        st, secs, hit, data = self.collect(self.submit(lo2.source))
        self.stats["compile_s"] += secs
        self.stats["recompiled"] = self.stats.get("recompiled", 0) + 1
        if st != 0:
            return None
        funcs = self.load(key + ":nvrtc", data, [k.entry for k in lo2.kernels])
        t0 = time.perf_counter()
        m = ctx.measure(lo2, funcs, self.min_ms, self.max_repeat, self.min_repeat)
        if m.status == 2:
            self.faulted = True
            return None
        self.stats["gpu_s"] += time.perf_counter() - t0
        self.io["d2h"] += 4
        return m

    def _remeasure_safe(self, lo, key, entries, ctx, opts):
        """Recompile a PTX candidate with the other ptxas level and measure it again
        (None on failure)."""
        st, secs, hit, data = self.collect(self.submit(lo.source, opts))
        self.stats["compile_s"] += secs
        self.stats["recompiled"] = self.stats.get("recompiled", 0) + 1
        if st != 0:
            return None
        funcs = self.load(key + (":O1" if opts == PTX_SAFE_OPTS else ":O3"), data, entries)
        t0 = time.perf_counter()
        m = ctx.measure(lo, funcs, self.min_ms, self.max_repeat, self.min_repeat)
        if m.status == 2:
            self.faulted = True
            return None
        self.stats["gpu_s"] += time.perf_counter() - t0
        self.io["d2h"] += 4
        return m


# ---- the measuring process -------------------------------------------------
# A faulting candidate kills every CUDA context of its process on the device
# (measured: torch's primary context and a fresh cuCtxCreate context both fail
# after one illegal-address fault), so candidates run in a child process that
# owns the RunnerCore; the parent (torch, NCCL, the scoring/training kernels)
# never sees a device fault.  A fault ends the child's batch; the parent starts
# a fresh child and measures the rest of the batch there.

FAULT_PTX = b""".version 8.7
.target sm_100a
.address_size 64
.visible .entry lt_fault()
{
  .reg .b64 %rd<2>;
  .reg .b32 %r<2>;
  mov.u64 %rd1, 16;
  mov.u32 %r1, 7;
  st.global.u32 [%rd1], %r1;
  ret;
}
"""


def _delta(after: dict, before: dict) -> dict:
    return {k: v - before.get(k, 0) for k, v in after.items() if isinstance(v, (int, float))}


class _Server:
    """Commands the parent's `Runner` sends to the measuring process."""

    def __init__(self, kw: dict):
        self.core = RunnerCore(**kw)

    def measure(self, programs, seed, stage=None):
        c = self.core
        if len(c._dag_keys) > 256:         # every call unpickles fresh DAG objects
            c._dag_keys.clear()
        s0, io0 = dict(c.stats), dict(c.io)
        recs = c.measure_programs(programs, seed, stage)
        return recs, _delta(c.stats, s0), _delta(c.io, io0)

    def prepare(self, dag, seed):
        c = self.core
        io0 = dict(c.io)
        c.context(dag, seed)
        return _delta(c.io, io0)

    def refresh(self):
        c = self.core
        io0 = dict(c.io)
        for ctx in c.ctx.values():
            ctx.refresh()
        return _delta(c.io, io0)

    def drop_contexts(self):
        c = self.core
        for ctx in c.ctx.values():
            ctx.release()
        c.ctx.clear()
        c._dag_keys.clear()

    def download(self, dag, seed, name, numel, fp64):
        return self.core.context(dag, seed).download(name, numel, fp64)

    def forget_compiled(self, cache_dir):
        self.core.forget_compiled(cache_dir)

    def set_max_modules(self, n):
        self.core.max_modules = n

    def set_force_recompile(self, on):
        self.core.force_recompile = bool(on)

    def inject_fault(self):
        """Test hook: run a kernel that stores to an unmapped address."""
        c = self.core
        m = c.lib.lt_module_load(c.device, FAULT_PTX, len(FAULT_PTX))
        if not m:
            raise rt.NativeError(c.lib.lt_last_error().decode())
        fn = c.lib.lt_module_function(m, b"lt_fault")
        task = c.lib.lt_task_create(c.device)
        launches = (rt.Launch * 1)()
        launches[0].func = fn
        launches[0].grid[:] = (1, 1, 1)
        launches[0].block[:] = (32, 1, 1)
        launches[0].n_args = 0
        rec = rt.MeasureRecord()
        zi, zl = np.zeros(1, np.int32), np.zeros(1, np.int64)
        rt.check(c.lib.lt_measure(task, ctypes.addressof(launches), 1, rt.ptr(zi, rt.c_i32p), rt.ptr(zl, rt.c_i64p),
                                  0, 1, 5, 1.0, ctypes.addressof(rec)), "lt_measure")
        c.faulted = c.faulted or rec.status == 2
        return rec.status, rec.detail.decode(errors="replace")


def _serve(conn, kw: dict) -> None:
    """Measuring-process main loop: (command, args) in, (ok, result) out."""
    import traceback
    try:
        srv = _Server(kw)
    except BaseException as e:         # surfaced in the parent
        conn.send((False, f"{type(e).__name__}: {e}"))
        return
    conn.send((True, os.getpid()))
    while True:
        try:
            cmd, args = conn.recv()
        except (EOFError, OSError):
            break
        if cmd == "close":
            srv.core.close()
            conn.send((True, None))
            break
        try:
            res = getattr(srv, cmd)(*args)
            conn.send((True, (res, srv.core.faulted)))
        except BaseException:
            conn.send((False, traceback.format_exc()))
        if srv.core.faulted:
            srv.core.abandon()
            conn.close()
            os._exit(0)              # the CUDA state is gone: no teardown calls into it


class _ChildDied(RuntimeError):
    pass


class Runner:
    """The process-wide GPU runner as the rest of the package sees it: forwards
    to a `RunnerCore` in a child measuring process (spawned on first use,
    replaced after a kernel fault).  Cumulative `stats` / `io` and the last
    batch's records (`last_records`) are kept here."""

    def __init__(self, device: int = 0, **kw):
        self.device = device
        self._kw = dict(device=device, **kw)
        self.backend = kw.get("backend", "ptx")
        self.min_ms = kw.get("min_ms", 1.0)
        self.stats: dict = {"compiled": 0, "recompiled": 0, "cache_hits": 0, "compile_s": 0.0, "measured": 0,
                            "kernels_compiled": 0, "kernels_shared": 0, "lower_s": 0.0, "gpu_s": 0.0,
                            "load_s": 0.0, "idle_s": 0.0, "wall_s": 0.0, "restarts": 0}
        self.io = {"h2d": 0, "d2h": 0}
        self.last_records: list = []
        self._max_modules = None
        self._prepared: list = []          # (dag, seed) made resident; re-made after a restart
        self._proc = None
        self._conn = None
        self.pid = None
        self._start()

    # -- process management ----------------------------------------------------
    def _start(self) -> None:
        import multiprocessing as mp
        ctx = mp.get_context("spawn")
        parent, child = ctx.Pipe()
        proc = ctx.Process(target=_serve, args=(child, self._kw), name="lt-measure", daemon=False)
        proc.start()
        child.close()
        try:
            ok, payload = parent.recv()
        except EOFError:
            proc.join(5)
            raise rt.NativeError(f"measuring process exited at start (code {proc.exitcode})")
        if not ok:
            proc.join(5)
            raise rt.NativeError(f"measuring process failed to start: {payload}")
        self._proc, self._conn, self.pid = proc, parent, payload
        _LIVE.add(self)
        if self._max_modules is not None:
            self._call("set_max_modules", self._max_modules)
        for dag, seed in self._prepared:
            self._call("prepare", dag, seed)

    def _reap(self) -> None:
        if self._conn is not None:
            self._conn.close()
        if self._proc is not None:
            self._proc.join(10)
            if self._proc.is_alive():
                self._proc.kill()
                self._proc.join(5)
        self._proc = self._conn = None
        _LIVE.discard(self)

    def _call(self, cmd: str, *args):
        if self._proc is None:
            self._start()
            self.stats["restarts"] += 1
        try:
            self._conn.send((cmd, args))
            ok, payload = self._conn.recv()
        except (EOFError, OSError) as e:
            code = self._proc.exitcode if self._proc is not None else None
            self._reap()
            raise _ChildDied(f"measuring process died (exit code {code})") from e
        if not ok:
            raise rt.NativeError(f"measuring process: {payload}")
        res, faulted = payload
        if faulted:
            self._reap()                    # it exits by itself; the next call starts a fresh one
            self.stats["device_faults"] = self.stats.get("device_faults", 0) + 1
        return res

    def close(self) -> None:
        if self._proc is not None:
            try:
                self._conn.send(("close", ()))
                self._conn.recv()
            except (EOFError, OSError):
                pass
            self._reap()

    # -- API -------------------------------------------------------------------
    def measure_programs(self, programs: list, seed: int = 0, stage: list | None = None) -> list:
        """Records in input order.  Candidates a fault cut off are measured again
        in a fresh process; if the process dies outright (not a reported fault),
        the rest is measured one candidate per call so the culprit is isolated.
        `stage`: the next batch's programs, lowered and compiled in the measuring
        process behind this batch (RunnerCore.stage)."""
        programs = list(programs)
        recs: list = [None] * len(programs)
        todo = list(range(len(programs)))
        solo = False
        first = True
        while todo:
            chunk = todo[:1] if solo else todo
            try:
                got, dstats, dio = self._call("measure", [programs[i] for i in chunk], seed,
                                              list(stage) if (stage and first) else None)
                first = False
            except _ChildDied as e:
                if len(chunk) == 1:
                    recs[chunk[0]] = Record(detail=f"gpu: {e}", done=True)
                    todo = todo[1:]
                solo = True
                continue
            for k, v in dstats.items():
                self.stats[k] = self.stats.get(k, 0) + v
            for k, v in dio.items():
                self.io[k] = self.io.get(k, 0) + v
            for i, r in zip(chunk, got):
                if r.done:
                    recs[i] = r
            todo = [i for i in todo if recs[i] is None]
        self.last_records = recs
        return recs

    def prepare(self, dag, seed: int = 0) -> None:
        """Make a DAG's inputs and fp64 ground truth resident (kept across restarts)."""
        if not any(d is dag and s == seed for d, s in self._prepared):
            self._prepared.append((dag, seed))
        dio = self._call("prepare", dag, seed)
        for k, v in dio.items():
            self.io[k] += v

    def refresh(self) -> None:
        """Re-upload every resident DAG's inputs and recompute its ground truth."""
        for k, v in self._call("refresh").items():
            self.io[k] += v

    def drop_contexts(self) -> None:
        self._prepared.clear()
        self._call("drop_contexts")

    def download(self, dag, seed: int, name: str, numel: int, fp64: bool = False) -> np.ndarray:
        """A buffer of the last candidate measured on `dag` (fp64: its ground truth)."""
        return self._call("download", dag, seed, name, numel, fp64)

    def forget_compiled(self, cache_dir: str) -> None:
        self._kw["cache_dir"] = cache_dir
        self._call("forget_compiled", cache_dir)

    @property
    def max_modules(self):
        return self._max_modules

    @max_modules.setter
    def max_modules(self, n: int) -> None:
        self._max_modules = n
        self._call("set_max_modules", n)

    def inject_fault(self):
        return self._call("inject_fault")

    def force_recompile(self, on: bool) -> None:
        """Test hook: every PTX candidate's first verification counts as failed, so
        the recompile-at-the-other-ptxas-level path runs."""
        self._call("set_force_recompile", on)


_RUNNER: Runner | None = None
_LIVE: set = set()      # Runners that own a live measuring process (strong refs: a dropped Runner's
                        # process would otherwise outlive it and hang multiprocessing's exit join)


def _shutdown() -> None:
    """Close every runner's measuring process (also runners that were replaced
    by configure() and restarted their process on a later call)."""
    global _RUNNER
    for r in list(_LIVE):
        r.close()
    _RUNNER = None


atexit.register(_shutdown)


def get_runner(**kw) -> Runner:
    global _RUNNER
    if _RUNNER is None:
        _RUNNER = Runner(**kw)
    return _RUNNER


def configure(**kw) -> Runner:
    """(Re)create the process-wide runner (device, workers, cache_dir, min_ms...)."""
    global _RUNNER
    if _RUNNER is not None:
        _RUNNER.close()
    _RUNNER = Runner(**kw)
    return _RUNNER


def normalise(recs: list, best_cost=None, cost_ceiling=None) -> list:
    """Records -> MeasureResults with the reference's statuses and normalisation."""
    results, costs = [], []
    for r in recs:
        if r.status != VALID:
            results.append(MeasureResult(math.inf, 0.0, INVALID, r.detail))
            costs.append(None)
        elif cost_ceiling is not None and r.cost_us >= cost_ceiling:
            results.append(MeasureResult(r.cost_us, 0.0, TIMEOUT))
            costs.append(None)
        else:
            results.append(MeasureResult(r.cost_us, 0.0, VALID))
            costs.append(r.cost_us)
    valid = [c for c in costs if c is not None]
    if best_cost is not None:
        valid.append(best_cost)
    if not valid:
        return results
    best = min(valid)
    return [replace(r, throughput=best / c) if c is not None else r for r, c in zip(results, costs)]


def measure_batch(programs, spec=None, limits=None, best_cost=None) -> list:
    """Drop-in for `loomtune.machine.measure_batch` (`src/machine.py:249-285`)."""
    limits = limits if limits is not None else MeasureLimits()
    runner = get_runner()
    recs = runner.measure_programs(list(programs), seed=getattr(limits, "check_seed", 0))
    return normalise(recs, best_cost, getattr(limits, "cost_ceiling", None))
