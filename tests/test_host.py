"""CPU-only checks: host data model, encoder, lowering/codegen, native library surface."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2006_06762_b200 import encode, lower
from paper_2006_06762_b200.state import build, history_to_json, naive_program, validate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_corpus_replays_and_validates(corpus):
    # every golden State replays through the reference's IR and round-trips its history JSON
    for p, e in zip(corpus.programs, corpus.entries):
        assert history_to_json(p.history) == e["history"]
        assert validate(p) == []


def test_host_data_model_is_the_reference():
    # the product imports the reference's own State types (no mirror of them)
    import loomtune.ir
    from paper_2006_06762_b200 import state
    assert state.Program is loomtune.ir.Program and state.validate is loomtune.ir.validate
    assert state.replay is loomtune.ir.replay and state.ComputeDAG.__module__ == "loomtune.graph"


def test_encoder_records(corpus):
    words, stmt_off, prog_off = encode.encode_batch(corpus.programs)
    assert stmt_off[-1] == len(words)
    assert prog_off[-1] == len(stmt_off) - 1 == len(corpus.rows)
    for i in range(len(corpus.programs)):
        assert prog_off[i + 1] - prog_off[i] == corpus.offsets[i + 1] - corpus.offsets[i]
    # header sanity: n_nest, own_start, n_views within kernel limits
    for s in range(len(stmt_off) - 1):
        r = words[stmt_off[s]:stmt_off[s + 1]]
        assert 0 <= r[1] <= r[0] <= 32 and r[2] <= 64 and r[3] <= 24 and 1 <= r[4] <= 12


def test_native_encoder_equals_python_encoder(corpus):
    """The native encoder (csrc/encode_ext.cpp, the default) writes exactly the
    records of encode.py's Python restatement: the golden corpus (incl. evolved,
    rfactor, cache and packed States), stream slices of every config, and the
    error raised for a decode over an unknown loop."""
    from paper_2006_06762_b200 import build as B
    B.build()
    import bench
    from paper_2006_06762_b200.state import replay
    sets = [list(corpus.programs)]
    for cfg in ("RC", "G10", "CL", "TBG"):
        dag, stream = bench.load_stream(cfg)
        sets.append([replay(dag, h) for h in stream[:200]])
    for progs in sets:
        a = encode.encode_batch(progs, native=False)
        b = encode.encode_batch(progs, native=True)
        for x, y in zip(a, b):
            assert x.dtype == y.dtype and np.array_equal(x, y)
    import dataclasses

    import loomtune.ir as IR
    p = corpus.programs[0]
    s0 = next(s for s in p.stages if s.index_map)
    bad = dataclasses.replace(s0, index_map=((s0.index_map[0][0], IR.DVar("nope")),) + tuple(s0.index_map[1:]))
    q = dataclasses.replace(p, stages=tuple(bad if s is s0 else s for s in p.stages))
    for native in (False, True):
        with pytest.raises(encode.EncodeError, match="unknown loop 'nope'"):
            encode.encode_batch([q], native=native)


def test_lowering_covers_corpus(corpus):
    ok = illegal = 0
    for p in corpus.programs:
        try:
            lo = lower.lower(p)
        except lower.LoweringError as e:
            assert re.search(r"threads|shared memory|accumulators|virtual threads|unrolled", str(e)), str(e)
            illegal += 1
            continue
        ok += 1
        assert lo.kernels and all(k.block <= 1024 and k.smem <= lower.MAX_SMEM for k in lo.kernels)
        assert set(lo.outputs) == set(p.dag.outputs)
    assert ok > 0.8 * len(corpus.programs), (ok, illegal)


def test_identical_kernels_for_cpu_only_differences():
    """Fusing the parallel band differently (a CPU decision) must not change the GPU kernel."""
    from paper_2006_06762_b200.state import Annotate, Fuse, Split, Reorder, apply_step, SetPragma
    dag = build("matmul", n=64, m=64, k=64)
    p = naive_program(dag)
    for st in (Split("C", "i", (2, 4, 2, 1)), Split("C", "j", (2, 4, 2, 2)), Split("C", "k", (4, 4)),
               Reorder("C", ("i.0", "j.0", "i.1", "j.1", "i.2", "j.2", "k.0", "k.1", "i.3", "j.3", "k.2",
                             "i.4", "j.4")), SetPragma("C", 512)):
        p = apply_step(p, st)
    a = apply_step(apply_step(p, Fuse("C", "i.0", "j.0")), Annotate("C", "i.0@j.0", "parallel"))
    b = apply_step(p, Annotate("C", "i.0", "parallel"))
    assert lower.lower(a).source == lower.lower(b).source
    info = lower.lower(a).kernels[0].info
    assert info["template"] == "tiled" and info["threads"] == 4 * 4 and info["blocks"] == 4 * 2 and info["vthreads"] == 2 * 2


def test_reference_lowering_is_fp64():
    lo = lower.reference_lowering(build("conv2d", h=6, w=6, ci=4, co=4))
    assert "double" in lo.source and "float*" not in lo.source
    assert [k.info["template"] for k in lo.kernels] == ["naive", "naive"]


def test_library_loads_and_exports_header_symbols():
    from paper_2006_06762_b200 import build as B
    from paper_2006_06762_b200 import runtime as rt
    B.build()
    lib = ctypes.CDLL(B.LIB)
    with open(os.path.join(ROOT, "include", "loomtune_b200.h")) as fh:
        hdr = fh.read()
    declared = set(re.findall(r"\b(lt_[a-z_0-9]+)\s*\(", hdr))
    assert declared, "no declarations found"
    for name in sorted(declared):
        getattr(lib, name)  # raises AttributeError if not exported
    assert set(rt.EXPORTS) <= declared
    assert os.access(B.WORKER, os.X_OK)


def test_nvrtc_pool_compiles_generated_kernel(tmp_path):
    """The compile service works without a GPU (NVRTC cross-compiles sm_100a)."""
    from paper_2006_06762_b200 import runtime as rt
    from paper_2006_06762_b200.measure import NVRTC_OPTS
    lib = rt.load(require_device=False)
    rt.check(lib.lt_pool_start(2, str(tmp_path).encode(), 120.0), "pool")
    try:
        src = lower.lower(naive_program(build("matmul", n=16, m=16, k=16))).source.encode()
        ids = [lib.lt_compile_submit(src, len(src), NVRTC_OPTS.encode()) for _ in range(2)]
        for j in ids:
            st, secs, hit, n = ctypes.c_int(), ctypes.c_double(), ctypes.c_int(), ctypes.c_int64()
            rt.check(lib.lt_compile_wait(j, ctypes.byref(st), ctypes.byref(secs), ctypes.byref(hit),
                                         ctypes.byref(n)), "wait")
            buf = ctypes.create_string_buffer(n.value)
            rt.check(lib.lt_compile_fetch(j, buf, n.value), "fetch")
            assert st.value == 0 and buf.raw[:4] == b"\x7fELF"
        # second submission of the same source is a cache hit
        j = lib.lt_compile_submit(src, len(src), NVRTC_OPTS.encode())
        st, secs, hit, n = ctypes.c_int(), ctypes.c_double(), ctypes.c_int(), ctypes.c_int64()
        lib.lt_compile_wait(j, ctypes.byref(st), ctypes.byref(secs), ctypes.byref(hit), ctypes.byref(n))
        lib.lt_compile_fetch(j, None, 0)
        assert hit.value == 1
    finally:
        lib.lt_pool_stop()


def test_pack_matches_reference_semantics():
    from paper_2006_06762_b200.measure import pack
    rng = np.random.default_rng(0)
    B = rng.random((8, 12))
    desc = ((1, 3), (0, 2), (1, 4), (0, 4))
    P = pack(B, desc)
    for a in range(3):
        for b in range(2):
            for c in range(4):
                for d in range(4):
                    assert P[a, b, c, d] == B[b * 4 + d, a * 4 + c]


def test_device_pack_parameters_reproduce_pack():
    """`lt_task_pack`'s index map (physical digits x `pack_strides` multipliers into the
    flat logical offset), emulated in numpy, equals the host restatement `pack` on
    every packed layout of the golden streams; a descriptor that does not tile its
    dims is refused."""
    import bench
    from paper_2006_06762_b200.measure import pack, pack_strides, random_inputs
    from paper_2006_06762_b200.ptxgen import lower_ptx
    from paper_2006_06762_b200.state import replay
    seen = set()
    for cfg in ("G10", "RC", "TBG", "CL"):
        dag, stream = bench.load_stream(cfg)
        inputs = random_inputs(dag, 0)
        for h in stream[:48]:
            p = replay(dag, h)
            if validate(p):
                continue
            try:
                lo = lower_ptx(p)
            except Exception:
                continue
            for b in lo.buffers.values():
                if b.role != "packed" or (b.source, b.desc) in seen:
                    continue
                seen.add((b.source, b.desc))
                a = inputs[b.source].astype(np.float32)
                ext, mult = pack_strides(a.shape, b.desc)
                r = np.arange(int(np.prod(ext)))
                off = np.zeros_like(r)
                for j in range(len(ext) - 1, -1, -1):
                    off += (r % ext[j]) * mult[j]
                    r //= ext[j]
                assert np.array_equal(a.reshape(-1)[off], np.ascontiguousarray(pack(a, b.desc)).reshape(-1))
    assert len(seen) >= 20
    with pytest.raises(ValueError, match="does not tile"):
        pack_strides((8, 12), ((1, 3), (0, 2), (1, 4), (0, 3)))


def test_ptx_backend_legality_and_assembly(corpus, tmp_path):
    """PTX and CUDA-C lowerings agree on legality; generated PTX assembles (ptxas, no GPU)."""
    import subprocess
    from paper_2006_06762_b200 import ptxgen
    for i, p in enumerate(corpus.programs):
        a = b = None
        try:
            lower.lower(p)
        except lower.LoweringError as e:
            a = str(e)
        try:
            lo = ptxgen.lower_ptx(p)
        except lower.LoweringError as e:
            b = str(e)
        assert a == b, i
        if b is None and i % 25 == 0:
            path = tmp_path / "k.ptx"
            path.write_text(lo.source)
            r = subprocess.run(["/usr/local/cuda/bin/ptxas", "-arch=sm_100a", str(path), "-o",
                                str(tmp_path / "k.cubin")], capture_output=True, text=True)
            assert r.returncode == 0, r.stderr[:500]


def test_magic_division():
    from paper_2006_06762_b200.ptxgen import _magic
    import random
    rnd = random.Random(0)
    for d in list(range(3, 3000)) + [rnd.randrange(3, 1 << 20) for _ in range(300)]:
        if d & (d - 1) == 0:
            continue
        m, s = _magic(d)
        for x in list(range(2048)) + [rnd.randrange(0, 1 << 31) for _ in range(50)]:
            assert ((x * m) >> 32) >> s == x // d
