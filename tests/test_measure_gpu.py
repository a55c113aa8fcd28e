"""GPU runner parity: every candidate the runner accepts computes the reference's outputs."""

import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def runner():
    from paper_2006_06762_b200 import measure
    r = measure.configure(device=0, cache_dir="")
    yield r


def test_small_corpus_all_outputs_correct(corpus, runner):
    from paper_2006_06762_b200.measure import VALID
    small = [i for i, e in enumerate(corpus.entries) if ":" in e["dag"] and not e["dag"].startswith("tune")]
    progs = [corpus.programs[i] for i in small]
    recs = runner.measure_programs(progs)
    n_valid = sum(r.status == VALID for r in recs)
    wrong = [(small[k], r.detail) for k, r in enumerate(recs) if "differs from reference" in r.detail]
    faults = [(small[k], r.detail) for k, r in enumerate(recs) if "compile failed" in r.detail]
    assert not wrong, wrong[:5]
    assert not faults, faults[:3]
    assert n_valid >= 0.8 * len(progs), (n_valid, len(progs))
    for r in recs:
        if r.status == VALID:
            assert r.max_rel_err <= 1e-4 and math.isfinite(r.cost_us) and r.cost_us > 0
    print(f"small corpus: {n_valid}/{len(progs)} VALID")


def test_evolved_states_correct(corpus, runner):
    idx = [i for i, e in enumerate(corpus.entries) if e["dag"].startswith("tune")]
    recs = runner.measure_programs([corpus.programs[i] for i in idx])
    wrong = [(idx[k], r.detail) for k, r in enumerate(recs) if "differs" in r.detail or "compile failed" in r.detail]
    assert not wrong, wrong[:5]


def test_ground_truth_matches_reference_outputs(runner):
    """The device fp64 ground truth equals the reference's `reference_outputs` (golden)."""
    from paper_2006_06762_b200.state import build
    outs = np.load(os.path.join(GOLDEN, "outputs.npz"))
    shapes = {"matmul": dict(n=64, m=64, k=64), "conv2d": dict(h=6, w=6, ci=8, co=8, n=2),
              "batch_matmul": dict(b=4, n=16, m=16, k=8), "conv_bn_relu": dict(n=2, h=6, w=6, ci=8, co=8),
              "norm2": dict(n=8, m=32), "grouped_conv2d": dict(h=6, w=6, ci=8, co=8)}
    for name, kw in shapes.items():
        dag = build(name, **kw)
        runner.prepare(dag, 0)
        for o in dag.outputs:
            want = outs[f"{name}/{o}"]
            got = runner.download(dag, 0, o, want.size, fp64=True).reshape(want.shape)
            np.testing.assert_allclose(got, want, rtol=1e-12, atol=0)


def test_candidate_outputs_match_reference_outputs(corpus, runner):
    """Download a candidate's fp32 output and compare with the golden reference outputs."""
    from paper_2006_06762_b200.measure import VALID
    outs = np.load(os.path.join(GOLDEN, "outputs.npz"))
    checked = 0
    for i, e in enumerate(corpus.entries):
        name = e["dag"].split(":")[0]
        if name not in ("matmul", "conv2d", "batch_matmul", "conv_bn_relu") or e["dag"].startswith("tune"):
            continue
        p = corpus.programs[i]
        (rec,) = runner.measure_programs([p])
        if rec.status != VALID:
            continue
        for o in p.dag.outputs:
            want = outs[f"{name}/{o}"]
            got = runner.download(p.dag, 0, o, want.size).reshape(want.shape).astype(np.float64)
            rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
            assert float(rel.max()) <= 1e-4, (i, float(rel.max()))
        checked += 1
    assert checked >= 20


def test_status_semantics_match_reference(runner):
    """validate() failures carry the reference's detail; normalisation is the reference's."""
    from paper_2006_06762_b200.measure import INVALID, VALID, measure_batch
    from paper_2006_06762_b200.state import ComputeDAG, history_from_json, replay
    with open(os.path.join(GOLDEN, "corpus.json")) as fh:
        dags = json.load(fh)["dags"]
    with open(os.path.join(GOLDEN, "measure.json")) as fh:
        cases = json.load(fh)
    for case in cases:
        dag = ComputeDAG.from_json(dags[case["dag"]])
        progs = [replay(dag, history_from_json(h)) for h in case["histories"]]
        res = measure_batch(progs)
        for r, bad in zip(res, case["validate"]):
            if bad:
                assert r.status == INVALID and r.detail == bad[0] and r.cost == math.inf and r.throughput == 0.0
        valid = [r for r in res if r.status == VALID]
        best = min(r.cost for r in valid)
        for r in valid:
            assert r.throughput == best / r.cost
        anchored = measure_batch(progs[:1], best_cost=best / 2)
        if anchored[0].status == VALID:
            assert anchored[0].throughput == (best / 2) / anchored[0].cost


def test_timeout_ceiling(runner):
    from paper_2006_06762_b200.measure import TIMEOUT, MeasureLimits, measure_batch
    from paper_2006_06762_b200.state import build, naive_program
    (r,) = measure_batch([naive_program(build("matmul", n=64, m=64, k=64))], limits=MeasureLimits(cost_ceiling=1e-3))
    assert r.status == TIMEOUT and math.isfinite(r.cost) and r.throughput == 0.0


def test_baseline_configs_measure(corpus, runner):
    """BASELINE-shape States (G5, G10, RC, TBG, CL): every accepted candidate is correct."""
    from paper_2006_06762_b200.measure import VALID
    idx = [i for i, e in enumerate(corpus.entries) if e["dag"] in ("G5", "G10", "RC", "TBG", "CL")]
    recs = runner.measure_programs([corpus.programs[i] for i in idx])
    wrong = [(idx[k], r.detail) for k, r in enumerate(recs) if "differs" in r.detail or "compile failed" in r.detail]
    assert not wrong, wrong[:5]
    print("baseline configs:", sum(r.status == VALID for r in recs), "/", len(recs), "VALID")
    for k, r in enumerate(recs):
        if r.status == VALID:
            print("  ", corpus.entries[idx[k]]["dag"], f"{r.cost_us:.1f} us", r.info["kernels"][0].get("template"))


def test_kernel_fault_is_contained_in_the_measuring_process():
    """A faulting candidate (illegal address) kills every CUDA context of its
    process on the device, so candidates run in a child measuring process: the
    fault comes back as a status, the parent's torch tensors and cost-model
    state stay valid, and measurement carries on in a fresh child."""
    import numpy as np
    import torch
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200.model import GpuCostModel
    from paper_2006_06762_b200.state import build, naive_program
    r = measure.configure(device=0, cache_dir="")
    try:
        dag = build("matmul", n=64, m=64, k=64)
        p = naive_program(dag)
        (a,) = r.measure_programs([p])
        assert a.status == "valid"
        x = torch.arange(1 << 20, dtype=torch.float32, device="cuda")
        m = GpuCostModel(base=1.0)
        s0 = m.predict_batch([p])
        pid0 = r.pid
        status, detail = r.inject_fault()
        assert status == 2 and "kernel fault" in detail, detail
        assert r.stats["device_faults"] == 1
        torch.cuda.synchronize()                                  # the parent's CUDA state is healthy
        assert float(x[-1]) == float((1 << 20) - 1)
        assert np.array_equal(m.predict_batch([p]), s0)
        (b,) = r.measure_programs([p])                           # a fresh measuring process
        assert b.status == "valid" and r.pid != pid0 and r.stats["restarts"] == 1
    finally:
        measure._shutdown()


def test_naive_multi_point_steps_verify():
    """The naive template's LT_NAIVE_POINTS option (several output points per
    grid-stride step, guarded loads and stores for the tail) verifies on naive
    stream candidates, reductions and fused padding included."""
    from bench import load_stream
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200.state import replay
    old = os.environ.get("LT_NAIVE_POINTS")
    os.environ["LT_NAIVE_POINTS"] = "4"             # read by ptxgen in the measuring process
    r = measure.configure(device=0, cache_dir="", lower_workers=1)   # lower in that process
    try:
        for cfg in ("RC", "G10", "CL"):
            dag, stream = load_stream(cfg)
            progs = [replay(dag, h) for h in stream[:12]]
            recs = r.measure_programs(progs)
            naive = [x for x in recs if any(k.get("points_per_thread_step") == 4 for k in x.info.get("kernels", []))]
            assert naive, cfg
            assert all(x.status == "valid" for x in recs), [(x.status, x.detail) for x in recs]
    finally:
        if old is None:
            os.environ.pop("LT_NAIVE_POINTS")
        else:
            os.environ["LT_NAIVE_POINTS"] = old
        measure._shutdown()


def test_module_eviction_keeps_shared_memory_grants_valid():
    """Candidate modules are evicted LRU; a function handle value reused by a
    later module must get its own >48 KB dynamic shared-memory grant (stale
    grants made such launches fail with 'invalid argument')."""
    from bench import load_stream
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200.state import replay
    dag, stream = load_stream("TBG")
    runner = measure.configure(device=0, cache_dir="")
    runner.max_modules = 4
    try:
        recs = runner.measure_programs([replay(dag, h) for h in stream[:48]])
    finally:
        measure._shutdown()
    big = [r for r in recs if any((k.get("smem") or 0) > 48 * 1024 for k in r.info.get("kernels", []))]
    assert big
    for i, r in enumerate(recs):
        assert r.status == "valid", (i, r.detail)


def test_recompile_path_after_failed_verification(runner):
    """A candidate whose first verification fails is recompiled at the other ptxas
    level and measured again (measure.RunnerCore._remeasure_safe); the test hook
    makes every first verification fail, so the path runs for every candidate."""
    import bench
    from paper_2006_06762_b200.state import replay
    dag, stream = bench.load_stream("G5")
    progs = [replay(dag, h) for h in stream[3:11]]
    before = runner.stats.get("recompiled", 0)
    runner.force_recompile(True)
    try:
        recs = runner.measure_programs(progs)
    finally:
        runner.force_recompile(False)
    assert runner.stats.get("recompiled", 0) > before
    for r in recs:
        if r.key:                                   # lowered to a PTX candidate
            assert r.status == "valid", r.detail
            assert "ptxas" in r.info and r.max_rel_err <= 1e-4


def test_batch_edge_cases(runner):
    """Empty batch; a State repeated in one batch (its kernels compile once);
    States of two different DAGs and an invalid State mixed in one batch —
    results in input order, statuses per State (src/machine.py:249-285)."""
    import bench
    from paper_2006_06762_b200.measure import INVALID, VALID, measure_batch
    from paper_2006_06762_b200.state import ComputeDAG, history_from_json, replay
    assert measure_batch([]) == []
    dag5, s5 = bench.load_stream("G5")
    dagt, st = bench.load_stream("TBG")
    p = replay(dag5, s5[7])
    q = replay(dagt, st[20])
    with open(os.path.join(GOLDEN, "measure.json")) as fh:
        case = json.load(fh)[0]                        # golden case 0, State 6: two parallel loops
    with open(os.path.join(GOLDEN, "corpus.json")) as fh:
        gdag = ComputeDAG.from_json(json.load(fh)["dags"][case["dag"]])
    bad = replay(gdag, history_from_json(case["histories"][6]))
    assert case["validate"][6]
    res = measure_batch([p, q, p, bad, q])
    assert [r.status for r in res] == [VALID, VALID, VALID, INVALID, VALID], res
    assert res[3].cost == math.inf and res[3].throughput == 0.0 and res[3].detail == case["validate"][6][0]
    best = min(r.cost for r in res if r.status == VALID)
    assert max(r.throughput for r in res) == 1.0 and all(
        r.throughput == best / r.cost for r in res if r.status == VALID)


def test_staged_next_batch(runner):
    """A batch measured with the next batch staged: the next batch's programs are
    lowered and compiled behind it, then measured from the staged work with the
    same verdicts as a from-scratch measurement."""
    import bench
    from paper_2006_06762_b200.state import replay
    dag, stream = bench.load_stream("G10")
    a = [replay(dag, h) for h in stream[100:116]]
    b = [replay(dag, h) for h in stream[116:132]]
    runner.measure_programs(a, stage=b)
    s0 = runner.stats.get("staged", 0)
    got = runner.measure_programs(b)
    assert runner.stats.get("staged", 0) - s0 == len(b)
    runner.forget_compiled("")
    want = runner.measure_programs(b)
    assert [r.status for r in got] == [r.status for r in want]
    assert [r.key for r in got] == [r.key for r in want]
    assert all(r.max_rel_err <= 1e-4 for r in got if r.status == "valid")


def test_device_packing_equals_host_pack():
    """Packed constants (LayoutRewrite) are laid out on the device by `lt_task_pack`
    from the resident fp32 input; every physical copy equals the host restatement
    `measure.pack` bit for bit, and the candidates that read them verify."""
    import ctypes
    from bench import load_stream
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200.state import replay
    seen = 0
    for cfg in ("G10", "RC"):
        dag, stream = load_stream(cfg)
        core = measure.RunnerCore(device=0, cache_dir="")
        try:
            recs = core.measure_programs([replay(dag, h) for h in stream[:24]])
            assert all(r.status == "valid" for r in recs), [r.detail for r in recs if r.status != "valid"]
            ctx = core.context(dag, 0)
            for h in stream[24:40]:
                lo = core.lower(replay(dag, h))
                for b in lo.buffers.values():
                    if b.role != "packed":
                        continue
                    sid = ctx.buffer_slot(b, False)
                    want = np.ascontiguousarray(measure.pack(ctx.inputs[b.source], b.desc), dtype=np.float32).ravel()
                    got = np.empty_like(want)
                    assert core.lib.lt_task_download(ctx.task, sid, got.ctypes.data_as(ctypes.c_void_p),
                                                     got.nbytes) == 0
                    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), b.desc
                    seen += 1
        finally:
            core.close()
    assert seen >= 10


def test_states_both_ptx_builds_get_wrong_are_measured_through_nvrtc():
    """Register-overflowing tiles whose PTX is assembled wrongly at both ptxas levels
    (tests/golden/ptx_rejected_states.json, found by tools/invalid_probe.py) are legal
    States: the runner re-lowers them to CUDA C, compiles with NVRTC, verifies again
    and reports them VALID, as the reference does."""
    from paper_2006_06762_b200 import measure, resnet50
    from paper_2006_06762_b200.state import history_from_json, replay
    data = json.load(open(os.path.join(GOLDEN, "ptx_rejected_states.json")))
    dags = {n: d for n, d, _ in resnet50.tasks()}
    core = measure.RunnerCore(device=0, cache_dir="")
    try:
        progs = [replay(dags[s["task"]], history_from_json(s["history"])) for s in data["states"]]
        recs = [core.measure_programs([p])[0] for p in progs]
    finally:
        core.close()
    for s, r in zip(data["states"], recs):
        assert r.status == "valid", (s["task"], s["i"], r.detail)
        assert r.max_rel_err <= 1e-4
        assert r.cost_us > 0 and math.isfinite(r.cost_us)
