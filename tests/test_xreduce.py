"""Cross-thread reductions: States from the reference's rule 6
(ReductionFactorization, `src/sketch.py:307-329`: fuse the reduction loops,
rfactor, then the annotation phase fuses `rf` with the space loops and marks it
parallel) lower to ONE kernel that binds rf to threadIdx.x and combines the
partials with warp shuffles (`ptxgen._xreduce`).  CPU tests pin which States
take that lowering; the GPU tests verify every one against the fp64 ground
truth (max relative error <= 1e-4, north star)."""

import pytest

from paper_2006_06762_b200.state import ComputeDAG, history_from_json, replay
from paper_2006_06762_b200.state import workloads as W
from paper_2006_06762_b200.state import Lin, Read, Reduce
from paper_2006_06762_b200.state import compute, placeholder


def rfactor_history(stage, red, factor, space, pragma=64, annotate=True):
    """The step sequence the reference sampler emits for a rule-6 sketch
    (see the norm2 draws in tools/: fuse reduce loops, rfactor, fuse rf with the
    space loops, parallel annotation, unroll pragma)."""
    h, fused = [], red[0]
    for nxt in red[1:]:
        h.append({"k": "fuse", "stage": stage, "outer": fused, "inner": nxt})
        fused = f"{fused}@{nxt}"
    h.append({"k": "rfactor", "stage": stage, "loop": fused, "factor": factor})
    if annotate:
        outer = "rf"
        for n in space:
            h.append({"k": "fuse", "stage": f"{stage}.rf", "outer": outer, "inner": n})
            outer = f"{outer}@{n}"
        h.append({"k": "annotate", "stage": f"{stage}.rf", "loop": outer, "ann": "parallel"})
    h.append({"k": "pragma", "stage": f"{stage}.rf", "unroll": pragma})
    h.append({"k": "simplify"})
    return history_from_json(h)


def rows_dag(rows=3000, cols=64, op="max"):
    """r[u] = op_j x[u, j]: many output points (grid-stride blocks)."""
    body = Read("x", (Lin.var("u"), Lin.var("j")))
    return ComputeDAG((placeholder("x", (rows, cols), iters=("x0", "x1")),
                       compute("r", (("u", rows),), Reduce(op, ("j",), body), reduce=(("j", cols),))))


CASES = [
    # (name, dag builder, stage, reduce loops, space loops, rfactor factors)
    ("norm2", lambda: W.build("norm2", n=768, m=1024), "r", ["i", "j"], ["u"],
     [1, 3, 32, 96, 512, 1024, 2048, 8192]),
    ("rowmax", lambda: rows_dag(3000, 64, "max"), "r", ["j"], ["u"], [1, 16, 64]),
    ("rowsum", lambda: rows_dag(40, 4096, "sum"), "r", ["j"], ["u"], [4, 128, 4096]),
]


def programs():
    out = []
    for name, mk, stage, red, space, factors in CASES:
        dag = mk()
        for f in factors:
            for annotate in (True, False):
                out.append((f"{name}/rf{f}/{'ann' if annotate else 'raw'}",
                            replay(dag, rfactor_history(stage, red, f, space, annotate=annotate))))
    return out


def test_rule6_states_lower_to_one_cross_thread_kernel():
    from paper_2006_06762_b200.ptxgen import lower_ptx
    for name, p in programs():
        lo = lower_ptx(p)
        ks = [k.info["template"] for k in lo.kernels]
        assert ks[0] == "xreduce", (name, ks)
        k = lo.kernels[0]
        assert k.block % 32 == 0 and k.block <= 1024, name
        assert "r.rf" not in lo.buffers, name            # the partial is never materialised
        assert k.smem == (4 * k.block // 32 if k.block > 32 else 0), name   # one slot per warp


def test_reordered_partial_keeps_the_naive_lowering():
    from paper_2006_06762_b200.ptxgen import lower_ptx
    dag = rows_dag(48, 64, "sum")
    h = list(rfactor_history("r", ["j"], 8, ["u"], annotate=False))
    from paper_2006_06762_b200.state import Reorder
    h.insert(-1, Reorder("r.rf", ("u", "rf", "rk")))
    lo = lower_ptx(replay(dag, tuple(h)))
    assert [k.info["template"] for k in lo.kernels] == ["naive", "naive"]


@pytest.mark.gpu
def test_cross_thread_reductions_verify_on_the_device():
    from paper_2006_06762_b200 import measure
    r = measure.configure(device=0, cache_dir="")
    try:
        cases = programs()
        recs = r.measure_programs([p for _, p in cases])
        for (name, _), rec in zip(cases, recs):
            assert rec.status == "valid", (name, rec.detail)
            assert rec.max_rel_err <= 1e-4, (name, rec.max_rel_err)
            assert rec.info["kernels"][0]["template"] == "xreduce", name
    finally:
        measure._shutdown()
