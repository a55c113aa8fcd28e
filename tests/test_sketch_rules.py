"""The paper's two GPU sketch rules (`paper_2006_06762_b200/sketch_rules.py`,
PAPER.md:687) through the reference's own rule engine
(`generate_sketches(extra_rules=...)`, `src/sketch.py:345-388`)."""

import numpy as np
import pytest

from paper_2006_06762_b200.sketch_rules import gpu_sketches, gpu_sketches_traced
from paper_2006_06762_b200.state import config_dag
from tests.test_xreduce import rows_dag


def test_reference_sketches_are_kept():
    """Extra rules only add branches: every reference sketch is still derived."""
    from loomtune.sketch import generate_sketches
    for cfg in ("RC", "CL", "G10", "TBG"):
        dag = config_dag(cfg)
        ref = generate_sketches(dag, structure="SSSRRSRS")
        ours = gpu_sketches(dag)
        keys = {repr([(s.name, s.compute_at, tuple(l.id for l in s.loops)) for s in p.stages]) for p in ours}
        for p in ref:
            assert repr([(s.name, s.compute_at, tuple(l.id for l in s.loops)) for s in p.stages]) in keys


def test_shared_memory_rule_attaches_the_padding_producer_at_r0():
    """Conv: the padding stage becomes the shared-memory caching node of every
    tiled consumer (attached at its innermost R0 loop); GEMM/TBG have no
    computed operand, so the rule adds nothing there."""
    for cfg, host in (("RC", ("C", "C.cache")), ("CL", ("C",))):
        traced = gpu_sketches_traced(config_dag(cfg))
        smem = [(p, path) for p, path in traced if "gpu_smem" in path]
        assert len(smem) >= 2, cfg
        for p, _ in smem:
            at = p.stage("P").compute_at
            assert at is not None and at[0] in host and at[1] == "rc.0", (cfg, at)
    for cfg in ("G10", "TBG"):
        assert not any("gpu_smem" in path for _, path in gpu_sketches_traced(config_dag(cfg)))


def test_shared_memory_rule_samples_lower_to_one_fused_kernel():
    """Sampled States of the rule's sketches lower with the padding computed
    inside the tiled kernel's shared-memory fetch (no separate pad kernel)."""
    from loomtune.annotate import AnnotationPolicy, sample_program
    from paper_2006_06762_b200.integrate import make_gpu_sampler
    from paper_2006_06762_b200.ptxgen import lower_ptx
    sample = make_gpu_sampler(sample_program)
    rng = np.random.default_rng(0)
    sk = [p for p, path in gpu_sketches_traced(config_dag("RC")) if "gpu_smem" in path]
    fused = 0
    for i in range(12):
        q = sample(sk[i % len(sk)], AnnotationPolicy(), rng)
        lo = lower_ptx(q)
        if q.stage("P").compute_at is not None:
            assert not any(k.info.get("stage") == "P" for k in lo.kernels)
            assert any(k.info.get("template") == "tiled" for k in lo.kernels)
            fused += 1
    assert fused >= 8


def test_cross_thread_reduction_rule_fires_where_the_cpu_rule_does_not():
    """Space 512 (>= small_space 256, so the CPU rule 6 stays off) with a 4096-long
    reduction: the GPU rule factors it; the pair lowers to one xreduce kernel."""
    from loomtune.sketch import generate_sketches_traced
    from paper_2006_06762_b200.ptxgen import lower_ptx
    dag = rows_dag(512, 4096, "sum")
    assert not any(6 in path for _, path in generate_sketches_traced(dag, structure="SSSRRSRS"))
    ctr = [(p, path) for p, path in gpu_sketches_traced(dag) if "gpu_ctr" in path]
    assert ctr
    from tests.test_xreduce import rfactor_history
    from paper_2006_06762_b200.state import replay
    q = replay(dag, rfactor_history("r", ["j"], 128, ["u"]))
    assert any(k.info.get("template") == "xreduce" for k in lower_ptx(q).kernels)
    p, _ = ctr[0]
    assert p.has_stage("r.rf")


def test_policy_with_gpu_rules_keeps_only_gpu_sketches():
    import loomtune as LT
    from paper_2006_06762_b200.integrate import GPU_SKETCH_RULES, gpu_sketch_policy
    dag = LT.ComputeDAG.from_json(config_dag("RC").to_json())
    task = LT.make_task("RC", dag, structure="SSSRRSRS")
    paths = gpu_sketch_policy(LT, task, gpu_rules=True)
    assert len(paths) == len(task.sketches)
    assert all(any(r in GPU_SKETCH_RULES for r in path) for path in paths)
    assert sum("gpu_smem" in path for path in paths) == 3


@pytest.mark.gpu
def test_shared_memory_rule_states_measure_correct_on_gpu():
    """States from the shared-memory rule's sketches run on the B200 with the
    padding fused into the fetch; every output verified against fp64 (<= 1e-4)."""
    from loomtune.annotate import AnnotationPolicy, sample_program
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200.integrate import make_gpu_sampler
    sample = make_gpu_sampler(sample_program)
    rng = np.random.default_rng(1)
    for cfg in ("RC", "CL"):
        sk = [p for p, path in gpu_sketches_traced(config_dag(cfg)) if "gpu_smem" in path]
        progs = [sample(sk[i % len(sk)], AnnotationPolicy(), rng) for i in range(8)]
        recs = measure.get_runner().measure_programs(progs)
        assert all(r.status == "valid" and r.max_rel_err <= 1e-4 for r in recs), [r.detail for r in recs]
