"""install(): the reference's unchanged tuner runs on the B200 path."""

import numpy as np
import pytest

from paper_2006_06762_b200.reference import loomtune as LT     # baseline/_ref travels with the repo


class CpuBatchModel:
    """Reference CostModel with a CPU predict_batch (same arithmetic)."""

    def __init__(self, m):
        self.m = m

    def predict(self, p):
        return self.m.predict(p)

    def predict_batch(self, ps):
        return np.asarray([self.m.predict(p) for p in ps])


def test_batched_evolve_matches_reference_evolve():
    import importlib
    ev = importlib.import_module("loomtune.evolve")
    from loomtune.model import TrainHyper, TrainingRecord, train
    from loomtune.sketch import generate_sketches
    from paper_2006_06762_b200.integrate import make_evolve_batched
    dag = LT.build("matmul", n=32, m=32, k=32)
    rng = np.random.default_rng(0)
    sk = generate_sketches(dag, structure="SSSRRSRS")
    init = [LT.sample_program(sk[i % len(sk)], LT.AnnotationPolicy(), rng) for i in range(24)]
    from loomtune.features import extract_features
    recs = [TrainingRecord("t", p.history, float(rng.random()) + 0.1, feats=extract_features(p)) for p in init]
    model = train(recs, TrainHyper(trees=5))
    cfg = LT.EvolutionConfig(population=24, generations=2, k=8, seed=3)
    want = ev.evolve(init, model, cfg)
    got = make_evolve_batched(ev)(init, CpuBatchModel(model), cfg)
    assert [c.fitness for c in got] == [c.fitness for c in want]
    assert [ev._state_key(c.program) for c in got] == [ev._state_key(c.program) for c in want]


def test_gpu_sketch_policy_keeps_gpu_rule_sketches():
    from paper_2006_06762_b200.integrate import gpu_sketch_policy
    t = LT.make_task("mm", LT.build("matmul", n=64, m=64, k=64), structure="SSSRRSRS")
    before = list(t.sketches)
    paths = gpu_sketch_policy(LT, t)
    assert paths and all({3, 4, 6} & set(p) for p in paths)
    assert 0 < len(t.sketches) < len(before)
    assert all(any(s is b for b in before) for s in t.sketches)        # a subset, order kept
    n2 = LT.make_task("n2", LT.build("norm2", n=32, m=64), structure="SSSRRSRS")
    assert [6 in p for p in gpu_sketch_policy(LT, n2)] == [True]        # rfactor -> cross-thread
    ew = LT.make_task("ew", LT.build("elemwise_chain", n=256), structure="SSSRRSRS")
    k = len(ew.sketches)
    gpu_sketch_policy(LT, ew)
    assert len(ew.sketches) == k                                        # no GPU rule applies: unchanged


def test_gpu_sampler_draws_legal_gpu_sane_states():
    from loomtune.ir import validate
    from paper_2006_06762_b200.integrate import gpu_sane, make_gpu_sampler
    t = LT.make_task("mm", LT.build("matmul", n=256, m=256, k=128), structure="SSSRRSRS")
    sample = make_gpu_sampler(LT.sample_program)
    rng = np.random.default_rng(0)
    for i in range(24):
        p = sample(t.sketches[i % len(t.sketches)], LT.AnnotationPolicy(), rng)
        assert p.is_concrete() and not validate(p)
        assert gpu_sane(p)


def test_install_rebinds_and_restores():
    from paper_2006_06762_b200 import integrate, measure
    import importlib
    sched, cli = importlib.import_module("loomtune.sched"), importlib.import_module("loomtune.cli")
    from paper_2006_06762_b200 import replay
    logio = importlib.import_module("loomtune.logio")
    orig = integrate.install(LT)
    try:
        assert sched.measure_batch is measure.measure_batch
        assert cli.measure_batch is measure.measure_batch
        assert cli.cmd_replay is replay.cmd_replay
        assert logio.LogWriter.write is not orig["logio.LogWriter.write"]
    finally:
        integrate.uninstall(LT, orig)
    assert sched.measure_batch is orig["measure_batch"]
    assert cli.cmd_replay is orig["cli.cmd_replay"]
    assert logio.LogWriter.write is orig["logio.LogWriter.write"]


@pytest.mark.gpu
def test_tune_runs_on_gpu_path():
    """A short reference `tune` with every hot-path call on the B200."""
    from paper_2006_06762_b200 import integrate, measure
    from paper_2006_06762_b200.model import GpuCostModel
    measure.configure(device=0, cache_dir="")
    orig = integrate.install(LT)
    try:
        dag = LT.build("matmul", n=256, m=256, k=256)
        task = LT.make_task("mm", dag, structure="SSSRRSRS")
        res = LT.tune([task], LT.Objective(), 3, LT.TuneSettings(), LT.SchedulerParams(), seed=0)
        assert task.best_program is not None and np.isfinite(task.best_cost)
        assert isinstance(res.model, GpuCostModel)
    finally:
        integrate.uninstall(LT, orig)
        measure._shutdown()
