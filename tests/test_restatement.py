"""CPU: the independent fp64 restatement the GPU parity tests use at full
shapes (torch CPU conv / matmul / pooling, tests/test_parity_layers_gpu.py)
is pinned to the reference's own state-free `reference_outputs`
(`src/interp.py:46-74`, imported unchanged) at reduced shapes, for every DAG
kind it covers — including the two pooling subgraphs added for the
whole-network task list."""

import numpy as np
import pytest

from tests.test_parity_layers_gpu import TOL_GT, _rel, _torch_fp64

CASES = [
    ("matmul", dict(n=24, m=20, k=16)),
    ("batch_matmul", dict(b=3, n=8, m=12, k=5)),
    ("conv2d", dict(h=9, w=9, ci=4, co=6, kernel=3, stride=1, pad=1, n=2)),
    ("conv2d", dict(h=11, w=11, ci=3, co=4, kernel=7, stride=2, pad=3, n=1)),
    ("conv2d", dict(h=8, w=8, ci=6, co=5, kernel=1, stride=2, pad=0, n=2)),
    ("conv_bn_relu", dict(n=2, h=6, w=6, ci=4, co=5, kernel=3, stride=1, pad=1)),
    ("max_pool", dict(n=2, h=10, c=3, kernel=3, stride=2, pad=1)),
    ("global_avg_pool", dict(n=3, h=4, c=5)),
]


@pytest.mark.parametrize("kind,kw", CASES, ids=[f"{k}-{i}" for i, (k, _) in enumerate(CASES)])
def test_torch_restatement_equals_reference_outputs(kind, kw):
    from loomtune.interp import random_inputs, reference_outputs
    from paper_2006_06762_b200 import resnet50
    from paper_2006_06762_b200.measure import random_inputs as our_inputs
    from paper_2006_06762_b200.state import build
    if kind == "max_pool":
        dag = resnet50.max_pool(**kw)
    elif kind == "global_avg_pool":
        dag = resnet50.global_avg_pool(**kw)
    else:
        dag = build(kind, **kw)
    ref_in = random_inputs(dag, np.random.default_rng(0))
    ours = our_inputs(dag, 0)
    for k in ref_in:
        assert np.array_equal(ref_in[k], ours[k])
    want = reference_outputs(dag, ref_in)
    got = _torch_fp64(kind, kw, ours)
    for out in dag.outputs:
        assert _rel(got[out], want[out]) <= TOL_GT, (kind, out)


def test_resnet50_task_list():
    """23 distinct convs + the classifier + max-pool + global average pool; every
    task has SSSRRSRS sketches under the reference's own generator."""
    from loomtune.sketch import generate_sketches
    from paper_2006_06762_b200 import resnet50
    tasks = resnet50.tasks()
    assert len(tasks) == 26
    assert sum(w for _, _, w in tasks) == 56
    for name, dag, _ in tasks:
        assert generate_sketches(dag, structure="SSSRRSRS"), name


def test_resnet50_fused_task_list():
    """The conv+BN+ReLU fusion variant of the task list: same shapes and weights,
    every task a ConvLayer-style DAG with SSSRRSRS sketches."""
    from loomtune.sketch import generate_sketches
    from paper_2006_06762_b200 import resnet50
    plain = resnet50.tasks()
    fused = resnet50.tasks(fusion="conv_bn_relu")
    assert [w for _, _, w in plain] == [w for _, _, w in fused]
    for (n1, d1, _), (n2, d2, _) in zip(plain, fused):
        if n1.startswith("conv"):
            assert n2 == n1 + "_bn_relu" and d2.outputs == ("E",)
            assert d2.node("C").space == d1.node("C").space
            assert generate_sketches(d2, structure="SSSRRSRS"), n2
