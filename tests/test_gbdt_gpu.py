"""GPU GBDT training (csrc/gbdt.cu via paper_2006_06762_b200.gbdt) vs the
reference's own `train` on the golden cases (bit-exact model JSON and losses),
and vs the oracle's `fit_tree` on tie-heavy random matrices."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class _Rec:
    def __init__(self, feats, y):
        self.feats, self.y, self.dag_id = feats, float(y), "d"


def test_gpu_train_reproduces_reference_models():
    from paper_2006_06762_b200 import gbdt
    from paper_2006_06762_b200.model import Hyper
    from tests.test_oracle import _train_cases
    for name, mats, y, hyper, want, losses in _train_cases():
        m = gbdt.train([_Rec(f, v) for f, v in zip(mats, y)], Hyper(**hyper))
        assert m.to_json() == want, name
        if losses is not None:
            assert m.train_losses == losses, name


@pytest.mark.parametrize("n,levels,depth,seed", [(7, 2, 3, 0), (300, 3, 6, 1), (2000, 5, 6, 2), (5000, 50, 7, 3)])
def test_gpu_fit_tree_matches_oracle(n, levels, depth, seed):
    from oracle import train as OT
    from paper_2006_06762_b200 import gbdt
    rng = np.random.default_rng(seed)
    X = rng.integers(0, levels, (n, 164)).astype(np.float64)
    X[:, ::7] = rng.random((n, len(range(0, 164, 7))))            # some continuous columns
    target = np.round(rng.normal(size=n), 2)
    w = rng.integers(1, 4, n) / 4.0
    got = gbdt.fit_tree(X, target, w, depth)
    want = OT.fit_tree(X, target, w, depth)
    assert got.feature.tolist() == want["feature"]
    assert got.threshold.tolist() == want["threshold"]
    assert got.left.tolist() == want["left"] and got.right.tolist() == want["right"]
    assert got.value.tolist() == want["value"]
