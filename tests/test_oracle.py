"""The oracle is pinned to the reference's own outputs (golden fixtures)."""

import numpy as np

from oracle import features as OF
from oracle import predict as OP


def test_oracle_features_reproduce_reference_exactly(corpus):
    for i, p in enumerate(corpus.programs):
        got = OF.extract_features(p)
        want = corpus.features_of(i)
        assert got.shape == want.shape, corpus.entries[i]["origin"]
        assert np.array_equal(got, want), (i, corpus.entries[i]["dag"], np.argwhere(got != want)[:4])


def test_oracle_scores_reproduce_reference_exactly(corpus):
    model = OP.load_model(corpus.model_json)
    for i in range(0, len(corpus.programs), 7):
        got = OP.predict_matrix(model, corpus.features_of(i))
        assert got == corpus.scores[i], i


def test_onehot_mask_matches_layout():
    names = []
    kinds = ("add", "sub", "mul", "div", "minmax", "cmp", "math_call", "select", "other")
    pos = OF.POS
    names += ["float_" + k for k in kinds] + ["int_" + k for k in kinds]
    for blk in ("vec", "unroll", "par"):
        names += [blk + "_len"] + [f"{blk}_pos_{p}" for p in pos] + [blk + "_prod", blk + "_num"]
    names += ["gpu"] * 8 + ["intensity"] * 10
    for b in range(5):
        names += [f"buf{b}_acc_{t}" for t in OF.ACC] + ["x"] * 4 + [f"buf{b}_reuse_{t}" for t in OF.REUSE] + ["x"] * 8
    names += ["x"] * 5
    assert len(names) == 164
    want = np.array([("_pos_" in n or "_acc_" in n or "_reuse_" in n) for n in names])
    assert (OF.ONEHOT == want).all()
