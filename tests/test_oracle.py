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


def test_oracle_reference_outputs_match_golden():
    import os
    from oracle import interp as OI
    from paper_2006_06762_b200.state import build
    from tests.tools_shapes import SMALL
    outs = np.load(os.path.join(os.path.dirname(__file__), "golden", "outputs.npz"))
    for name, kw in SMALL.items():
        dag = build(name, **kw)
        got = OI.reference_outputs(dag, OI.random_inputs(dag, np.random.default_rng(0)), chunk=1 << 12)
        for o, arr in got.items():
            np.testing.assert_allclose(arr, outs[f"{name}/{o}"], rtol=1e-13, atol=0)


def test_oracle_interpret_matches_ground_truth(corpus):
    """Every corpus State at small shape interprets to the reference ground truth."""
    from oracle import interp as OI
    for i, (p, e) in enumerate(zip(corpus.programs, corpus.entries)):
        if ":" not in e["dag"] or i % 3:
            continue
        ins = OI.random_inputs(p.dag, np.random.default_rng(0))
        got = OI.interpret(p, ins)
        want = OI.reference_outputs(p.dag, ins)
        for o in want:
            err = np.max(np.abs(got[o] - want[o]) / np.maximum(np.abs(want[o]), 1e-30))
            assert err <= 1e-9, (i, e["dag"], err)


def test_oracle_measure_batch_matches_reference(corpus):
    """Statuses, details, exact analytical costs and throughputs of the reference."""
    import json
    import math
    import os
    from oracle import machine as OM
    from paper_2006_06762_b200.state import ComputeDAG, history_from_json, replay
    with open(os.path.join(os.path.dirname(__file__), "golden", "measure.json")) as fh:
        cases = json.load(fh)
    for case in cases:
        dag = corpus.dags[case["dag"]]
        progs = [replay(dag, history_from_json(h)) for h in case["histories"]]
        res = OM.measure_batch(progs)
        for r, (cost, thr, status, detail) in zip(res, case["results"]):
            assert r.status == status and r.detail == detail
            assert (r.cost == math.inf) if cost == "inf" else (r.cost == cost)
            assert r.throughput == thr


def _train_cases():
    import json
    import os
    import numpy as np
    from tests.golden_corpus import GOLDEN, load_corpus
    c = load_corpus()
    t = np.load(os.path.join(GOLDEN, "train.npz"))
    mats = [c.features_of(i) for i in range(len(c.programs))]
    out = [("corpus (tests/golden/model.json)", mats, t["y"], {"trees": 30, "depth": 6, "shrinkage": 0.3},
            c.model_json, None)]
    for case in json.load(open(os.path.join(GOLDEN, "train_models.json"))):
        offs = case["offsets"]
        if case["source"] == "corpus":
            rows = c.rows
        elif case["source"]:
            rows = np.vstack([np.round(mats[i], 1) for i in range(0, len(mats), 3)])
        else:
            rows = np.asarray(case["rows"], np.float64)
        m = [rows[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
        out.append((case["name"], m, np.asarray(case["y"]), case["hyper"], case["model"], case["train_losses"]))
    return out


def test_oracle_train_reproduces_reference_models():
    """oracle/train.py == the reference's own `train` on every golden case (exact)."""
    from oracle import train as OT
    for name, mats, y, hyper, want, losses in _train_cases():
        got = OT.train(mats, y, **hyper)
        got_losses = got.pop("train_losses")
        assert got == want, name
        if losses is not None:
            assert got_losses == losses, name
