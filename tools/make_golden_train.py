"""Golden fixtures for GBDT training (run HERE, with the reference importable).

  python tools/make_golden_train.py

Writes tests/golden/train.npz and tests/golden/train_models.json:

* the per-program labels `y` the reference's `train` saw when tools/make_golden.py
  produced tests/golden/model.json (best machine cost of the program's DAG over
  the program's machine cost, `src/machine.py:104`), checked to reproduce
  model.json exactly through the reference's own `train` (`src/model.py:275`);
* models the reference's `train` produces on variants that stress the exact
  greedy split (`src/model.py:158-255`): tied feature values, quantised labels
  (tied gains), other depths / tree counts / shrinkage, and a one-row program
  set.  Each case stores its rows, labels and the reference model JSON.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import loomtune as LT  # noqa: E402
from loomtune.machine import machine_cost  # noqa: E402
from loomtune.model import TrainHyper, TrainingRecord, train  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def main() -> None:
    raw = json.load(open(os.path.join(GOLD, "corpus.json")))
    dags = {k: LT.ComputeDAG.from_json(v) for k, v in raw["dags"].items()}
    progs = [(e["dag"], LT.replay(dags[e["dag"]], LT.ir.history_from_json(e["history"])))
             for e in raw["programs"]]
    f = np.load(os.path.join(GOLD, "features.npz"))
    rows, offs = f["rows"], f["offsets"]
    feats = [rows[offs[i]:offs[i + 1]] for i in range(len(progs))]
    costs = [machine_cost(p) for _, p in progs]
    best: dict = {}
    for (key, _), c in zip(progs, costs):
        best[key] = min(best.get(key, math.inf), c)
    y = np.asarray([best[key] / c for (key, _), c in zip(progs, costs)])
    recs = [TrainingRecord(key, p.history, float(yy), feats=ff) for (key, p), yy, ff in zip(progs, y, feats)]
    model = train(recs, TrainHyper())
    want = json.load(open(os.path.join(GOLD, "model.json")))
    assert model.to_json() == want, "labels do not reproduce tests/golden/model.json"
    np.savez_compressed(os.path.join(GOLD, "train.npz"), y=y, offsets=offs)

    rng = np.random.default_rng(7)
    cases = []

    def case(name, rws, ofs, yy, hyper, source=None):
        """source: how tests rebuild the rows from the corpus (None = rows stored)."""
        rs = [TrainingRecord("d", (), float(v), feats=rws[ofs[i]:ofs[i + 1]]) for i, v in enumerate(yy)]
        m = train(rs, hyper)
        cases.append({"name": name, "source": source, "rows": None if source else rws.tolist(),
                      "offsets": [int(x) for x in ofs], "y": [float(v) for v in yy],
                      "hyper": {"trees": hyper.trees, "depth": hyper.depth, "shrinkage": hyper.shrinkage},
                      "model": m.to_json(), "train_losses": [float(v) for v in m.train_losses]})

    # tied feature values and tied (quantised) labels on a corpus subset
    sub = np.arange(0, len(progs), 3)
    r2 = np.vstack([np.round(feats[i], 1) for i in sub])
    o2 = np.concatenate([[0], np.cumsum([len(feats[i]) for i in sub])])
    y2 = np.round(y[sub] * 4) / 4 + 0.25
    case("rounded_features_quantised_labels", r2, o2, y2, TrainHyper(trees=12, depth=5, shrinkage=0.5),
         source="corpus programs 0::3, features rounded to 1 decimal")
    # other hyperparameters on the full corpus
    case("full_depth3_trees8", rows, offs, y, TrainHyper(trees=8, depth=3, shrinkage=0.3), source="corpus")
    # small random integer-valued matrix: many ties everywhere
    n_prog = 40
    lens = rng.integers(1, 4, n_prog)
    o3 = np.concatenate([[0], np.cumsum(lens)])
    r3 = rng.integers(0, 4, (int(o3[-1]), 164)).astype(np.float64)
    y3 = rng.integers(1, 5, n_prog) / 4.0
    case("random_integer_ties", r3, o3, y3, TrainHyper(trees=10, depth=6, shrinkage=1.0))
    # single-row programs, constant labels (no useful split)
    r4 = np.ones((5, 164))
    case("constant", r4, np.arange(6), np.full(5, 0.5), TrainHyper(trees=3, depth=2, shrinkage=0.3))
    with open(os.path.join(GOLD, "train_models.json"), "w") as fh:
        json.dump(cases, fh)
    print(f"train.npz: {len(y)} labels; {len(cases)} extra cases: "
          + ", ".join(f"{c['name']} ({len(c['model']['trees'])} trees)" for c in cases))


if __name__ == "__main__":
    main()
