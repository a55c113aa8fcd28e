"""ORACLE (test infrastructure only): CPU restatement of GBDT inference,
`Tree.predict` / `CostModel.predict_rows` / `predict_matrix`
(`src/model.py:75-108`).

Pinned against the reference: `tests/golden/model.json` is a model trained by
the reference's own `train` on corpus features, and `tests/golden/scores.npy`
holds the reference's `CostModel.predict` for every corpus State;
`tests/test_oracle.py` requires this restatement to reproduce them exactly.

Arithmetic order is the reference's: per row `base`, then each tree's
`value[leaf] * eta` added in list order; a program's score is numpy's sum of
its rows.
"""

from __future__ import annotations

import json

import numpy as np


def load_model(obj) -> dict:
    """Model dict in the reference's `CostModel.to_json` layout."""
    if isinstance(obj, (str, bytes)):
        obj = json.loads(obj)
    return obj


def leaf(tree: dict, x: np.ndarray) -> int:
    node = 0
    feat, thr, left, right = tree["feature"], tree["threshold"], tree["left"], tree["right"]
    for _ in range(64):
        f = feat[node]
        if f < 0:
            break
        node = left[node] if x[f] <= thr[node] else right[node]
    return node


def predict_rows(model: dict, X: np.ndarray) -> np.ndarray:
    out = np.full(len(X), float(model["base"]))
    for t in model["trees"]:
        vals = np.asarray(t["value"], dtype=np.float64)
        contrib = np.asarray([vals[leaf(t, x)] for x in X], dtype=np.float64) * float(t["eta"])
        out += contrib
    return out


def predict_matrix(model: dict, X: np.ndarray) -> float:
    return float(predict_rows(model, X).sum())
