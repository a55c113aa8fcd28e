"""Loader for the golden fixtures made by tools/make_golden.py from the reference."""

import json
import os

import numpy as np

from paper_2006_06762_b200.state import ComputeDAG, history_from_json, replay

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Corpus:
    def __init__(self):
        with open(os.path.join(GOLDEN, "corpus.json")) as fh:
            raw = json.load(fh)
        self.dags = {k: ComputeDAG.from_json(v) for k, v in raw["dags"].items()}
        self.entries = raw["programs"]
        self.programs = [replay(self.dags[e["dag"]], history_from_json(e["history"])) for e in self.entries]
        f = np.load(os.path.join(GOLDEN, "features.npz"))
        self.rows, self.offsets = f["rows"], f["offsets"]
        self.scores = np.load(os.path.join(GOLDEN, "scores.npy"))
        with open(os.path.join(GOLDEN, "model.json")) as fh:
            self.model_json = json.load(fh)

    def features_of(self, i):
        return self.rows[self.offsets[i]:self.offsets[i + 1]]


_CACHE = {}


def load_corpus():
    if "c" not in _CACHE:
        _CACHE["c"] = Corpus()
    return _CACHE["c"]
