"""GPU-backed cost model: drop-in for the reference's `CostModel`
(`src/model.py:91-150`) with a batched population scorer.

`GpuCostModel` keeps the reference's public fields (`base`, `trees`, `hyper`,
`train_losses`) and methods (`predict_rows`, `predict_matrix`, `predict`,
`to_json`/`from_json`/`dumps`/`loads`) and adds `predict_batch(programs)`, which
scores a whole population in one fused device pass (encode on the host ->
features kernel -> tree kernel -> per-program sum).  Training stays the
reference's `train` (north star: "train interface stays unchanged"); `wrap`
converts its result.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from . import runtime as rt
from .encode import encode_batch

N_FEATURES = 164


@dataclass
class Tree:
    """Same fields as `src/model.py:66-73`."""
    feature: np.ndarray
    threshold: np.ndarray
    left: np.ndarray
    right: np.ndarray
    value: np.ndarray
    eta: float


@dataclass(frozen=True)
class Hyper:
    trees: int = 30
    depth: int = 6
    shrinkage: float = 0.3


@dataclass
class GpuCostModel:
    base: float = 0.0
    trees: list = field(default_factory=list)
    hyper: object = field(default_factory=Hyper)
    train_losses: list = field(default_factory=list)
    _handle: int = field(default=0, repr=False, compare=False)
    gpu_features: bool = field(default=False, compare=False)   # opt-in gpu_* feature slots
    _epoch: int = field(default=-1, repr=False, compare=False)

    # -- construction ------------------------------------------------------
    @staticmethod
    def wrap(model) -> "GpuCostModel":
        """From any object with the reference CostModel's fields."""
        if isinstance(model, GpuCostModel):
            return model
        m = GpuCostModel(base=float(model.base), hyper=model.hyper,
                         train_losses=list(getattr(model, "train_losses", [])))
        m.trees = [Tree(np.asarray(t.feature, np.int64), np.asarray(t.threshold, np.float64),
                        np.asarray(t.left, np.int64), np.asarray(t.right, np.int64),
                        np.asarray(t.value, np.float64), float(t.eta)) for t in model.trees]
        return m

    def to_json(self) -> dict:
        return {"base": self.base, "n_features": N_FEATURES, "shrinkage": self.hyper.shrinkage,
                "depth": self.hyper.depth,
                "trees": [{"eta": t.eta, "feature": np.asarray(t.feature).tolist(),
                           "threshold": np.asarray(t.threshold).tolist(), "left": np.asarray(t.left).tolist(),
                           "right": np.asarray(t.right).tolist(), "value": np.asarray(t.value).tolist()}
                          for t in self.trees]}

    @staticmethod
    def from_json(obj: dict) -> "GpuCostModel":
        if obj.get("n_features") != N_FEATURES:
            raise ValueError("model was built for a different feature layout")
        m = GpuCostModel(base=float(obj["base"]),
                         hyper=Hyper(len(obj["trees"]), int(obj.get("depth", 6)), float(obj["shrinkage"])))
        for t in obj["trees"]:
            m.trees.append(Tree(np.asarray(t["feature"], np.int64), np.asarray(t["threshold"], np.float64),
                                np.asarray(t["left"], np.int64), np.asarray(t["right"], np.int64),
                                np.asarray(t["value"], np.float64), float(t["eta"])))
        return m

    def dumps(self) -> str:
        return json.dumps(self.to_json(), sort_keys=True, separators=(",", ":"))

    @staticmethod
    def loads(s: str) -> "GpuCostModel":
        return GpuCostModel.from_json(json.loads(s))

    # -- device model --------------------------------------------------------
    def handle(self) -> int:
        if self._handle and self._epoch == rt.epoch:
            return self._handle
        self._handle = 0                    # created before a device reset: gone
        lib = rt.load()
        n = len(self.trees)
        off = np.zeros(n + 1, np.int64)
        for i, t in enumerate(self.trees):
            off[i + 1] = off[i] + len(t.feature)
        cat = lambda name, dt: (np.concatenate([np.asarray(getattr(t, name), dt) for t in self.trees])  # noqa: E731
                                if n else np.zeros(1, dt))
        feat, left, right = cat("feature", np.int32), cat("left", np.int32), cat("right", np.int32)
        thr, val = cat("threshold", np.float64), cat("value", np.float64)
        eta = np.asarray([t.eta for t in self.trees] or [0.0], np.float64)
        h = lib.lt_model_create(n, rt.ptr(off, rt.c_i64p), rt.ptr(feat, rt.c_i32p), rt.ptr(thr, rt.c_f64p),
                                rt.ptr(left, rt.c_i32p), rt.ptr(right, rt.c_i32p), rt.ptr(val, rt.c_f64p),
                                rt.ptr(eta, rt.c_f64p), float(self.base), N_FEATURES)
        if not h:
            raise rt.NativeError(f"lt_model_create: {lib.lt_last_error().decode()}")
        self._handle, self._epoch = h, rt.epoch
        return h

    def __del__(self):
        if self._handle and self._epoch == rt.epoch and rt._lib is not None:
            try:
                rt._lib.lt_model_destroy(self._handle)
            except Exception:
                pass

    # -- reference API ---------------------------------------------------------
    def predict_rows(self, X: np.ndarray) -> np.ndarray:
        X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, N_FEATURES)
        off = np.arange(len(X) + 1, dtype=np.int64)
        out = np.empty(len(X), np.float64)
        if len(X):
            lib = rt.load()
            rt.check(lib.lt_predict_batch(self.handle(), rt.ptr(X, rt.c_f64p), rt.ptr(off, rt.c_i64p), len(X),
                                          rt.ptr(out, rt.c_f64p)), "lt_predict_batch")
        return out

    def predict_matrix(self, X: np.ndarray) -> float:
        return float(self.predict_matrices([X])[0])

    def predict_matrices(self, mats: list) -> np.ndarray:
        """Scores of several row matrices (one per program) in one launch."""
        off = np.zeros(len(mats) + 1, np.int64)
        for i, m in enumerate(mats):
            off[i + 1] = off[i] + len(m)
        X = (np.ascontiguousarray(np.vstack(mats), dtype=np.float64) if off[-1]
             else np.zeros((1, N_FEATURES)))
        out = np.empty(len(mats), np.float64)
        if len(mats):
            lib = rt.load()
            rt.check(lib.lt_predict_batch(self.handle(), rt.ptr(X, rt.c_f64p), rt.ptr(off, rt.c_i64p), len(mats),
                                          rt.ptr(out, rt.c_f64p)), "lt_predict_batch")
        return out

    def predict(self, program) -> float:
        return float(self.predict_batch([program])[0])

    def predict_batch(self, programs, return_rows: bool = False):
        """Scores (and optionally the feature rows) of a whole population."""
        lib = rt.load()
        words, stmt_off, prog_off = encode_batch(programs, self.gpu_features)
        n_stmt = len(stmt_off) - 1
        scores = np.empty(len(programs), np.float64)
        rows = np.empty((n_stmt, N_FEATURES), np.float64) if return_rows else None
        if programs:
            rt.check(lib.lt_score_batch(self.handle(), rt.ptr(words, rt.c_i32p), rt.ptr(stmt_off, rt.c_i64p),
                                        n_stmt, rt.ptr(prog_off, rt.c_i64p), len(programs),
                                        rt.ptr(scores, rt.c_f64p),
                                        rt.ptr(rows, rt.c_f64p) if return_rows else None), "lt_score_batch")
        if return_rows:
            return scores, [rows[prog_off[i]:prog_off[i + 1]] for i in range(len(programs))]
        return scores
