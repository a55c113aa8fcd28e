"""GBDT training on the B200: drop-in for the reference's `train`
(`src/model.py:275-320`) with `_fit_tree` (`src/model.py:158-255`) on the GPU.

`train(records, hyper)` keeps the reference's interface and returns a
`GpuCostModel` whose `to_json()` equals the reference model's, bit for bit
(tests/test_gbdt_gpu.py against tests/golden/train*.{npz,json}).  The boosting
loop is O(programs) host arithmetic in numpy, in the reference's exact
operation order (base from throughput-weighted statement counts, residual
shared evenly by a program's statements, per-program `np.bincount` of the tree
outputs, halving line search); each tree is one `lt_gbdt_fit_tree` call on a
device-resident copy of the training matrix whose feature columns are sorted
once per `train` call (`csrc/gbdt.cu`).  No CPU fallback: without the library
or a device, `train` raises.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import runtime as rt
from .model import GpuCostModel, Hyper, N_FEATURES, Tree

EPS_GAIN = 1e-12          # src/model.py:26
MAX_HALVINGS = 12         # src/model.py:27


class DeviceMatrix:
    """A training matrix resident on the device with its per-feature sort order."""

    def __init__(self, X: np.ndarray):
        self.lib = rt.load()
        X = np.ascontiguousarray(X, dtype=np.float64)
        self.n, self.nf = X.shape
        self.h = self.lib.lt_gbdt_create(rt.ptr(X, rt.c_f64p), self.n, self.nf)
        self.epoch = rt.epoch
        if not self.h:
            raise rt.NativeError(f"lt_gbdt_create: {self.lib.lt_last_error().decode()}")

    def fit_tree(self, target: np.ndarray, w: np.ndarray, depth: int) -> Tree:
        cap = (2 << depth) - 1
        feat = np.empty(cap, np.int32)
        left = np.empty(cap, np.int32)
        right = np.empty(cap, np.int32)
        thr = np.empty(cap, np.float64)
        val = np.empty(cap, np.float64)
        nn = ctypes.c_int32()
        t = np.ascontiguousarray(target, np.float64)
        ww = np.ascontiguousarray(w, np.float64)
        rt.check(self.lib.lt_gbdt_fit_tree(self.h, rt.ptr(t, rt.c_f64p), rt.ptr(ww, rt.c_f64p), int(depth), cap,
                                           rt.ptr(feat, rt.c_i32p), rt.ptr(thr, rt.c_f64p), rt.ptr(left, rt.c_i32p),
                                           rt.ptr(right, rt.c_i32p), rt.ptr(val, rt.c_f64p), ctypes.byref(nn)),
                 "lt_gbdt_fit_tree")
        k = nn.value
        return Tree(feat[:k].astype(np.int64), thr[:k].copy(), left[:k].astype(np.int64),
                    right[:k].astype(np.int64), val[:k].copy(), 1.0)

    def close(self):
        if self.h and self.epoch == rt.epoch:     # after rt.shutdown() the library is torn down
            self.lib.lt_gbdt_destroy(self.h)
        self.h = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


MAX_DEPTH = 7       # csrc/gbdt.cu GB_MAX_FRONTIER = 64 nodes per level


_LAST: list = [None, None]      # (weakref to the host matrix, DeviceMatrix)


def fit_tree(X: np.ndarray, target: np.ndarray, w: np.ndarray, depth: int) -> Tree:
    """`_fit_tree(X, target, w, depth)` (src/model.py:158) on the device.  The
    device copy of X (and its sort order) is reused while the caller keeps
    passing the same matrix object, as `train` does for all its trees."""
    ref, dm = _LAST
    if ref is None or ref() is not X or dm.n != len(X):
        if dm is not None:
            dm.close()
        dm = DeviceMatrix(X)
        _LAST[0], _LAST[1] = weakref.ref(X), dm
    return dm.fit_tree(target, w, depth)


def _tree_predict(t: Tree, X: np.ndarray) -> np.ndarray:
    """`Tree.predict` (src/model.py:75-88): value[leaf] * eta, level-synchronous."""
    idx = np.zeros(len(X), np.int64)
    if len(X) == 0:
        return np.zeros(0)
    rows = np.arange(len(X))
    for _ in range(64):
        f = t.feature[idx]
        inner = f >= 0
        if not inner.any():
            break
        fx = X[rows, np.maximum(f, 0)]
        idx = np.where(inner, np.where(fx <= t.threshold[idx], t.left[idx], t.right[idx]), idx)
    return t.value[idx] * t.eta


def train(records, hyper=None) -> GpuCostModel:
    """`train(records, hyper)` (src/model.py:275): records with y > 0 and
    attached features; returns a GpuCostModel equal to the reference's model."""
    hyper = hyper if hyper is not None else Hyper()
    if not 1 <= hyper.depth <= MAX_DEPTH:
        raise ValueError(f"gbdt.train fits trees of depth 1..{MAX_DEPTH} on the device (got {hyper.depth})")
    usable = [r for r in records if r.y > 0]
    if not usable:
        raise ValueError("training needs at least one record with positive throughput")
    for r in usable:
        if r.feats is None:
            raise ValueError(f"record for {r.dag_id} has no features attached")
    X = np.vstack([r.feats for r in usable])
    if X.shape[1] != N_FEATURES:
        raise ValueError("feature rows must be 164 wide")
    prog = np.concatenate([np.full(len(r.feats), i, dtype=np.int64) for i, r in enumerate(usable)])
    y = np.asarray([r.y for r in usable])
    n_stmt = np.asarray([len(r.feats) for r in usable], dtype=np.float64)
    wp = y.copy()
    row_w = wp[prog]
    denom = float((wp * n_stmt * n_stmt).sum())
    base = float((wp * y * n_stmt).sum() / denom) if denom > 0 else 0.0
    model = GpuCostModel(base=base, hyper=hyper)
    pred = base * n_stmt

    def loss_of(p: np.ndarray) -> float:
        return float((wp * (p - y) ** 2).sum())

    loss = loss_of(pred)
    model.train_losses.append(loss)
    dm = DeviceMatrix(X)
    try:
        for _ in range(hyper.trees):
            target = ((y - pred) / n_stmt)[prog]
            tree = dm.fit_tree(target, row_w, hyper.depth)
            per_prog = np.bincount(prog, weights=_tree_predict(tree, X), minlength=len(usable))
            eta = hyper.shrinkage
            for _h in range(MAX_HALVINGS + 1):
                new_loss = loss_of(pred + eta * per_prog)
                if new_loss <= loss:
                    break
                eta *= 0.5
            else:
                eta, new_loss = 0.0, loss
            if eta == 0.0:
                model.train_losses.append(loss)
                continue
            tree.eta = eta
            model.trees.append(tree)
            pred = pred + eta * per_prog
            loss = new_loss
            model.train_losses.append(loss)
    finally:
        dm.close()
    return model
