"""ORACLE (test infrastructure only): CPU restatement of GBDT training,
`train` and `_fit_tree` (`src/model.py:158-320`).

Pinned against the reference: `tests/golden/train.npz` holds the labels with
which the reference's own `train` produced `tests/golden/model.json`, and
`tests/golden/train_models.json` holds reference-trained models on tie-heavy
variants (made by tools/make_golden_train.py with the reference imported);
`tests/test_oracle.py` requires this restatement to reproduce every one of
them exactly (`to_json` equality).

The arithmetic is the reference's, operation for operation, because split
choice and leaf values are compared bit-for-bit:

* rows of the frontier, per feature, in (node id, feature value, row) order;
  one running float64 `cumsum` of w and of w*target across the whole
  concatenation (`src/model.py:179-191`); left/right sums are differences of
  that running sum with the value before the node's first row;
* gain = ((sl*sl/max(wl,tiny)) + (sr*sr/max(wr,tiny))) - (gs*gs/max(gw,tiny)),
  candidates only between distinct neighbouring values with wl>0, wr>0
  (`src/model.py:193-208`); per node the first position of the maximum gain,
  features visited in order and replaced only by a strictly larger gain,
  threshold 0.5*(x[p]+x[p+1]) (`src/model.py:209-220`);
* children numbered in frontier order; leaf value = numpy sum of w*target over
  the leaf's rows in row order / numpy sum of w (`src/model.py:239-247`);
* boosting: base from throughput-weighted statement counts, residual split
  evenly over a program's statements, per-program sums of tree outputs in row
  order (`np.bincount`), halving line search of at most 12 halvings
  (`src/model.py:275-320`).
"""

from __future__ import annotations

import numpy as np

EPS_GAIN = 1e-12
MAX_HALVINGS = 12
TINY = 1e-300


def tree_predict(tree: dict, X: np.ndarray) -> np.ndarray:
    """Per-row tree output (value[leaf] * eta), vectorised level by level."""
    feat = np.asarray(tree["feature"], np.int64)
    thr = np.asarray(tree["threshold"], np.float64)
    left = np.asarray(tree["left"], np.int64)
    right = np.asarray(tree["right"], np.int64)
    value = np.asarray(tree["value"], np.float64)
    idx = np.zeros(len(X), np.int64)
    if len(X) == 0:
        return np.zeros(0)
    for _ in range(64):
        f = feat[idx]
        inner = f >= 0
        if not inner.any():
            break
        fx = X[np.arange(len(X)), np.maximum(f, 0)]
        idx = np.where(inner, np.where(fx <= thr[idx], left[idx], right[idx]), idx)
    return value[idx] * tree["eta"]


def fit_tree(X: np.ndarray, target: np.ndarray, w: np.ndarray, depth: int) -> dict:
    n, nf = X.shape
    order = [np.argsort(X[:, f], kind="stable") for f in range(nf)]
    feature, threshold, left, right = [-1], [0.0], [0], [0]
    node_of = np.zeros(n, np.int64)
    frontier = [0]
    for _ in range(depth):
        if not frontier:
            break
        in_frontier = np.isin(node_of, frontier)
        best: dict = {}
        for f in range(nf):
            o = order[f]
            o = o[in_frontier[o]]
            if len(o) < 2:
                continue
            # group by node id (ascending), keeping value order inside a node
            rows = o[np.argsort(node_of[o], kind="stable")]
            g = node_of[rows]
            xw, xv = w[rows], X[rows, f]
            cw = np.cumsum(xw)
            cs = np.cumsum(xw * target[rows])
            bounds = np.flatnonzero(np.diff(g)) + 1
            starts = np.concatenate([[0], bounds]).astype(np.int64)
            ends = np.concatenate([bounds, [len(g)]]).astype(np.int64)
            gid = np.repeat(np.arange(len(starts)), ends - starts)
            bw = np.where(starts > 0, cw[np.maximum(starts - 1, 0)], 0.0)
            bs = np.where(starts > 0, cs[np.maximum(starts - 1, 0)], 0.0)
            gw, gs = cw[ends - 1] - bw, cs[ends - 1] - bs
            wl, sl = cw - bw[gid], cs - bs[gid]
            wr, sr = gw[gid] - wl, gs[gid] - sl
            ok = np.zeros(len(g), bool)
            ok[:-1] = xv[:-1] != xv[1:]
            ok[ends - 1] = False
            ok &= (wl > 0) & (wr > 0)
            parent = gs * gs / np.maximum(gw, TINY)
            with np.errstate(invalid="ignore", over="ignore"):
                gain = np.where(ok, sl * sl / np.maximum(wl, TINY) + sr * sr / np.maximum(wr, TINY) - parent[gid],
                                -np.inf)
            for k, (a, b) in enumerate(zip(starts, ends)):
                seg = gain[a:b]
                if np.isnan(seg).any():
                    continue
                gmax = seg.max()
                if not (gmax > EPS_GAIN) or not np.isfinite(gmax):
                    continue
                p = int(a + np.flatnonzero(seg == gmax)[0])
                nd = int(g[a])
                if nd not in best or gmax > best[nd][0]:
                    best[nd] = (float(gmax), f, float(0.5 * (xv[p] + xv[p + 1])))
        nxt = []
        for nd in frontier:
            if nd not in best:
                continue
            _, f, thr = best[nd]
            li = len(feature)
            feature[nd], threshold[nd], left[nd], right[nd] = f, thr, li, li + 1
            feature += [-1, -1]
            threshold += [0.0, 0.0]
            left += [0, 0]
            right += [0, 0]
            here = node_of == nd
            go = here & (X[:, f] <= thr)
            node_of[go] = li
            node_of[here & ~go] = li + 1
            nxt += [li, li + 1]
        frontier = nxt
    value = np.zeros(len(feature))
    for nd in range(len(feature)):
        if feature[nd] >= 0:
            continue
        here = node_of == nd
        ww = w[here]
        tot = ww.sum()
        if tot > 0:
            value[nd] = float((ww * target[here]).sum() / tot)
    return {"feature": feature, "threshold": threshold, "left": left, "right": right,
            "value": value.tolist(), "eta": 1.0}


def train(mats: list, y: np.ndarray, trees: int = 30, depth: int = 6, shrinkage: float = 0.3,
          fit=fit_tree) -> dict:
    """mats: one feature matrix per program (positive labels y).  Returns the
    model in the reference's `CostModel.to_json` layout plus "train_losses"."""
    y = np.asarray(y, np.float64)
    X = np.vstack(mats)
    prog = np.concatenate([np.full(len(m), i, np.int64) for i, m in enumerate(mats)])
    n_stmt = np.asarray([len(m) for m in mats], np.float64)
    wp = y.copy()
    row_w = wp[prog]
    denom = float((wp * n_stmt * n_stmt).sum())
    base = float((wp * y * n_stmt).sum() / denom) if denom > 0 else 0.0
    pred = base * n_stmt

    def loss_of(p):
        return float((wp * (p - y) ** 2).sum())

    loss = loss_of(pred)
    losses = [loss]
    out = []
    for _ in range(trees):
        target = ((y - pred) / n_stmt)[prog]
        tree = fit(X, target, row_w, depth)
        per_prog = np.bincount(prog, weights=tree_predict(tree, X), minlength=len(mats))
        eta = shrinkage
        for _h in range(MAX_HALVINGS + 1):
            new_loss = loss_of(pred + eta * per_prog)
            if new_loss <= loss:
                break
            eta *= 0.5
        else:
            eta, new_loss = 0.0, loss
        if eta == 0.0:
            losses.append(loss)
            continue
        tree["eta"] = eta
        out.append(tree)
        pred = pred + eta * per_prog
        loss = new_loss
        losses.append(loss)
    return {"base": base, "n_features": X.shape[1], "shrinkage": shrinkage, "depth": depth,
            "trees": out, "train_losses": losses}
