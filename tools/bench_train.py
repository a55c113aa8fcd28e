"""GBDT training time: `gbdt.train` (trees on the B200) vs the CPU reference
(`loomtune.model.train` when importable, else oracle/train.py, the restatement
pinned to it) on record sets of tuning-run sizes.

  python tools/bench_train.py [N1,N2,...] [--cpu-only]

Records: golden-stream States of all four configs (features from the
reference-exact feature path), labels U(0.05, 1) with seed 0.  Prints one JSON
line per size with both times and whether the two models are identical.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


class Rec:
    def __init__(self, feats, y):
        self.feats, self.y, self.dag_id = feats, float(y), "d"


def main() -> None:
    sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 and sys.argv[1][0].isdigit()
                              else "600,1500,4000").split(",")]
    cpu_only = "--cpu-only" in sys.argv
    from bench import load_stream
    from paper_2006_06762_b200.state import replay
    feats = []
    if cpu_only:
        from oracle.features import extract_features
        ext = lambda ps: [extract_features(p) for p in ps]  # noqa: E731
    else:
        from paper_2006_06762_b200.features import extract_features_batch as ext
    for cfg in ("RC", "G10", "CL", "TBG"):
        dag, stream = load_stream(cfg)
        feats += ext([replay(dag, h) for h in stream[:max(sizes) // 4 + 1]])
    while len(feats) < max(sizes):          # beyond the streams: repeat programs (labels differ)
        feats += feats[:max(sizes) - len(feats)]
    rng = np.random.default_rng(0)
    ref = None
    for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "loomtune")):
            sys.path.insert(0, cand)
            try:
                from loomtune.model import TrainHyper, TrainingRecord, train as ref_train
                ref = (TrainHyper, TrainingRecord, ref_train)
            except ImportError:
                ref = None
            break
    for n in sizes:
        fs = feats[:n]
        y = rng.uniform(0.05, 1.0, len(fs))
        t0 = time.perf_counter()
        if ref is not None:
            TH, TR, rtrain = ref
            want = rtrain([TR("d", (), float(v), feats=f) for f, v in zip(fs, y)], TH()).to_json()
            kind = "reference loomtune.model.train"
        else:
            from oracle import train as OT
            want = OT.train(fs, y)
            want.pop("train_losses")
            kind = "oracle/train.py (restated reference)"
        cpu_s = time.perf_counter() - t0
        line = {"programs": len(fs), "rows": int(sum(len(f) for f in fs)), "cpu_s": cpu_s, "cpu_kind": kind}
        if not cpu_only:
            from paper_2006_06762_b200 import gbdt
            from paper_2006_06762_b200.model import Hyper
            gbdt.train([Rec(f, v) for f, v in zip(fs[:50], y[:50])], Hyper(trees=2))   # warm-up
            t0 = time.perf_counter()
            got = gbdt.train([Rec(f, v) for f, v in zip(fs, y)], Hyper()).to_json()
            line.update(gpu_s=time.perf_counter() - t0, identical=got == want)
            line["speedup"] = cpu_s / line["gpu_s"]
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
