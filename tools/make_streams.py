"""Candidate-State streams for bench.py, generated with the REFERENCE's sampler.

Run in the build container:  python tools/make_streams.py [n_per_config]

For each BASELINE config (SURVEY.md §8(a) short names) draw States with the
reference's own `sample_program` over `generate_sketches(dag, "SSSRRSRS")`
(round-robin over sketches, fixed seed, default AnnotationPolicy), keep the
ones that have a legal B200 launch under `paper_2006_06762_b200.lower`
(threads <= 1024, smem <= 227 KB, ...), de-duplicated by generated source, and
write tests/golden/streams/<CFG>.json.gz = {"dag": DAG JSON, "histories": [...]}.
The sampler is not GPU-aware (SURVEY.md §7 hard part 2), so this filter is the
only selection applied; evolution is not involved.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.environ.get("LOOMTUNE_REF", "/root/reference/pkg/src"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

import loomtune as LT  # noqa: E402
from loomtune.ir import history_to_json  # noqa: E402
from loomtune.sketch import generate_sketches  # noqa: E402

from paper_2006_06762_b200 import lower as LW  # noqa: E402
from paper_2006_06762_b200.state import ComputeDAG, history_from_json, replay  # noqa: E402
from paper_2006_06762_b200.state import workloads as W  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "streams")


def stream(cfg: str, n: int, max_draws: int = int(os.environ.get("LT_MAX_DRAWS", "250000"))) -> dict:
    name, kw = W.CONFIGS[cfg]
    ours = W.build(name, **kw)
    ref = LT.ComputeDAG.from_json(ours.to_json())
    sketches = generate_sketches(ref, structure="SSSRRSRS")
    rng = np.random.default_rng(2024)
    seen, hist = set(), []
    draws = 0
    t0 = time.time()
    while len(hist) < n and draws < max_draws:
        sk = sketches[draws % len(sketches)]
        draws += 1
        p = LT.sample_program(sk, LT.AnnotationPolicy(), rng)
        h = history_to_json(p.history)
        q = replay(ours, history_from_json(h))
        try:
            lo = LW.lower(q)
        except LW.LoweringError:
            continue
        key = hashlib.sha1(lo.source.encode()).hexdigest()
        if key in seen:
            continue
        seen.add(key)
        hist.append(h)
    print(f"{cfg}: {len(hist)} legal distinct of {draws} draws ({time.time() - t0:.0f}s)")
    return {"config": cfg, "dag": ours.to_json(), "histories": hist, "draws": draws}


def main() -> None:
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    cfgs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["RC", "G10", "TBG", "CL", "G5"]
    os.makedirs(OUT, exist_ok=True)
    for cfg in cfgs:
        data = stream(cfg, n)
        with gzip.open(os.path.join(OUT, f"{cfg}.json.gz"), "wt") as fh:
            json.dump(data, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()
