"""Template-capability sweep: measure many legal SSSRRSRS tilings of a config
directly (no cost model, no evolution) to see what the tiled template reaches.

  python tools/sweep_tilings.py CFG N [SEED]

Draws N random tilings with GPU-sane factor choices (threads 32-1024, vthread
<= 8, accumulators 8-128), measures them with the runner, prints the top ten.
Calibration only: the search itself stays the reference's.
"""

from __future__ import annotations

import json
import os
import random
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from hand_states import tiled  # noqa: E402

from paper_2006_06762_b200.lower import LoweringError, lower  # noqa: E402
from paper_2006_06762_b200.state import config_dag  # noqa: E402


def divisors(n):
    return [d for d in range(1, n + 1) if n % d == 0]


def draw(rng, ext, parts):
    """Random ordered factorization of ext into `parts` factors (outer first)."""
    out, rest = [], ext
    for _ in range(parts - 1):
        d = rng.choice(divisors(rest))
        out.append(d)
        rest //= d
    out.append(rest)
    rng.shuffle(out)
    return out


def main() -> None:
    cfg, n = sys.argv[1], int(sys.argv[2])
    rng = random.Random(int(sys.argv[3]) if len(sys.argv) > 3 else 0)
    dag = config_dag(cfg)
    stage = next(s for s in dag.nodes if s.reduce)
    name = stage.name
    progs, seen = [], set()
    tries = 0
    while len(progs) < n and tries < n * 400:
        tries += 1
        sp = {a: draw(rng, e, 5)[1:] for a, e in stage.space}
        rd = {r: draw(rng, e, 3)[1:] for r, e in stage.reduce}
        p = tiled(dag, name, sp, rd, unroll=rng.choice([64, 512]))
        try:
            lo = lower(p)
        except LoweringError:
            continue
        k = next(x for x in lo.kernels if x.info["template"] == "tiled").info
        if not (64 <= k["threads"] <= 512 and 8 <= k["acc"] <= 128 and k["blocks"] >= 64):
            continue
        if lo.source in seen:
            continue
        seen.add(lo.source)
        progs.append((p, sp, rd))
    from bench import FLOPS
    from paper_2006_06762_b200 import measure
    r = measure.configure(device=0, cache_dir="")
    recs = r.measure_programs([p for p, _, _ in progs])
    res = sorted(((rec.cost_us, i) for i, rec in enumerate(recs) if rec.status == "valid"))
    print(json.dumps({"config": cfg, "drawn": len(progs), "valid": len(res)}))
    for us, i in res[:10]:
        info = next(x for x in recs[i].info["kernels"] if x["template"] == "tiled")
        print(json.dumps({"us": us, "tflops": FLOPS[cfg] / (us * 1e-6) / 1e12, "threads": info["threads"],
                          "blocks": info["blocks"], "acc": info["acc"], "vthreads": info["vthreads"],
                          "smem": info["smem"], "space": progs[i][1], "reduce": progs[i][2]}))
    measure._shutdown()


if __name__ == "__main__":
    main()
