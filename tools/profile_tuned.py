"""Profile the best program the tuner found per operator (profiles/r02_tuned_best.json, or the
file named by LT_TUNED_BEST):
measure it through the runner, then relaunch its kernels 3x inside NVTX range "profile".

  ncu --set full --nvtx --nvtx-include "profile/" ... python tools/profile_tuned.py CFG
"""

import ctypes
import hashlib
import json
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


def main() -> None:
    import torch
    from bench import FLOPS
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200 import runtime as rt
    from paper_2006_06762_b200.state import config_dag, history_from_json, replay
    cfg = sys.argv[1]
    best = json.load(open(os.environ.get("LT_TUNED_BEST", os.path.join(ROOT, "profiles", "r02_tuned_best.json"))))[cfg]
    p = replay(config_dag(cfg), history_from_json(best["history"]))
    r = measure.RunnerCore(device=0, cache_dir="")
    (rec,) = r.measure_programs([p])
    lo = r.lower(p)
    print(json.dumps({"config": cfg, "status": rec.status, "us": rec.cost_us,
                      "tflops": FLOPS[cfg] / (rec.cost_us * 1e-6) / 1e12 if rec.status == "valid" else None,
                      "tuned_us": best["best_us"], "kernels": [k.info for k in lo.kernels]}), flush=True)
    funcs = []
    for ents, text, opts in measure._modules_of(lo):
        funcs += r.load(hashlib.sha1((opts or "").encode() + text.encode()).hexdigest(), b"", ents)
    ctx = r.context(p.dag, 0)
    launches = ctx._launches(lo, funcs)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("profile")
    for _ in range(3):
        rt.check(r.lib.lt_task_run(ctx.task, ctypes.addressof(launches), len(lo.kernels)), "run")
    torch.cuda.nvtx.range_pop()
    measure._shutdown()


if __name__ == "__main__":
    main()
