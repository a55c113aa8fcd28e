"""Profiling driver (run under ncu on the GPU box).

  python tools/profile_best.py CFG N [OFFSET]
                                         measure N stream States of CFG from OFFSET
                                         (bench.py's timed steps are RC 128 from 96),
                                         then re-launch the best one's kernels 3x
                                         inside an NVTX range "profile"; writes
                                         gpurun_out/best_CFG.json (kernel hashes)
  python tools/profile_best.py --scoring  run the population-scoring kernels once
                                         inside the NVTX range

ncu --nvtx --nvtx-include "profile/" --set full ... python tools/profile_best.py RC 64
"""

from __future__ import annotations

import ctypes
import json
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


def best_candidate(cfg: str, n: int, offset: int = 0) -> None:
    import torch
    from bench import load_stream
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200 import runtime as rt
    from paper_2006_06762_b200.state import replay
    dag, stream = load_stream(cfg)
    runner = measure.RunnerCore(device=0, cache_dir="")
    progs = [replay(dag, h) for h in stream[offset:offset + n]]
    recs = runner.measure_programs(progs)
    best = min((r.cost_us, i) for i, r in enumerate(recs) if r.status == "valid")
    p = progs[best[1]]
    lo = runner.lower(p)
    key = __import__("hashlib").sha1(lo.source.encode()).hexdigest()
    out = {"config": cfg, "best_us": best[0], "index": offset + best[1], "source_sha1": key,
           "kernels": [k.entry for k in lo.kernels], "info": lo.info}
    print(json.dumps(out), flush=True)
    with open(os.path.join(ROOT, "gpurun_out", f"best_{cfg}.json"), "w") as fh:
        json.dump(out, fh)
    with open(os.path.join(ROOT, "gpurun_out", f"best_{cfg}.src"), "w") as fh:
        fh.write(lo.source)
    funcs = []                  # one module per kernel (measure._modules_of), keyed as the runner keys them
    for ents, text, opts in measure._modules_of(lo):
        kkey = __import__("hashlib").sha1((opts or "").encode() + text.encode()).hexdigest()
        funcs += runner.load(kkey, b"", ents)
    ctx = runner.context(p.dag, 0)
    launches = ctx._launches(lo, funcs)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("profile")
    for _ in range(3):
        rt.check(runner.lib.lt_task_run(ctx.task, ctypes.addressof(launches), len(lo.kernels)), "run")
    torch.cuda.nvtx.range_pop()
    measure._shutdown()


def scoring() -> None:
    import torch
    from bench import load_stream, scoring_bench
    from paper_2006_06762_b200.state import replay
    dag, stream = load_stream("RC")
    progs = [replay(dag, h) for h in stream[:256]]
    torch.cuda.nvtx.range_push("profile")
    print(json.dumps(scoring_bench(0, progs, reps=1)))
    torch.cuda.nvtx.range_pop()


if __name__ == "__main__":
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    if sys.argv[1] == "--scoring":
        scoring()
    else:
        best_candidate(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 0)
