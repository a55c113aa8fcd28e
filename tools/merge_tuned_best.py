"""Merge tools/tune_gpu.py outputs (gpurun_out/tune_<CFG>_s<SEED>[_rules].json.gz)
into profiles/r02_tuned_best.json: per config the best program over all seeds,
plus every seed's best in `seeds` (the seed spread).

  python tools/merge_tuned_best.py [GLOB] [--fresh]
"""

import glob
import gzip
import json
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    pattern = args[0] if args else os.path.join(ROOT, "gpurun_out", "tune_*.json.gz")
    path = os.path.join(ROOT, "profiles", "r02_tuned_best.json")
    # seeds already merged (earlier tune batches whose outputs are gone) are kept
    out = json.load(open(path)) if "--fresh" not in sys.argv and os.path.exists(path) else {}
    for tpath in sorted(glob.glob(pattern)):
        with gzip.open(tpath, "rt") as fh:
            d = json.load(fh)
        cfg = d["config"]
        entry = {"best_us": d["best_us"], "best_tflops": d["best_tflops"], "seed": d["seed"],
                 "trials": d["measured"], "valid": d["valid"], "wall_s": d["wall_s"], "timers": d["timers"],
                 "source": f"tools/tune_gpu.py {cfg} {d['budget']} {d['seed']} --gpu-sampler"
                           f"{' --gpu-rules' if d.get('gpu_rules') else ' --gpu-sketches'} (round 2)",
                 "history": d["best_history"]}
        cur = out.get(cfg)
        seeds = [x for x in (cur or {}).get("seeds", []) if x["seed"] != entry["seed"]]
        seeds += [{k: entry[k] for k in ("seed", "best_us", "best_tflops", "trials", "wall_s", "source")}]
        if cur is None or entry["best_us"] < cur["best_us"]:
            cur = entry
        cur["seeds"] = sorted(seeds, key=lambda x: x["seed"])
        out[cfg] = cur
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    for c, v in out.items():
        print(c, round(v["best_us"], 2), round(v["best_tflops"], 2), "seeds:",
              [(s["seed"], round(s["best_us"], 1)) for s in v["seeds"]])


if __name__ == "__main__":
    main()
