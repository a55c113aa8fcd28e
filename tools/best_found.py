"""Measure the best-found program per operator (profiles/r02_tuned_best.json, or
the file named by LT_TUNED_BEST) through the runner, three times each, and print
µs / TFLOP/s / fraction of the FFMA peak.  Used for template A/B runs
(LT_PTX_OFF=...) on the programs the search actually found.

  python tools/best_found.py [CFG,...]
"""

import ctypes
import json
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


def main():
    from bench import FLOPS
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200 import runtime as rt
    from paper_2006_06762_b200.state import config_dag, history_from_json, replay
    path = os.environ.get("LT_TUNED_BEST", os.path.join(ROOT, "profiles", "r02_tuned_best.json"))
    best = json.load(open(path))
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else list(best)
    r = measure.configure(device=0, cache_dir="")
    lib = rt.load()
    tf, ms = ctypes.c_double(), ctypes.c_double()
    rt.check(lib.lt_ffma_peak(0, ctypes.byref(tf), ctypes.byref(ms)), "peak")
    for cfg in cfgs:
        p = replay(config_dag(cfg), history_from_json(best[cfg]["history"]))
        us = []
        for _ in range(3):
            r.drop_contexts()
            (rec,) = r.measure_programs([p])
            us.append(rec.cost_us if rec.status == "valid" else float("nan"))
        u = min(us)
        print(json.dumps({"config": cfg, "us": us, "best_us": u, "tflops": FLOPS[cfg] / u / 1e6,
                          "frac": FLOPS[cfg] / u / 1e6 / tf.value, "peak": tf.value, "status": rec.status,
                          "detail": rec.detail, "off": os.environ.get("LT_PTX_OFF", ""),
                          "kernels": rec.info.get("kernels")}), flush=True)
    measure._shutdown()


if __name__ == "__main__":
    main()
