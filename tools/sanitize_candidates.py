"""One candidate per template path, measured through the runner so that
compute-sanitizer can watch the candidate kernels (SURVEY.md §5 race detection):

  compute-sanitizer --tool racecheck --target-processes all python tools/sanitize_candidates.py
  compute-sanitizer --tool memcheck  --target-processes all python tools/sanitize_candidates.py

Paths: naive; tiled synchronous staging; tiled cp.async double-buffered;
register-overflow tile at -O1; register double buffer; 16-byte fetch quads;
conv with the padding fused into the fetch (zero-fill cp.async); cross-thread
reduction.  Shapes are reduced so every launch finishes quickly under the tool;
each candidate runs once (warm-up + one timed run)."""

import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


def states():
    import numpy as np
    import bench
    from loomtune.annotate import AnnotationPolicy, sample_program
    from paper_2006_06762_b200.integrate import make_gpu_sampler
    from paper_2006_06762_b200.sketch_rules import gpu_sketches_traced
    from paper_2006_06762_b200.state import build, replay
    from tests.test_xreduce import rfactor_history
    out = []
    dag, stream = bench.load_stream("G5")
    for i, label in ((0, "naive"), (3, "tiled sync"), (7, "tiled cp.async double-buffered"), (4, "tiled -O1"),
                     (26, "tiled register double buffer -O1")):
        out.append((f"G5#{i} {label}", replay(dag, stream[i])))
    dag, stream = bench.load_stream("TBG")
    out.append(("TBG#20 16-byte fetch quads", replay(dag, stream[20])))
    sample = make_gpu_sampler(sample_program)
    rng = np.random.default_rng(3)
    small = build("conv2d", h=14, w=14, ci=16, co=32, kernel=3, stride=1, pad=1, n=2)
    sk = [p for p, path in gpu_sketches_traced(small) if "gpu_smem" in path]
    for j in range(3):
        out.append((f"conv 2x14x14x16->32 padding fused into the fetch #{j}", sample(sk[j % len(sk)],
                                                                                 AnnotationPolicy(), rng)))
    nd = build("norm2", n=256, m=256)
    out.append(("norm2 cross-thread reduction", replay(nd, rfactor_history("r", ["i", "j"], 256, ["u"]))))
    return out


def main():
    """Optional argument: the index of one candidate (run one per process so a
    slow tool pass can be bounded per candidate with `timeout`)."""
    from paper_2006_06762_b200 import measure
    from paper_2006_06762_b200.ptxgen import lower_ptx
    r = measure.configure(device=0, cache_dir="", min_ms=0.0, max_repeat=1, workers=8)
    bad = 0
    chosen = states()
    if len(sys.argv) > 1:
        chosen = [chosen[int(sys.argv[1])]]
    for label, p in chosen:
        (rec,) = r.measure_programs([p])
        kinds = [k.info.get("template") for k in lower_ptx(p).kernels]
        print(f"{label}: {rec.status} {kinds} max_rel_err={rec.max_rel_err:.2e} {rec.detail}", flush=True)
        bad += rec.status != "valid"
    measure._shutdown()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
