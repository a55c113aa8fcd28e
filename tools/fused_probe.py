"""Fused vs unfused ResNet-50 task, same sampler: measure K GPU-sampled States of
each and print best / median cost and the best State's kernels.  Diagnoses a
whole-network search that stays near naive on a fused task.

  python tools/fused_probe.py [TASK] [K]
"""
import collections
import json
import os
import statistics
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


def main() -> None:
    import numpy as np
    from paper_2006_06762_b200 import integrate, measure, resnet50, sketch_rules
    import loomtune.annotate as AN
    import loomtune.ir as IR
    import loomtune.sketch as SK
    task = sys.argv[1] if len(sys.argv) > 1 else "conv7_2048_512_k1s1"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 96
    fused = {n: d for n, d, _ in resnet50.tasks(fusion="conv_bn_relu")}
    plain = {n: d for n, d, _ in resnet50.tasks()}
    samp = integrate.make_gpu_sampler(AN.sample_program)
    r = measure.configure(device=0, cache_dir="")
    for name, dag in ((task, plain[task]), (task + "_bn_relu", fused[task + "_bn_relu"])):
        traced = SK.generate_sketches_traced(dag, extra_rules=sketch_rules.GPU_RULES, structure="SSSRRSRS")
        keep = [i for i, (_, path) in enumerate(traced) if any(x in integrate.GPU_SKETCH_RULES for x in path)]
        keep = keep or list(range(len(traced)))
        rng = np.random.default_rng(0)
        progs = [samp(traced[keep[i % len(keep)]][0], AN.AnnotationPolicy(), rng) for i in range(k)]
        recs = r.measure_programs(progs)
        ok = [x for x in recs if x.status == "valid"]
        st = collections.Counter(x.status for x in recs)
        best = min(ok, key=lambda x: x.cost_us) if ok else None
        naive = r.measure_programs([IR.naive_program(dag)])[0]
        print(json.dumps({"task": name, "statuses": st, "best_us": best.cost_us if best else None,
                          "median_us": statistics.median(x.cost_us for x in ok) if ok else None,
                          "naive_us": naive.cost_us, "best_kernels": best.info.get("kernels") if best else None,
                          "invalid_details": collections.Counter(x.detail[:80] for x in recs if x.status != "valid")
                          .most_common(3)}), flush=True)
    measure._shutdown()


if __name__ == "__main__":
    main()
