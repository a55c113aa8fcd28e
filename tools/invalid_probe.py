"""Candidates the runner rejects as wrong ("output ... differs from reference"):
regenerate the GPU-sampled States of a ResNet-50 task (tools/fused_probe.py's
sampler and seed), and for each rejected one print its kernels, the PTX-backend
error and the NVRTC (CUDA C) backend's verdict on the same State.

  python tools/invalid_probe.py [TASK] [K]
"""
import json
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


def main() -> None:
    import numpy as np
    from paper_2006_06762_b200 import integrate, measure, resnet50, sketch_rules
    from paper_2006_06762_b200.state import history_to_json
    import loomtune.annotate as AN
    import loomtune.sketch as SK
    task = sys.argv[1] if len(sys.argv) > 1 else "conv7_2048_512_k1s1"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 96
    dags = {n: d for n, d, _ in resnet50.tasks()}
    dags.update({n: d for n, d, _ in resnet50.tasks(fusion="conv_bn_relu")})
    dag = dags[task]
    samp = integrate.make_gpu_sampler(AN.sample_program)
    traced = SK.generate_sketches_traced(dag, extra_rules=sketch_rules.GPU_RULES, structure="SSSRRSRS")
    keep = [i for i, (_, path) in enumerate(traced) if any(x in integrate.GPU_SKETCH_RULES for x in path)]
    keep = keep or list(range(len(traced)))
    rng = np.random.default_rng(0)
    progs = [samp(traced[keep[i % len(keep)]][0], AN.AnnotationPolicy(), rng) for i in range(k)]
    ptx = measure.RunnerCore(device=0, cache_dir="", backend="ptx")
    recs = ptx.measure_programs(progs)
    bad = [(i, r) for i, r in enumerate(recs) if r.status != "valid"]
    nv = measure.RunnerCore(device=0, cache_dir="", backend="nvrtc")
    nrecs = nv.measure_programs([progs[i] for i, _ in bad]) if bad else []
    for (i, r), nr in zip(bad, nrecs):
        print(json.dumps({"i": i, "ptx": r.detail, "ptx_err": r.max_rel_err, "ptx_info": r.info,
                          "nvrtc": nr.status, "nvrtc_detail": nr.detail, "nvrtc_err": nr.max_rel_err,
                          "history": history_to_json(progs[i].history)}, default=str), flush=True)
    print(json.dumps({"task": task, "k": k, "rejected": len(bad)}))
    measure._shutdown()


if __name__ == "__main__":
    main()
