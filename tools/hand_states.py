"""Hand-built SSSRRSRS States (good GPU tilings) to calibrate the tiled template.

  python tools/hand_states.py        measure them on cuda:0 and print TFLOP/s

Each State is an ordinary rewrite history (Split x axes, Reorder, SetPragma) of
the kind the sketch/annotation passes produce, so it lowers through exactly the
same path as searched candidates.
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

from paper_2006_06762_b200.state import Reorder, SetPragma, Split, apply_step, config_dag, naive_program  # noqa: E402


def tiled(dag, stage: str, space: dict, red: dict, unroll: int = 512):
    """space/red: axis -> inner factors (S1..S4) / (R1, R2), outer inferred."""
    p = naive_program(dag)
    s = p.stage(stage)
    for a, _ in s.space:
        p = apply_step(p, Split(stage, a, tuple(space[a])))
    for r, _ in s.reduce:
        p = apply_step(p, Split(stage, r, tuple(red[r])))
    sp = [a for a, _ in s.space]
    rd = [r for r, _ in s.reduce]
    order = []
    for lv in ("S0", "S1", "S2", "R0", "R1", "S3", "R2", "S4"):
        axes = sp if lv[0] == "S" else rd
        order += [f"{a}.{lv[1]}" for a in axes]
    p = apply_step(p, Reorder(stage, tuple(order)))
    return apply_step(p, SetPragma(stage, unroll))


def states():
    out = []
    g = config_dag("G10")
    # 128x128 block, 16x16 threads, 2x2 vthreads, 4x4 per vthread, k tile 8
    out.append(("G10 128x128/256thr/8x8", tiled(g, "C", {"i": (2, 16, 1, 4), "j": (2, 16, 1, 4)}, {"k": (1, 8)})))
    out.append(("G10 128x64/128thr/8x8", tiled(g, "C", {"i": (2, 16, 1, 4), "j": (2, 8, 1, 4)}, {"k": (1, 8)})))
    out.append(("G10 64x64/64thr/8x8", tiled(g, "C", {"i": (2, 8, 1, 4), "j": (2, 8, 1, 4)}, {"k": (1, 16)})))
    out.append(("G10 64x128/256thr/4x8", tiled(g, "C", {"i": (1, 16, 1, 4), "j": (2, 16, 1, 4)}, {"k": (1, 8)})))
    rc = config_dag("RC")
    # conv: n 16, h 56, w 56, co 64; reduce rh 3, rw 3, rc 64
    out.append(("RC 2x8x56 co64", tiled(rc, "C", {"cn": (1, 1, 1, 1), "ch": (1, 4, 1, 2), "cw": (2, 7, 1, 4),
                                                  "cc": (2, 8, 1, 4)},
                                        {"rh": (1, 3), "rw": (1, 3), "rc": (1, 8)})))
    out.append(("RC 4x8x28 co64", tiled(rc, "C", {"cn": (1, 1, 1, 1), "ch": (1, 4, 1, 1), "cw": (2, 7, 1, 2),
                                                  "cc": (2, 8, 1, 4)},
                                        {"rh": (1, 1), "rw": (1, 3), "rc": (1, 8)})))
    tbg = config_dag("TBG")
    # batched GEMM: 1 batch x 64x64 per block, 16x16 threads, 4x4 per thread, k tile 16
    out.append(("TBG 64x64/256thr/4x4", tiled(tbg, "C", {"b": (1, 1, 1, 1), "i": (1, 16, 1, 4), "j": (1, 16, 1, 4)},
                                              {"k": (1, 16)})))
    out.append(("TBG 128x64/256thr/8x4", tiled(tbg, "C", {"b": (1, 1, 1, 1), "i": (2, 16, 1, 4),
                                                          "j": (1, 16, 1, 4)}, {"k": (1, 8)})))
    return out


def main() -> None:
    from bench import FLOPS
    from paper_2006_06762_b200 import measure
    r = measure.configure(device=0, cache_dir="", backend=sys.argv[1] if len(sys.argv) > 1 else "ptx")
    for name, p in states():
        (rec,) = r.measure_programs([p])
        cfg = name.split()[0]
        tf = FLOPS[cfg] / (rec.cost_us * 1e-6) / 1e12 if rec.status == "valid" else None
        print(json.dumps({"state": name, "status": rec.status, "detail": rec.detail, "us": rec.cost_us,
                          "tflops": tf, "err": rec.max_rel_err,
                          "kernels": [{k: v for k, v in x.items() if k != "factors"} for x in rec.info.get("kernels", [])]}))
    measure._shutdown()


if __name__ == "__main__":
    main()
