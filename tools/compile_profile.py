"""Where ptxas time goes: lower a slice of a golden stream on the host, assemble
every kernel module with the runner's ptxas options (the `ptxas` binary, same
flags as the in-process nvPTXCompiler), and print per-kernel seconds next to the
kernel's template facts.  CPU only.

    python tools/compile_profile.py RC 96 224 [--jobs 8]
"""
import argparse
import hashlib
import json
import os
import subprocess
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("lo", type=int)
    ap.add_argument("hi", type=int)
    ap.add_argument("--jobs", type=int, default=os.cpu_count())
    ap.add_argument("--opt", default="-O3 --allow-expensive-optimizations=false")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import bench
    from paper_2006_06762_b200.measure import _modules_of, PTX_SAFE_OPTS
    from paper_2006_06762_b200.ptxgen import Unsupported, lower_ptx
    from paper_2006_06762_b200.state import replay, validate
    dag, stream = bench.load_stream(a.cfg)
    mods = {}
    lower_s = []
    for i in range(a.lo, a.hi):
        p = replay(dag, stream[i])
        t0 = time.perf_counter()
        if validate(p):
            continue
        try:
            lo = lower_ptx(p)
        except Exception:
            continue
        lower_s.append(time.perf_counter() - t0)
        for (ents, text, opts), k in zip(_modules_of(lo), lo.kernels):
            key = hashlib.sha1((opts or "").encode() + text.encode()).hexdigest()
            mods.setdefault(key, (i, text, opts, k.info))
    os.makedirs("/tmp/ptx", exist_ok=True)

    def run(item):
        key, (i, text, opts, info) = item
        path = f"/tmp/ptx/{key}.ptx"
        open(path, "w").write(text)
        flags = ["-O1"] if opts == PTX_SAFE_OPTS else a.opt.split()
        t0 = time.perf_counter()
        r = subprocess.run(["ptxas", "-arch=sm_100a", *flags, path, "-o", path + ".cubin"], capture_output=True)
        return key, i, time.perf_counter() - t0, len(text), info, r.returncode
    with ThreadPoolExecutor(a.jobs) as ex:
        rows = list(ex.map(run, mods.items()))
    rows.sort(key=lambda r: -r[2])
    tot = sum(r[2] for r in rows)
    print(f"{len(rows)} modules from {a.hi - a.lo} States; ptxas total {tot:.2f} s, mean {tot / len(rows):.3f}; "
          f"lower mean {sum(lower_s) / max(1, len(lower_s)) * 1000:.1f} ms")
    for key, i, s, n, info, rc in rows[:25]:
        print(f"{s:6.3f}s  #{i:<4} {n // 1024:5d} KB  {info.get('template')} thr={info.get('threads')} acc={info.get('acc')} "
              f"unr={info.get('unrolled')} db={info.get('double_buffered')} async={info.get('async_copy')} "
              f"regs_in={info.get('acc_in_regs')} ptxas={info.get('ptxas_opt') or info.get('ptxas')} stages={info.get('n_stage')}")
    if a.out:
        with open(a.out, "w") as fh:
            for key, i, s, n, info, rc in rows:
                fh.write(json.dumps({"i": i, "s": s, "ptx_bytes": n, "rc": rc,
                                     **{k: v for k, v in info.items() if isinstance(v, (int, float, str, bool))}}) + "\n")


if __name__ == "__main__":
    main()
