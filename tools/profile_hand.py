"""Run one hand-built State (tools/hand_states.py index) 3x inside NVTX range "profile" for ncu."""
import ctypes, hashlib, os, sys
ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from hand_states import states
from paper_2006_06762_b200 import measure, runtime as rt
name, p = states()[int(sys.argv[1])]
r = measure.RunnerCore(device=0, cache_dir="")
(rec,) = r.measure_programs([p])
print(name, rec.status, rec.cost_us, flush=True)
lo = r.lower(p)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
open(os.path.join(ROOT, "gpurun_out", f"hand{sys.argv[1]}.ptx"), "w").write(lo.source)
funcs = r.load(hashlib.sha1(lo.source.encode()).hexdigest(), b"", [k.entry for k in lo.kernels])
ctx = r.context(p.dag, 0)
L = ctx._launches(lo, funcs)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profile")
for _ in range(3):
    rt.check(r.lib.lt_task_run(ctx.task, ctypes.addressof(L), len(lo.kernels)), "run")
torch.cuda.nvtx.range_pop()
measure._shutdown()
