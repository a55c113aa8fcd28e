"""Debug helper: run one stream candidate (CFG:i) with the PTX and the NVRTC
backend and report where the outputs differ (decoded output coordinates)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from bench import load_stream
from paper_2006_06762_b200 import measure
from paper_2006_06762_b200.state import replay
cfg, i = sys.argv[1].split(":")
dag, st = load_stream(cfg)
p = replay(dag, st[int(i)])
outs = {}
for be in ("nvrtc", "ptx"):
    r = measure.RunnerCore(device=0, cache_dir="", backend=be)
    (rec,) = r.measure_programs([p])
    ctx = r.context(dag, 0)
    name = dag.outputs[0]
    shape = dag.node(name).shape
    outs[be] = ctx.download(name, int(np.prod(shape))).reshape(shape)
    print(be, rec.status, rec.detail, rec.cost_us, flush=True)
    measure._shutdown()
a, b = outs["nvrtc"], outs["ptx"]
bad = ~np.isclose(a, b, rtol=1e-4) | np.isnan(b)
print("mismatch", int(bad.sum()), "of", bad.size, "nan", int(np.isnan(b).sum()))
idx = np.argwhere(bad)
for d in range(idx.shape[1]):
    print("dim", d, "bad coords:", np.unique(idx[:, d])[:40])
print(idx[:20].tolist())
