"""Measure stream candidates CFG:i[,j...] under both backends (debug helper)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from bench import load_stream
from paper_2006_06762_b200 import measure
from paper_2006_06762_b200.state import replay
cfg, idx = sys.argv[1].split(":")
dag, st = load_stream(cfg)
progs = [replay(dag, st[int(i)]) for i in idx.split(",")]
r = measure.configure(device=0, cache_dir="", backend=sys.argv[2] if len(sys.argv) > 2 else "ptx")
for rec in r.measure_programs(progs):
    print(rec.status, rec.detail, rec.cost_us, rec.max_rel_err, flush=True)
measure._shutdown()
