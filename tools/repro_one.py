"""Measure one State given as (dag key in tests/golden/corpus.json, history JSON file)."""
import json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2006_06762_b200 import measure
from paper_2006_06762_b200.state import ComputeDAG, history_from_json, replay
G = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")
dags = json.load(open(os.path.join(G, "corpus.json")))["dags"]
dag = ComputeDAG.from_json(dags[sys.argv[1]])
p = replay(dag, history_from_json(json.load(open(sys.argv[2]))))
r = measure.configure(device=0, cache_dir="")
print(r.measure_programs([p]))
