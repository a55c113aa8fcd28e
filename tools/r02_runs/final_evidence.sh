# final round-2 evidence: ncu of the best-found programs (+ their DRAM bytes into profiles/traffic.json,
# read by bench.py's roofline.traffic), the bench line, the bench's launch list, features-kernel occupancy A/B
python -m paper_2006_06762_b200.build >/dev/null 2>&1
CFGS=${CFGS:-"RC CL G10 TBG"}
for c in $CFGS; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -c 4 \
      -o gpurun_out/c10_best_$c -f python tools/profile_tuned.py $c > gpurun_out/c10_best_$c.log 2>&1
done
python - <<'PY' > gpurun_out/c10_best_per_operator_ncu.txt
import hashlib, json, os, subprocess, sys
sys.path.insert(0, ".")
import bench
from paper_2006_06762_b200.state import replay
from paper_2006_06762_b200.ptxgen import lower_ptx
print("# ncu --set full --clock-control none --import-source on: the best-found program per operator "
      "(profiles/r02_tuned_best.json; tools/profile_tuned.py CFG relaunches its kernels 3x in NVTX range 'profile'; "
      "first launch summarised).  The 'us' in each header is the runner's measurement inside the profiled process "
      "(not a bench number).")
for c in os.environ.get("CFGS", "RC CL G10 TBG").split():
    dag, hist, src = bench.best_found_programs()[c]
    key = hashlib.sha1(lower_ptx(replay(dag, hist)).source.encode()).hexdigest()
    head = next((l for l in open(f"gpurun_out/c10_best_{c}.log") if l.startswith("{")), "{}")[:160]
    print()
    sys.stdout.flush()
    subprocess.run([sys.executable, "tools/ncu_summary.py", f"gpurun_out/c10_best_{c}.ncu-rep", "--header",
                    f"{c} ({src}): {head}", "--traffic-key", key, "--config", c], check=False)
PY
# scoring kernels on the bench's own population: DRAM bytes per launch -> traffic.json "scoring:<kernel>"
timeout 600 ncu --set full --clock-control none --nvtx --nvtx-include "profile/" -c 3 -o gpurun_out/c10_scoring -f \
    python tools/profile_scoring.py 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/c10_scoring.ncu-rep --header "population scoring, 65,536 programs (tools/profile_scoring.py)" \
    > gpurun_out/c10_scoring_ncu.txt 2>&1
python - <<'PY'
import csv, io, json, subprocess
out = subprocess.run(["ncu", "-i", "gpurun_out/c10_scoring.ncu-rep", "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out[out.find('"'):])))
h, units, body = rows[0], rows[1], rows[2:]
ix = {k: i for i, k in enumerate(h)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
data = json.load(open("profiles/traffic.json"))
for r in body:
    name = r[ix["Kernel Name"]].split("(")[0]
    key = f"scoring:{name}"
    if key in data and data[key].get("round") == "r02-final":
        continue
    tot = sum(float(r[ix[m]].replace(",", "")) * scale.get(units[ix[m]], 1)
              for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    data[key] = {"config": "scoring", "dram_bytes_per_launch": tot, "round": "r02-final",
                 "source": "ncu --set full --clock-control none, tools/profile_scoring.py 1 (65,536 programs)"}
json.dump(data, open("profiles/traffic.json", "w"), indent=1)
PY
cp profiles/traffic.json gpurun_out/c10_traffic.json
timeout 700 python bench.py > gpurun_out/c10_bench.json 2> gpurun_out/c10_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all -c 4000 --csv \
    --log-file gpurun_out/c10_launches.csv python bench.py --steps 1 --warmup 1 --no-scoring --no-cpu \
    --sub-configs "" > gpurun_out/c10_bench_under_ncu.log 2>&1
for b in 0 2 3 4 6; do LT_FEAT_BLOCKS_PER_SM=$b timeout 300 python tools/profile_scoring.py 3 > gpurun_out/c10_feat_bps$b.log 2>&1; done
