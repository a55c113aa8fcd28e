# RC seeds 48-67, merged on the box; if the best RC program changed, its ncu DRAM bytes go into traffic.json
python -m paper_2006_06762_b200.build >/dev/null 2>&1
for s in $(seq 48 67); do timeout 400 python tools/tune_gpu.py RC 62 $s --gpu-sampler --gpu-rules > gpurun_out/c20_RC_$s.log 2>&1; done
python tools/merge_tuned_best.py > gpurun_out/c20_merge.log 2>&1
cp profiles/r02_tuned_best.json gpurun_out/c20_tuned_best.json
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -c 4 \
    -o gpurun_out/c20_best_RC -f python tools/profile_tuned.py RC > gpurun_out/c20_best_RC.log 2>&1
python - <<'PY' > gpurun_out/c20_best_RC_ncu.txt
import hashlib, subprocess, sys
sys.path.insert(0, ".")
import bench
from paper_2006_06762_b200.state import replay
from paper_2006_06762_b200.ptxgen import lower_ptx
dag, hist, src = bench.best_found_programs()["RC"]
key = hashlib.sha1(lower_ptx(replay(dag, hist)).source.encode()).hexdigest()
sys.stdout.flush()
subprocess.run([sys.executable, "tools/ncu_summary.py", "gpurun_out/c20_best_RC.ncu-rep", "--header", f"RC ({src})",
                "--traffic-key", key, "--config", "RC"], check=False)
PY
cp profiles/traffic.json gpurun_out/c20_traffic.json
