set -x
python -m paper_2006_06762_b200.build >/dev/null 2>&1
timeout 300 python tools/pipeline_probe.py RC 256 --offset 384 --out gpurun_out/probe_rc.jsonl > gpurun_out/probe_rc.log 2>&1
timeout 300 python tools/pipeline_probe.py G10 256 --offset 384 --out gpurun_out/probe_g10.jsonl > gpurun_out/probe_g10.log 2>&1
for c in RC CL G10 TBG; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -c 4 \
      -o gpurun_out/G_best_$c -f python tools/profile_tuned.py $c > gpurun_out/G_best_$c.log 2>&1
done
ls -la gpurun_out
