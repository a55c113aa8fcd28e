#!/bin/bash
# Round-2 ncu evidence, run on the GPU box:  bash tools/r02_runs/profile.sh
# (1) launch list of a short bench run: the candidates run in the measuring child
#     process, hence --target-processes all (a number printed under ncu is never a bench value);
# (2) one full capture per best-found program (profiles/r02_tuned_best.json);
# (3) the scoring kernels (default thread-per-statement features + tree-per-warp predict).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all -c 4000 --csv \
    --log-file gpurun_out/F_launches.csv python bench.py --steps 1 --warmup 1 --no-scoring --no-cpu \
    --sub-configs "" > gpurun_out/F_bench_under_ncu.log 2>&1
for c in RC CL G10 TBG; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -c 4 \
      -o gpurun_out/F_best_$c -f python tools/profile_tuned.py $c > gpurun_out/F_best_$c.log 2>&1
done
timeout 600 ncu --set full --clock-control none --nvtx --nvtx-include "profile/" -c 3 -o gpurun_out/F_scoring -f \
    python tools/profile_scoring.py 1 > /dev/null 2>&1
python tools/profile_scoring.py > gpurun_out/F_scoring_time.log 2>&1
du -sh gpurun_out
