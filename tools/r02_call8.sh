# final round-2 evidence on the current code: GPU tests, smoke, bench, launch list, ncu of the best-found programs
python -m paper_2006_06762_b200.build >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c8_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c8_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c8_smoke.log 2>&1
timeout 700 python bench.py > gpurun_out/c8_bench.json 2> gpurun_out/c8_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all -c 4000 --csv \
    --log-file gpurun_out/c8_launches.csv python bench.py --steps 1 --warmup 1 --no-scoring --no-cpu \
    --sub-configs "" > gpurun_out/c8_bench_under_ncu.log 2>&1
for c in RC CL G10 TBG; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -c 4 \
      -o gpurun_out/c8_best_$c -f python tools/profile_tuned.py $c > gpurun_out/c8_best_$c.log 2>&1
done
timeout 600 ncu --set full --clock-control none --nvtx --nvtx-include "profile/" -c 3 -o gpurun_out/c8_scoring -f \
    python tools/profile_scoring.py 1 > /dev/null 2>&1
python tools/profile_scoring.py > gpurun_out/c8_scoring_time.log 2>&1
# shared-load lookahead A/B on the best-found programs (default 64)
for la in 16 32 128; do LT_LOOKAHEAD=$la timeout 300 python tools/best_found.py RC,G10,CL,TBG > gpurun_out/c8_la$la.log 2>&1; done
timeout 300 python tools/best_found.py RC,G10,CL,TBG > gpurun_out/c8_la64.log 2>&1
