# health of the current code on the GPU + bench, and a shared-load lookahead A/B on the best-found programs
python -m paper_2006_06762_b200.build >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c8_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c8_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c8_smoke.log 2>&1
timeout 700 python bench.py > gpurun_out/c8_bench.json 2> gpurun_out/c8_bench.err
for la in 16 32 64 128; do LT_LOOKAHEAD=$la timeout 300 python tools/best_found.py RC,G10,CL,TBG > gpurun_out/c8_la$la.log 2>&1; done
