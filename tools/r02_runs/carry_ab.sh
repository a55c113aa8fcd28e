# template A/B: carried-operand pipelining of rolled reduction loops (LT_PTX_OFF=carry disables)
python -m paper_2006_06762_b200.build >/dev/null 2>&1
for off in carry none; do
  LT_PTX_OFF=$off timeout 300 python tools/best_found.py RC,CL,G10,TBG > gpurun_out/c5_best_$off.log 2>&1
  LT_PTX_OFF=$off timeout 600 python tools/template_bench.py 96 --out gpurun_out/c5_tb_$off.jsonl > gpurun_out/c5_tb_$off.log 2>&1
done
