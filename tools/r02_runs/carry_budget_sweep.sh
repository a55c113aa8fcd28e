python -m paper_2006_06762_b200.build >/dev/null 2>&1
for cr in 4 8 16; do
  LT_CARRY_REGS=$cr timeout 300 python tools/best_found.py RC,G10 > gpurun_out/c6_best_cr$cr.log 2>&1
done
LT_CARRY_REGS=8 timeout 600 python tools/template_bench.py 96 --configs RC,TBG --out gpurun_out/c6_tb_cr8.jsonl > gpurun_out/c6_tb_cr8.log 2>&1
