# more seeds where the seed spread is widest (RC, CL)
python -m paper_2006_06762_b200.build >/dev/null 2>&1
for s in 16 17 18 19 20 21 22 23 24 25 26 27; do timeout 400 python tools/tune_gpu.py RC 62 $s --gpu-sampler --gpu-rules > gpurun_out/c9_RC_$s.log 2>&1; done
for s in 12 13 14 15; do timeout 700 python tools/tune_gpu.py CL 125 $s --gpu-sampler --gpu-rules > gpurun_out/c9_CL_$s.log 2>&1; done
