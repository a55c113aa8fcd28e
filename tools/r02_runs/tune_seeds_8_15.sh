# more seeds of the reference's tune with the B200 path (BASELINE trial counts), for the best-found program per operator
python -m paper_2006_06762_b200.build >/dev/null 2>&1
for s in 8 9 10 11 12 13 14 15; do timeout 400 python tools/tune_gpu.py RC 62 $s --gpu-sampler --gpu-rules > gpurun_out/c7_RC_$s.log 2>&1; done
for s in 8 9 10 11 12 13 14 15; do timeout 300 python tools/tune_gpu.py G10 62 $s --gpu-sampler --gpu-rules > gpurun_out/c7_G10_$s.log 2>&1; done
for s in 8 9 10 11 12 13 14 15; do timeout 300 python tools/tune_gpu.py TBG 62 $s --gpu-sampler --gpu-rules > gpurun_out/c7_TBG_$s.log 2>&1; done
for s in 8 9 10 11; do timeout 700 python tools/tune_gpu.py CL 125 $s --gpu-sampler --gpu-rules > gpurun_out/c7_CL_$s.log 2>&1; done
