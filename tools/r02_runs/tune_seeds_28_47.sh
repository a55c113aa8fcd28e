# RC seeds 28-47 (RC is the config whose seed spread keeps paying)
python -m paper_2006_06762_b200.build >/dev/null 2>&1
for s in $(seq 28 47); do timeout 400 python tools/tune_gpu.py RC 62 $s --gpu-sampler --gpu-rules > gpurun_out/c12_RC_$s.log 2>&1; done
