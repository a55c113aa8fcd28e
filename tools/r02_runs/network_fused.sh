# whole-network ResNet-50 b16: unfused conv tasks and the conv+BN+ReLU fusion variant, 120 units each
python -m paper_2006_06762_b200.build >/dev/null 2>&1
timeout 900 python tools/tune_network.py 120 0 --gpu-sampler --gpu-rules > gpurun_out/c13_network_conv.log 2>&1
cp gpurun_out/tune_network.json gpurun_out/c13_network_conv.json
timeout 900 python tools/tune_network.py 120 0 --gpu-sampler --gpu-rules --fused > gpurun_out/c13_network_fused.log 2>&1
cp gpurun_out/tune_network.json gpurun_out/c13_network_fused.json
