# whole-network ResNet-50 b16, conv+BN+ReLU fusion variant, 480 units (the fused DAGs need more units per task)
python -m paper_2006_06762_b200.build >/dev/null 2>&1
timeout 1500 python tools/tune_network.py 480 0 --gpu-sampler --gpu-rules --fused > gpurun_out/c14_network_fused_480.log 2>&1
