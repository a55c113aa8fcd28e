# device packing + local-memory high-water flag: per-candidate breakdown A/B
python -m paper_2006_06762_b200.build >/dev/null 2>&1
timeout 300 python -m pytest tests/test_measure_gpu.py -q -k "packing or staged or edge" > gpurun_out/c3_tests.log 2>&1
for v in 0 1; do
  LT_LMEM_SHRINK=$v timeout 300 python tools/pipeline_probe.py RC 256 --offset 384 --out gpurun_out/c3_probe_rc_shrink$v.jsonl > gpurun_out/c3_probe_rc_shrink$v.log 2>&1
done
timeout 300 python tools/pipeline_probe.py G10 256 --offset 384 --out gpurun_out/c3_probe_g10.jsonl > gpurun_out/c3_probe_g10.log 2>&1
