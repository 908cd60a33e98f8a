python -m pytest tests/test_gpu_parity.py tests/test_gpu_patterns.py tests/test_gpu_spmm_exact.py tests/test_gpu_conv.py -m gpu -q -x > gpurun_out/r2_gpu3.log 2>&1
python tools/producers_probe.py > gpurun_out/r2_prod2.json 2>&1
python tools/spmm_probe.py > gpurun_out/r2_spmm3.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prune_thread -s 1 -c 1 -o gpurun_out/r2_prune3 python tools/producers_probe.py 16384 65536 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:spmm_tc -s 2 -c 1 -o gpurun_out/r2_k6_fc6 python tools/spmm_probe.py fc6 > /dev/null 2>&1
