python -m pytest tests/test_gpu_parity.py tests/test_gpu_patterns.py tests/test_gpu_spmm_exact.py -m gpu -q -x > gpurun_out/r2_gpu10.log 2>&1
python tools/producers_probe.py 65536 65536 1 2 3 4 8 16 > gpurun_out/r2_prod10.json 2>&1
