python -m pytest tests/test_gpu_spmm_exact.py -m gpu -q -x -k direct > gpurun_out/r2_gpu12.log 2>&1
BS_DIRECT_WAVES=1 python tools/direct_probe.py > gpurun_out/r2_direct5.jsonl 2>&1
BS_DIRECT_WAVES=2 python tools/direct_probe.py > gpurun_out/r2_direct5w2.jsonl 2>&1
