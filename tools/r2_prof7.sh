python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_parity.py tests/test_gpu_lstm.py -m gpu -q -x > gpurun_out/r2_gpu7.log 2>&1
python tools/direct_probe.py > gpurun_out/r2_direct2.jsonl 2>&1
