mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_conv.py tests/test_gpu_parity.py -m gpu -q -x -k "fused or conv or sp24 or k5 or k6 or spmm" > gpurun_out/r2_gpu63.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gpu63.log
