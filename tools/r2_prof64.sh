mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_spmm_exact.py -m gpu -q -x -k "conv or sp24 or k5 or fused" > gpurun_out/r2_gpu64.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2_gpu64.log
