mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_conv.py -m gpu -q -x > gpurun_out/r2_gpu56.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2_gpu56.log
