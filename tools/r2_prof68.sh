timeout 600 python -m pytest tests/test_gpu_conv.py -m gpu -q -x -k errors > gpurun_out/r2_gpu68.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/r2_gpu68.log
