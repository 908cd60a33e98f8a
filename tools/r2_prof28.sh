mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_exact.py -m gpu -q -x -k "sp24 or k5" > gpurun_out/r2_gpu28.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_gpu28.log
for st in 4 8; do BS_K5_STAGES=$st timeout 600 python tools/tc_probe.py sp24_16384 sp24_ctc_ih | sed "s/^/st=$st /" >> gpurun_out/r2_tc28.txt 2>&1; done
cat gpurun_out/r2_tc28.txt
