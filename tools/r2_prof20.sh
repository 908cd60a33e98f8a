# K5 RT = 2 (two row tiles per CTA): parity, then A/B RT = 1 vs auto on the K5 shapes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_parity.py -m gpu -q -x -k "spmm or sp24 or k6 or k5" > gpurun_out/r2_gpu20.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gpu20.log
for rt in 1 0; do BS_K5_RT=$rt timeout 600 python tools/tc_probe.py sp24_16384 sp24_ctc_ih | sed "s/^/rt=$rt /" >> gpurun_out/r2_tc20.txt 2>&1; done
timeout 600 python tools/tc_probe.py k6_fc6 k6_16384_90 | sed "s/^/k6 /" >> gpurun_out/r2_tc20.txt 2>&1
cat gpurun_out/r2_tc20.txt
