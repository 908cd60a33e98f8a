mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_parity.py tests/test_gpu_conv.py -m gpu -q -x -k "spmm or sp24 or k6 or k5 or conv" > gpurun_out/r2_gpu39.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_gpu39.log
for c in "512 4608 32 3 784" "4096 2048 32 4 64"; do timeout 120 python tools/k6_trace_probe.py $c >> gpurun_out/r2_k6_trace39.txt 2>&1; done
cat gpurun_out/r2_k6_trace39.txt
timeout 600 python tools/tc_probe.py k6_fc6 k6_ctc_ih k6_conv3_3 k6_conv4_2 sp24_ctc_ih > gpurun_out/r2_tc39.txt 2>&1; cat gpurun_out/r2_tc39.txt | cut -c1-120
