mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_parity.py tests/test_gpu_conv.py -m gpu -q -x -k "spmm or sp24 or k6 or k5 or conv" > gpurun_out/r2_gpu47.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_gpu47.log
for n in 16 256; do timeout 120 python tools/k6_trace_probe.py --k5 4096 2048 4 2 $n >> gpurun_out/r2_k5_trace47.txt 2>&1; done
cat gpurun_out/r2_k5_trace47.txt
timeout 600 python tools/tc_probe.py sp24_ctc_ih k6_ctc_ih k6_conv3_3 k6_conv4_2 > gpurun_out/r2_tc47.txt 2>&1; cat gpurun_out/r2_tc47.txt | cut -c1-110
