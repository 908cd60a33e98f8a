mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_parity.py tests/test_gpu_conv.py -m gpu -q -x -k "spmm or k6 or conv or small or random" > gpurun_out/r2_gpu60.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_gpu55.log

for i in 1 2; do
BS_LIB=$PWD/paper_1811_00206_b200/libbs_prev.so timeout 300 python tools/tc_probe.py k6_fc6 k6_ctc_ih k6_conv3_3 k6_conv4_2 | sed "s/^/prev /" >> gpurun_out/r2_tc60.txt 2>&1
timeout 300 python tools/tc_probe.py k6_fc6 k6_ctc_ih k6_conv3_3 k6_conv4_2 | sed "s/^/new /" >> gpurun_out/r2_tc60.txt 2>&1
done
cat gpurun_out/r2_tc60.txt | cut -c1-100
