mkdir -p gpurun_out
for ab in 0 1 2 3; do BS_K6_ABL=$ab timeout 600 python tools/tc_probe.py k6_fc6 k6_ctc_ih k6_conv4_2 | sed "s/^/abl=$ab /" >> gpurun_out/r2_tc30.txt 2>&1; done
cat gpurun_out/r2_tc30.txt | cut -c1-110
