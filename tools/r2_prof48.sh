mkdir -p gpurun_out
for i in 1 2; do for mc in 6 4 3; do BS_SPLITK_MIN_CHUNKS=$mc timeout 300 python tools/tc_probe.py sp24_ctc_ih | sed "s/^/mc=$mc /" >> gpurun_out/r2_tc48.txt 2>&1; done; done
cat gpurun_out/r2_tc48.txt | cut -c1-100
