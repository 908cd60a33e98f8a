timeout 300 ncu --set full --clock-control none --import-source on -k regex:spmm_tc -s 3 -c 1 -o gpurun_out/r2_k6_conv42 python tools/spmm_probe.py conv4_2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:spmm24 -s 3 -c 1 -o gpurun_out/r2_k5_ctc16 python tools/sp24_small_probe.py 16 > /dev/null 2>&1
bash tools/gpu_profile.sh r2a > gpurun_out/r2_gpuprofile.log 2>&1
