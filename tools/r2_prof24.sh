mkdir -p gpurun_out
BS_K5_PAIR=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm24_pair -s 2 -c 1 -o gpurun_out/r2_k5_pair_n128 python tools/k5_once.py 16384 16384 128 > gpurun_out/r2_k5_pair_ncu.log 2>&1; echo "ncu rc=$?"
BS_K5_PAIR=0 BS_K5_RT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm24_kernel -s 2 -c 1 -o gpurun_out/r2_k5_rt1_n128 python tools/k5_once.py 16384 16384 128 > gpurun_out/r2_k5_rt1_ncu.log 2>&1; echo "ncu rc=$?"
