mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm24_pair -s 2 -c 1 -o gpurun_out/r2_k5_pair_n256 python tools/k5_once.py 16384 16384 256 > gpurun_out/r2_k5_pair_n256.log 2>&1; echo "ncu rc=$?"
