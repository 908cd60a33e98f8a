mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:spmv_rows_kernel -s 3 -c 1 -o gpurun_out/r2_ptb_direct python tools/ptb_once.py > gpurun_out/r2_ptb_ncu.log 2>&1; echo "ncu rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:spmv_rows_kernel -s 3 -c 1 -o gpurun_out/r2_fc7_direct python tools/ptb_once.py 4096 4096 0.9 > gpurun_out/r2_fc7_ncu.log 2>&1; echo "ncu rc=$?"
