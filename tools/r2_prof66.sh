mkdir -p gpurun_out
timeout 600 python tools/spmm_probe.py 16384sq CTC_ih > gpurun_out/r2_k4_66.txt 2>&1; cat gpurun_out/r2_k4_66.txt
