mkdir -p gpurun_out
for n in 16 64 256; do timeout 120 python tools/k6_trace_probe.py --k5 4096 2048 4 2 $n >> gpurun_out/r2_k5_trace.txt 2>&1; done
cat gpurun_out/r2_k5_trace.txt
