mkdir -p gpurun_out
for c in "4096 25088 32 3 32" "4096 2048 32 4 64" "512 4608 32 3 784"; do timeout 120 python tools/k6_trace_probe.py $c >> gpurun_out/r2_k6_trace54.txt 2>&1; done
cat gpurun_out/r2_k6_trace54.txt
