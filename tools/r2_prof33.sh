mkdir -p gpurun_out
for thr in 2048 1000000; do BS_DIRECT_ROW_BYTES=$thr timeout 300 python tools/direct_probe.py | sed "s/^/thr=$thr /" >> gpurun_out/r2_direct33.txt 2>&1; done
cat gpurun_out/r2_direct33.txt | cut -c1-100
