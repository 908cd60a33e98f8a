mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_patterns.py -m gpu -q -x -k "prune or rank or random or mask" > gpurun_out/r2_gpu50.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_gpu50.log
for i in 1 2; do
BS_LIB=$PWD/paper_1811_00206_b200/libbs_old.so timeout 300 python tools/producers_probe.py 65536 65536 3 16 | sed "s/^/old /" >> gpurun_out/r2_prod50.txt 2>&1
timeout 300 python tools/producers_probe.py 65536 65536 3 16 | sed "s/^/new /" >> gpurun_out/r2_prod50.txt 2>&1
done
cat gpurun_out/r2_prod50.txt | cut -c1-300
