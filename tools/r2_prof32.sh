mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_parity.py -m gpu -q -x -k "direct or spmv" > gpurun_out/r2_gpu32.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_gpu32.log
for i in 1 2; do
BS_LIB=$PWD/paper_1811_00206_b200/libbs_old.so timeout 300 python tools/direct_probe.py | sed "s/^/old$i /" >> gpurun_out/r2_direct32.txt 2>&1
timeout 300 python tools/direct_probe.py | sed "s/^/new$i /" >> gpurun_out/r2_direct32.txt 2>&1
done
cat gpurun_out/r2_direct32.txt | cut -c1-100
