mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_lstm.py -m gpu -q -x -k "direct or lstm" > gpurun_out/r2_gpu44.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_gpu44.log
for i in 1 2; do for f in 0 1; do BS_DIRECT_XPF=$f timeout 300 python tools/direct_probe.py | sed "s/^/xpf=$f /" >> gpurun_out/r2_direct44.txt 2>&1; done; done
cat gpurun_out/r2_direct44.txt | cut -c1-90
