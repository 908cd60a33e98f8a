# half-warp rows A/B: parity tests of the direct kernel, then the probe with and without half-warp rows
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_spmm_exact.py -m gpu -q -x -k "direct" > gpurun_out/r2_gpu17.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gpu17.log
BS_DIRECT_HALF=0 timeout 300 python tools/direct_probe.py > gpurun_out/r2_direct17_nohalf.jsonl 2>&1
timeout 300 python tools/direct_probe.py > gpurun_out/r2_direct17_half.jsonl 2>&1
head -2 gpurun_out/r2_direct17_*.jsonl
