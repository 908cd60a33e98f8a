# Tensor-core grid order A/B (BS_TC_ORDER 0 = round-1 order, 1 = column tiles of a row tile adjacent) + parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_parity.py -m gpu -q -x -k "spmm or sp24 or k6 or k5" > gpurun_out/r2_gpu19.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_gpu19.log
for o in 0 1; do BS_TC_ORDER=$o timeout 600 python tools/tc_probe.py >> gpurun_out/r2_tc19.jsonl 2>&1; done
cat gpurun_out/r2_tc19.jsonl
