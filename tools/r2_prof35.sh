mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lstm.py tests/test_gpu_spmm_exact.py -m gpu -q -x -k "lstm or direct" > gpurun_out/r2_gpu35.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gpu35.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench, json, torch
class A: block=32; dtype='f16'
import paper_1811_00206_b200 as bs
l2=torch.cuda.get_device_properties(0).L2_cache_size
print(json.dumps(bench.lstm_rows(A(), bs, l2)))
" > gpurun_out/r2_lstm35.json 2>&1
cat gpurun_out/r2_lstm35.json | tail -1
timeout 300 python tools/direct_probe.py > gpurun_out/r2_direct35.jsonl 2>&1; cat gpurun_out/r2_direct35.jsonl | cut -c1-80
