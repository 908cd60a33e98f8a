python -m pytest tests/test_gpu_lstm.py tests/test_gpu_spmm_exact.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/r2_gpu14.log 2>&1
python -c "
import sys; sys.path.insert(0,'.')
import bench, json, torch
class A: block=32; dtype='f16'
import paper_1811_00206_b200 as bs
l2=torch.cuda.get_device_properties(0).L2_cache_size
print(json.dumps(bench.lstm_rows(A(), bs, l2)))
print(json.dumps(bench.epilogue_rows(A(), bs, l2)))
" > gpurun_out/r2_lstm14.json 2>&1
python tools/direct_probe.py > gpurun_out/r2_direct14.jsonl 2>&1
