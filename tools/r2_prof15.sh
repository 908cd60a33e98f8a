python -m pytest tests/test_gpu_lstm.py tests/test_gpu_spmm_exact.py -m gpu -q > gpurun_out/r2_gpu15.log 2>&1
python -c "
import sys; sys.path.insert(0,'.')
import bench, json, torch
class A: block=32; dtype='f16'
import paper_1811_00206_b200 as bs
l2=torch.cuda.get_device_properties(0).L2_cache_size
print(json.dumps(bench.lstm_rows(A(), bs, l2)))
" > gpurun_out/r2_lstm15.json 2>&1
python tools/direct_probe.py > gpurun_out/r2_direct15.jsonl 2>&1
for mc in 3 9 24 72; do BS_SPLITK_MIN_CHUNKS=$mc python tools/spmm_probe.py conv4_2 conv3_3 | sed "s/^/mc=$mc /" >> gpurun_out/r2_k6_split.txt 2>&1; done
