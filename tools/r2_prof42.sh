mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_conv.py -m gpu -q -x > gpurun_out/r2_gpu42.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_gpu42.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench, json, torch
class A: block=32; dtype='f16'
import paper_1811_00206_b200 as bs
l2=torch.cuda.get_device_properties(0).L2_cache_size
print(json.dumps(bench.conv_rows(A(), bs, l2)))
" > gpurun_out/r2_conv42.json 2>&1
cat gpurun_out/r2_conv42.json | tail -1
