mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_lib_exports.py -m "gpu or not gpu" -q -x > gpurun_out/r2_gpu61.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gpu61.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench, json, torch
class A: block=32; dtype='f16'
import paper_1811_00206_b200 as bs
l2=torch.cuda.get_device_properties(0).L2_cache_size
d=bench.conv_rows(A(), bs, l2)
print(json.dumps(d))
for r in d['conv']: print(r['layer'], r['ours_us'], r.get('ours_bias_relu_us'), r['cudnn_dense_us'], r.get('cudnn_bias_relu_us'))
" > gpurun_out/r2_conv61.txt 2>&1; tail -4 gpurun_out/r2_conv61.txt
