mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_conv.py tests/test_lib_exports.py -m "gpu or not gpu" -q -x -k "fused or conv or export or k6" > gpurun_out/r2_gpu62.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gpu62.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench, json, torch
class A: block=32; dtype='f16'
import paper_1811_00206_b200 as bs
l2=torch.cuda.get_device_properties(0).L2_cache_size
print(json.dumps(bench.fc_batch_rows(A(), bs, l2)))
" > gpurun_out/r2_fc62.txt 2>&1; tail -2 gpurun_out/r2_fc62.txt
