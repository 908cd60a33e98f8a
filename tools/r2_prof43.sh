mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_parity.py tests/test_gpu_conv.py -m gpu -q -x -k "spmm or sp24 or k6 or k5 or conv" > gpurun_out/r2_gpu43.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_gpu43.log
for f in 0 1; do BS_TC_FILL=$f timeout 600 python tools/tc_probe.py k6_fc6 k6_ctc_ih k6_conv3_3 k6_conv4_2 sp24_ctc_ih sp24_16384 | sed "s/^/fill=$f /" >> gpurun_out/r2_tc43.txt 2>&1; done
cat gpurun_out/r2_tc43.txt | cut -c1-110
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench, json, torch
class A: block=32; dtype='f16'
import paper_1811_00206_b200 as bs
l2=torch.cuda.get_device_properties(0).L2_cache_size
print(json.dumps(bench.conv_rows(A(), bs, l2)))
" > gpurun_out/r2_conv43.json 2>&1
cat gpurun_out/r2_conv43.json | tail -1
