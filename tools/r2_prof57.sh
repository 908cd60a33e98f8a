mkdir -p gpurun_out
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench, json, torch
class A: block=32; dtype='f16'
import paper_1811_00206_b200 as bs
l2=torch.cuda.get_device_properties(0).L2_cache_size
print(json.dumps(bench.conv_rows(A(), bs, l2)))
" > gpurun_out/r2_conv57.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/r2_conv57.json').read().strip().splitlines()[-1])
for r in d['conv']: print(r['layer'], r['path'], r['ours_us'], r['explicit_im2col_spmm_us'], r['im2col_us'], r['cudnn_dense_us'], r['speedup_vs_cudnn'])"
