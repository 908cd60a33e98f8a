mkdir -p gpurun_out
for mc in 3 12 18 36; do
BS_SPLITK_MIN_CHUNKS=$mc timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench, json, torch
class A: block=32; dtype='f16'
import paper_1811_00206_b200 as bs
l2=torch.cuda.get_device_properties(0).L2_cache_size
d=bench.conv_rows(A(), bs, l2)
print(json.dumps([(r['layer'], r['ours_us']) for r in d['conv']]))
" | sed "s/^/mc=$mc /" >> gpurun_out/r2_conv59.txt 2>&1
done
cat gpurun_out/r2_conv59.txt
