mkdir -p gpurun_out
for cfg in "6 128" "4 256" "4 128" "6 256"; do set -- $cfg
BS_SPLITK_MIN_CHUNKS=$1 BS_K5_BN_MAX=$2 timeout 300 python - <<'PY' | sed "s/^/mc=$1 bn=$2 /" >> gpurun_out/r2_tc69.txt 2>&1
import sys, json
sys.path.insert(0, '.')
import torch, paper_1811_00206_b200 as bs, synth
from bench import graph_time_us, rotating
l2 = torch.cuda.get_device_properties(0).L2_cache_size
M, K = 4096, 2048
W = synth.matrix(M, K, "f16", seed=3, device="cuda"); v, i, _ = bs.prune(W, 4, k=2)
ms = rotating(bs, bs.pack(v, i, K, 4, layout="sp24"), l2); C = len(ms)
out = {}
for N in (16, 32, 64, 128, 256):
    X = synth.vector(K, "f16", seed=4, n=N, device="cuda"); Y = torch.empty((N, M), dtype=torch.float16, device="cuda")
    out[N] = round(graph_time_us(lambda j: bs.spmm(ms[j % C], X, out=Y), 20 * C if C < 10 else 2 * C), 2)
print(json.dumps(out))
PY
done
cat gpurun_out/r2_tc69.txt
