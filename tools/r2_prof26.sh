mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_exact.py tests/test_gpu_parity.py -m gpu -q -x -k "spmm or sp24 or k6 or k5" > gpurun_out/r2_gpu26.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gpu26.log
cat > /tmp/c.py <<'PY'
import sys; sys.argv=['x']
PY
timeout 600 python - > gpurun_out/r2_tc26.txt 2>&1 <<'PY'
import sys, json, os
sys.path.insert(0, '.')
import torch, paper_1811_00206_b200 as bs, synth
from bench import graph_time_us, rotating, dense_from_canonical
l2 = torch.cuda.get_device_properties(0).L2_cache_size
for (M, K) in ((16384, 16384), (16384, 8192)):
    W = synth.matrix(M, K, "f16", seed=3, device="cuda"); v, i, _ = bs.prune(W, 4, k=2)
    ms = rotating(bs, bs.pack(v, i, K, 4, layout="sp24"), l2); Wd = dense_from_canonical(v, i, M, K, 4); del W
    for N in (1, 8, 32, 64, 128, 256, 512, 1024):
        X = synth.vector(K, "f16", seed=4, n=N, device="cuda"); Y = torch.empty((N, M), dtype=torch.float16, device="cuda"); C = len(ms)
        us = graph_time_us(lambda j: bs.spmm(ms[j % C], X, out=Y), 20 * C if C < 10 else 2 * C)
        cb = graph_time_us(lambda j: torch.matmul(X, Wd.t()), 20)
        print(json.dumps({"M": M, "K": K, "N": N, "us": round(us, 2), "cublas_us": round(cb, 2), "x": round(cb / us, 2), "TFLOPs_dense_equiv": round(2*M*K*N/us/1e6, 1)}), flush=True)
PY
cat gpurun_out/r2_tc26.txt
