mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gpu36.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2_gpu36.log
timeout 300 python - > gpurun_out/r2_b16_36.txt 2>&1 <<'PY'
import sys, json
sys.path.insert(0, '.')
import torch, paper_1811_00206_b200 as bs, synth
from bench import graph_time_us, rotating, dense_from_canonical
l2 = torch.cuda.get_device_properties(0).L2_cache_size
for (M, K, B, s) in ((65536, 65536, 16, 0.875), (16384, 16384, 16, 0.875), (4096, 25088, 16, 0.875)):
    W = synth.matrix(M, K, "f16", seed=1, device="cuda"); x = synth.vector(K, "f16", seed=2, device="cuda")
    v, i, k = bs.prune(W, B, sparsity=s); del W
    A = bs.pack(v, i, K, B); ms = rotating(bs, A, l2); C = len(ms)
    y = torch.empty(M, dtype=torch.float16, device="cuda")
    us = graph_time_us(lambda j: bs.spmv(ms[j % C], x, out=y), 20 * C if C < 10 else 2 * C)
    nnz = M * (K // B) * k
    print(json.dumps({"M": M, "K": K, "B": B, "k": k, "us": round(us, 2), "packed_MB": round(A.nbytes / 1e6, 1),
                      "B_per_nnz": round(A.nbytes / nnz, 3), "packed_GBps": round((A.nbytes + 2 * K + 2 * M) / us / 1e3, 1)}), flush=True)
    del v, i, A, ms
PY
cat gpurun_out/r2_b16_36.txt
