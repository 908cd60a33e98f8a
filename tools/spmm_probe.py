"""K4/K5/K6 on the batched shapes, graph-timed (same method as bench.py spmm rows):
python tools/spmm_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_00206_b200 as bs  # noqa: E402
import synth  # noqa: E402
from bench import graph_time_us, rotating, dense_from_canonical  # noqa: E402

l2 = torch.cuda.get_device_properties(0).L2_cache_size
dev = torch.device("cuda")
cases = [("fc6", 4096, 25088, 32, 3, [8, 32, 128]), ("CTC_ih", 4096, 2048, 32, 4, [16, 64, 256]),
         ("CTC_hh", 4096, 1024, 32, 4, [64, 256]), ("conv4_2", 512, 4608, 32, 3, [784]),
         ("conv3_3", 256, 2304, 32, 4, [3136]), ("16384sq", 16384, 16384, 32, 3, [8, 32, 256]),
         ("fc7_50", 4096, 4096, 32, 16, [32, 256])]
only = sys.argv[1:]
for name, M, K, B, k, Ns in cases:
    if only and name not in only:
        continue
    W = synth.matrix(M, K, "f16", seed=3, device=dev)
    v, i, _ = bs.prune(W, B, k=k)
    mats = {lay: rotating(bs, bs.pack(v, i, K, B, layout=lay), l2) for lay in ("spmv", "spmm")}
    Wd = dense_from_canonical(v, i, M, K, B)
    for N in Ns:
        X = synth.vector(K, "f16", seed=4, n=N, device=dev)
        Y = torch.empty((N, M), dtype=torch.float16, device=dev)
        row = {"case": name, "M": M, "K": K, "k": k, "N": N}
        for lay, ms in mats.items():
            C = len(ms)
            if lay == "spmv" and N > 64:
                continue
            row[lay + "_us"] = round(graph_time_us(lambda j: bs.spmm(ms[j % C], X, out=Y), 20 * C if C < 10 else 2 * C), 2)
        row["cublas_us"] = round(graph_time_us(lambda j: torch.matmul(X, Wd.t()), 20), 2)
        print(json.dumps(row), flush=True)
    del W, v, i, mats, Wd
