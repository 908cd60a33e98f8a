"""K5 (2:4 sparse MMA) and K6 (decompress -> dense MMA) at mid and large N, graph-timed with rotating
copies, next to cuBLAS on the same W_bs: python tools/tc_probe.py [case ...]. BS_TC_ORDER / BS_LIB for A/B."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_00206_b200 as bs  # noqa: E402

if os.environ.get("BS_LIB"):
    bs.LIB_PATH = os.environ["BS_LIB"]
import synth  # noqa: E402
from bench import graph_time_us, rotating, dense_from_canonical  # noqa: E402

l2 = torch.cuda.get_device_properties(0).L2_cache_size
dev = torch.device("cuda")
# (name, M, K, B, k, layout, Ns)
cases = [("sp24_16384", 16384, 16384, 4, 2, "sp24", [128, 256, 1024]),
         ("sp24_ctc_ih", 4096, 2048, 4, 2, "sp24", [16, 64, 256]),
         ("k6_16384_90", 16384, 16384, 32, 3, "spmm", [256, 1024]),
         ("k6_fc6", 4096, 25088, 32, 3, "spmm", [32, 128]),
         ("k6_ctc_ih", 4096, 2048, 32, 4, "spmm", [32, 64, 256]),
         ("k6_conv3_3", 256, 2304, 32, 4, "spmm", [3136]),
         ("k6_conv4_2", 512, 4608, 32, 3, "spmm", [784])]
only = sys.argv[1:]
for name, M, K, B, k, lay, Ns in cases:
    if only and name not in only:
        continue
    W = synth.matrix(M, K, "f16", seed=3, device=dev)
    v, i, _ = bs.prune(W, B, k=k)
    ms = rotating(bs, bs.pack(v, i, K, B, layout=lay), l2)
    Wd = dense_from_canonical(v, i, M, K, B)
    del W
    for N in Ns:
        X = synth.vector(K, "f16", seed=4, n=N, device=dev)
        Y = torch.empty((N, M), dtype=torch.float16, device=dev)
        C = len(ms)
        us = graph_time_us(lambda j: bs.spmm(ms[j % C], X, out=Y), 20 * C if C < 10 else 2 * C)
        cb = graph_time_us(lambda j: torch.matmul(X, Wd.t()), 20)
        fl = 2.0 * M * K * N
        print(json.dumps({"case": name, "M": M, "K": K, "N": N, "us": round(us, 2), "cublas_us": round(cb, 2),
                          "x_cublas": round(cb / us, 2), "dense_equiv_TFLOPs": round(fl / us / 1e6, 1),
                          "order": os.environ.get("BS_TC_ORDER", "1")}), flush=True)
    del v, i, ms, Wd
