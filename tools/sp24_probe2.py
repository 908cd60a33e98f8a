"""K5 (2:4 sparse tensor cores) A/B: CTC W_ih 4096x2048, W_hh 4096x1024 and 16384^2 at several N, graph-timed
with rotating copies, beside cuBLAS dense on the same W_bs. Tuning knobs: BS_SPLITK_MIN_CHUNKS, BS_K5_BN_MAX."""
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
tag = os.environ.get("TAG", "")
for name, M, K, Ns in (("CTC_ih", 4096, 2048, [16, 64, 128, 256]), ("CTC_hh", 4096, 1024, [16, 64, 256]),
                       ("16384sq", 16384, 16384, [32, 256, 1024])):
    W = synth.matrix(M, K, "f16", seed=3, device="cuda")
    v, i, _ = bs.prune(W, 4, k=2)
    mats = rotating(bs, bs.pack(v, i, K, 4, layout="sp24"), l2)
    C = len(mats)
    Wd = dense_from_canonical(v, i, M, K, 4)
    dens = [Wd] + [Wd.clone() for _ in range(max(1, -(-3 * l2 // (Wd.numel() * 2))) - 1)]
    Cd = len(dens)
    for N in Ns:
        X = synth.vector(K, "f16", seed=4, n=N, device="cuda")
        Y = torch.empty((N, M), dtype=torch.float16, device="cuda")
        t = graph_time_us(lambda j: bs.spmm(mats[j % C], X, out=Y), 20 * C if C < 10 else 2 * C)
        td = graph_time_us(lambda j: torch.matmul(X, dens[j % Cd].t()), 4 * Cd)
        print(json.dumps({"tag": tag, "case": name, "N": N, "k5_us": round(t, 2), "cublas_us": round(td, 2),
                          "speedup": round(td / t, 2)}), flush=True)
    del mats, dens, Wd, W, v, i
