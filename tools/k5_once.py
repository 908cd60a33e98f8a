"""Run K5 (SP24 bs_spmm) a few times on one shape, for ncu: python tools/k5_once.py M K N [layout B k]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_00206_b200 as bs  # noqa: E402
import synth  # noqa: E402

M, K, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
lay = sys.argv[4] if len(sys.argv) > 4 else "sp24"
B = int(sys.argv[5]) if len(sys.argv) > 5 else 4
k = int(sys.argv[6]) if len(sys.argv) > 6 else 2
dev = torch.device("cuda")
W = synth.matrix(M, K, "f16", seed=3, device=dev)
v, i, _ = bs.prune(W, B, k=k)
A = bs.pack(v, i, K, B, layout=lay)
del W, v, i
X = synth.vector(K, "f16", seed=4, n=N, device=dev)
Y = torch.empty((N, M), dtype=torch.float16, device=dev)
for _ in range(4):
    bs.spmm(A, X, out=Y)
torch.cuda.synchronize()
print("ok")
