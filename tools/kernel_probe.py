"""Run one product of a chosen path a few times (for ncu captures of a single kernel).

    python tools/kernel_probe.py LAYOUT M K s N [B]     e.g. spmm 16384 16384 0.9 8"""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1811_00206_b200 as bs  # noqa: E402
import synth  # noqa: E402

layout, M, K, s, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
B = int(sys.argv[6]) if len(sys.argv) > 6 else (4 if layout == "sp24" else 32)
W = synth.matrix(M, K, "f16", seed=3, device="cuda")
v, i, k = bs.prune(W, B, sparsity=s)
A = bs.pack(v, i, K, B, layout=layout)
X = synth.vector(K, "f16", seed=4, n=N, device="cuda")
for _ in range(3):
    Y = bs.spmm(A, X) if N > 1 or layout != "spmv" else bs.spmv(A, X[0])
torch.cuda.synchronize()
print("ok", layout, M, K, s, N, B, k)
