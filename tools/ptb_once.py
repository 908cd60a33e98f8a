"""Run the PTB layer's SpMV (6000 x 3008, 90 %, f16) a few times, for ncu: python tools/ptb_once.py [M K s]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_00206_b200 as bs  # noqa: E402
import synth  # noqa: E402

M, K, s = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (6000, 3008, 0.9)
W = synth.matrix(M, K, "f16", seed=1, device="cuda")
x = synth.vector(K, "f16", seed=2, device="cuda")
v, i, k = bs.prune(W, 32, sparsity=s)
A = bs.pack(v, i, K, 32)
y = torch.empty(M, dtype=torch.float16, device="cuda")
for _ in range(6):
    bs.spmv(A, x, out=y, flags=bs.SPMV_PDL | bs.SPMV_W_STATIC)
torch.cuda.synchronize()
print("ok")
