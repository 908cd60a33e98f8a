"""Run one small layer's SpMV a few times (for ncu): python tools/small_probe.py ptb|fc7|fc6 [sparsity]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_00206_b200 as bs  # noqa: E402
import synth  # noqa: E402

SHAPES = {"ptb": (6000, 3008), "fc7": (4096, 4096), "fc6": (4096, 25088), "ctc_hh": (4096, 1024), "big": (65536, 65536)}
name = sys.argv[1] if len(sys.argv) > 1 else "ptb"
s = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
M, K = SHAPES[name]
W = synth.matrix(M, K, "f16", seed=1, device="cuda")
x = synth.vector(K, "f16", seed=2, device="cuda")
v, i, k = bs.prune(W, 32, sparsity=s)
A = bs.pack(v, i, K, 32)
y = torch.empty(M, dtype=torch.float16, device="cuda")
for _ in range(int(os.environ.get("REPS", "8"))):
    bs.spmv(A, x, out=y)
torch.cuda.synchronize()
print(name, s, k, A.nbytes)
