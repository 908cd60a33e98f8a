"""Diagnose the 2:4 metadata interpretation of tcgen05.mma.sp: X = I (N = 128), so Y^T = W_bs as the tensor
core decoded it. Prints, for a few rows and groups, the expected (column, value) pairs and what came out."""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_1811_00206_b200 as bs  # noqa: E402

M, K, N = 128, 128, 128
torch.manual_seed(0)
W = (torch.randperm(M * K).reshape(M, K).float() / 1000 + 1).to(torch.float16).cuda()  # distinct, positive
X = torch.eye(K, dtype=torch.float16, device="cuda")[:N].contiguous()
v, i, _ = bs.prune(W, 4, k=2)
A = bs.pack(v, i, K, 4, layout="sp24")
Y = bs.spmm(A, X)
torch.cuda.synchronize()
G = Y.t().float().cpu().numpy()  # [M][K] as decoded
vals = v.float().cpu().numpy()
idx = i.cpu().numpy()
Wbs = np.zeros((M, K), np.float32)
for r in range(M):
    for b in range(K // 4):
        for t in range(2):
            Wbs[r, 4 * b + idx[r, b, t]] = vals[r, b, t]
print("max |diff|", np.abs(G - Wbs).max(), "rows ok", int((np.abs(G - Wbs).max(1) == 0).sum()))
for r in (0, 1, 2, 7, 8, 15, 16, 31, 32, 64):
    line = []
    for g in range(0, 32, 3):
        exp = [(int(4 * g + idx[r, g, t]), round(float(vals[r, g, t]), 3)) for t in range(2)]
        got = [(int(c), round(float(G[r, c]), 3)) for c in range(4 * g, 4 * g + 4) if G[r, c] != 0]
        line.append(f"g{g}:{exp}->{got}")
    print(f"row {r}: " + " ".join(line[:5]))
# where did row 0's values go? search the whole output for each expected value
for (r, g) in ((0, 0), (0, 1), (0, 8), (0, 16), (1, 0), (8, 0), (16, 0)):
    for t in range(2):
        val = vals[r, g, t]
        hits = np.argwhere(np.abs(G - val) < 1e-6)
        print(f"value of (row {r}, group {g}, t {t}) = {val:.3f} found at {hits[:4].tolist()}")
import os
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/sp24_probe.npz", G=G, vals=vals, idx=idx)
