"""K5 CTA-pair check: python tools/k5_pair_check.py OUT.pt. Computes Y = W·X on SP24 shapes that take the
pair kernel under BS_K5_PAIR=1 (integer-exact data checked against the oracle, Gaussian data saved for a
bit-compare against the single-CTA kernel run in another process)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1811_00206_b200 as bs  # noqa: E402
import synth  # noqa: E402

out = {}
for (M, K, N) in ((9600, 1024, 64), (9600 + 100, 1024, 40), (16384, 2048, 256)):
    W = synth.matrix(M, K, "f16", family="intexact", seed=11 + M)
    vals, idx, _ = bs.prune(W.cuda(), 4, k=2)
    A = bs.pack(vals, idx, K, 4, layout="sp24")
    X = synth.vector(K, "f16", family="intexact", seed=12 + N, n=N)
    Y = bs.spmm(A, X.cuda())
    ov, oi = oracle.prune(synth.to_numpy(W), oracle.F16, 4, 2)
    Yr, _ = oracle.spmm(ov, oi, oracle.F16, M, K, 4, 2, synth.to_numpy(X))
    yd = oracle.to_double(synth.to_numpy(Y), oracle.F16)
    bad = np.argwhere(yd != Yr)
    print("intexact", M, K, N, "mismatches", len(bad), bad[:5].tolist(), flush=True)
    Wg = synth.matrix(M, K, "f16", seed=21 + M).cuda()
    vg, ig, _ = bs.prune(Wg, 4, k=2)
    Ag = bs.pack(vg, ig, K, 4, layout="sp24")
    Xg = synth.vector(K, "f16", seed=22 + N, n=N).cuda()
    out[(M, K, N)] = bs.spmm(Ag, Xg).cpu()
torch.save(out, sys.argv[1])
print("saved", flush=True)
