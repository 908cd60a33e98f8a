"""K5 (2:4 sparse tensor cores) on the CTC W_ih layer 4096 x 2048 at N = 16 and 256, graph-timed."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_00206_b200 as bs  # noqa: E402
import synth  # noqa: E402
from bench import graph_time_us  # noqa: E402

W = synth.matrix(4096, 2048, "f16", seed=3, device="cuda")
v, i, _ = bs.prune(W, 4, k=2)
A = bs.pack(v, i, 2048, 4, layout="sp24")
for N in [int(a) for a in sys.argv[1:]] or [16, 256]:
    X = synth.vector(2048, "f16", seed=4, n=N, device="cuda")
    Y = torch.empty((N, 4096), dtype=torch.float16, device="cuda")
    print(json.dumps({"N": N, "k5_us": round(graph_time_us(lambda j: bs.spmm(A, X, out=Y), 20), 2)}), flush=True)
