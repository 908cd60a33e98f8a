"""A/B: the direct short-row SpMV kernel vs the streaming-ring kernel on the latency-regime layers (PTB,
fc7, CTC, fc6 at 97 %), graph-timed with rotating copies (> 3x L2), PDL + static weights."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_00206_b200 as bs  # noqa: E402

if os.environ.get("BS_LIB"):  # A/B against another build of the same ABI
    bs.LIB_PATH = os.environ["BS_LIB"]
import synth  # noqa: E402
from bench import graph_time_us, rotating  # noqa: E402

l2 = torch.cuda.get_device_properties(0).L2_cache_size
dev = torch.device("cuda")
for name, M, K, s in (("PTB", 6000, 3008, 0.9), ("fc7_90", 4096, 4096, 0.9), ("CTC_ih", 4096, 2048, 0.875),
                      ("CTC_hh", 4096, 1024, 0.875), ("fc6_97", 4096, 25088, 0.97), ("fc6_90", 4096, 25088, 0.9),
                      ("fc7_75", 4096, 4096, 0.75)):
    W = synth.matrix(M, K, "f16", seed=1, device=dev)
    x = synth.vector(K, "f16", seed=2, device=dev)
    y = torch.empty(M, dtype=torch.float16, device=dev)
    v, i, k = bs.prune(W, 32, sparsity=s)
    mats = rotating(bs, bs.pack(v, i, K, 32), l2)
    C = len(mats)
    n = 20 * C if C < 10 else 2 * C
    row = {"layer": name, "k": k}
    for lab, fl in (("direct", bs.SPMV_PDL | bs.SPMV_W_STATIC), ("ring", bs.SPMV_PDL | bs.SPMV_W_STATIC | bs.SPMV_RING),
                    ("direct_nopdl", 0), ("ring_nopdl", bs.SPMV_RING)):
        row[lab + "_us"] = round(graph_time_us(lambda j: bs.spmv(mats[j % C], x, out=y, flags=fl), n), 2)
    print(json.dumps(row), flush=True)
