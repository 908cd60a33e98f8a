"""Time bs_prune (K1) on the paper's shapes: python tools/prune_probe.py [BS_LIB path for A/B]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_00206_b200 as bs  # noqa: E402
import synth  # noqa: E402

if len(sys.argv) > 1:
    bs.LIB_PATH = sys.argv[1]
    bs._LIB = bs._load()
for name, M, K, dt in (("big", 65536, 65536, "f16"), ("fc6", 4096, 25088, "f16"), ("fc6_f32", 4096, 25088, "f32")):
    W = synth.matrix(M, K, dt, seed=1, device="cuda")
    for k in (3, 8, 16, 1):
        bs.prune(W, 32, k=k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            bs.prune(W, 32, k=k)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(json.dumps({"shape": name, "k": k, "ms": round(ms, 3), "dense_read_GBps": round(W.numel() * W.element_size() / ms / 1e6, 1),
                          "lib": os.path.basename(bs.LIB_PATH)}), flush=True)
    del W
