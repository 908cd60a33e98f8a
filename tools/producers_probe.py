"""The offline producers (bs_prune_k, bs_pack, bs_block_rank, bs_decode, masks) on a W of M x K f16, for ncu
and A/B timing:  python tools/producers_probe.py [M] [K] [k ...]"""
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

M = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
K = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
ks = [int(v) for v in sys.argv[3:]] or [3, 16]
W = synth.matrix(M, K, "f16", seed=1, device="cuda")
dense = W.numel() * 2


def t_ms(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"M": M, "K": K}
for k in ks:
    t = t_ms(lambda: bs.prune(W, 32, k=k))
    out[f"prune_k{k}_ms"] = round(t, 3)
    out[f"prune_k{k}_TBps"] = round(dense / t / 1e9, 2)
v, i, _ = bs.prune(W, 32, k=3)
t = t_ms(lambda: bs.pack(v, i, K, 32))
out["pack_ms"] = round(t, 3)
t = t_ms(lambda: bs.block_rank(W, 32))
out["block_rank_ms"] = round(t, 3)
out["block_rank_TBps"] = round((dense + W.numel()) / t / 1e9, 2)
D = torch.empty_like(W)
t = t_ms(lambda: bs.decode(v, i, K, 32, out=D))
out["decode_ms"] = round(t, 3)
print(json.dumps(out), flush=True)
