"""Every kernel of libbs.so once, on BASELINE configs[0] (64 x 64, f32, B = 16, s = 0.5) and on the VGG fc7
layer (4096 x 4096, f16, B = 32, s = 0.9), for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize_probe.py [cfg0|fc7]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_00206_b200 as bs  # noqa: E402
import synth  # noqa: E402
from paper_1811_00206_b200.dist import FusedRowShardedBS, row_range  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "fc7"
dev = torch.device("cuda")
if which == "cfg0":
    M, K, B, s, dt = 64, 64, 16, 0.5, "f32"
else:
    M, K, B, s, dt = 4096, 4096, 32, 0.9, "f16"
W = synth.matrix(M, K, dt, seed=1, device=dev)
x = synth.vector(K, dt, seed=2, device=dev)
vals, idx, k = bs.prune(W, B, sparsity=s)
A = bs.pack(vals, idx, K, B)
bs.unpack(A)
y = bs.spmv(A, x)
bs.spmv(A, x, bias=y[:M].clone() if M == K else None, act="relu")
X = synth.vector(K, dt, seed=3, n=12, device=dev)
bs.spmm(A, X)                       # K4 passes (16-bit) / per-column SpMV (f32)
bs.block_rank(W, B if B <= 32 else 32)
bs.decode(vals, idx, K, B)
bs.random_mask(W, s)
bs.block_mask(W, 8, 8, s, "mean")
if dt != "f32":
    bs.spmm(A, X[:2].contiguous())   # NV = 2
    Am = bs.pack(vals, idx, K, B, layout="spmm")
    bs.unpack(Am)
    bs.spmm(Am, X)                   # K6 (decompress + tcgen05.mma, split-K cluster)
    v4, i4, _ = bs.prune(W, 4, k=2)
    A4 = bs.pack(v4, i4, K, 4, layout="sp24")
    bs.spmm(A4, X)                   # K5 (tcgen05.mma.sp)
    bs.spmv(A4, x)                   # 2:4 CUDA-core SpMV
    c0 = torch.zeros(M // 4, dtype=torch.float32, device=dev)
    bs.lstm_step(A, x, c0)           # fused LSTM cell epilogue
    img = synth.vector(8 * 8 * 64, dt, seed=4, device=dev).view(1, 8, 8, 64)
    Wc = synth.matrix(64, 9 * 64, dt, seed=5, device=dev)
    vc, ic, _ = bs.prune(Wc, 32, k=3)
    bs.conv2d(bs.pack(vc, ic, 9 * 64, 32, layout="spmm"), img, 3, 3, 1, 1)
    P = 2
    peers = FusedRowShardedBS.make_peers(P, M, W.dtype, dev)
    layers = []
    for r in range(P):
        r0, r1 = row_range(M, P, r)
        vr, ir, _ = bs.prune(W[r0:r1].contiguous(), B, k=k)
        layers.append(FusedRowShardedBS(bs.pack(vr, ir, K, B), M, W.dtype, dev, rank=r, world=P, peers=peers))
    for layer in layers:
        layer.launch(x)
    for layer in layers:
        layer.wait()
torch.cuda.synchronize()
print("sanitize probe done:", which, M, K, B, k, dt)
