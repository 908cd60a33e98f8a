"""Every kernel of libbs.so once, on BASELINE configs[0] (64 x 64, f32, B = 16, s = 0.5) and on the VGG fc7
layer (4096 x 4096, f16, B = 32, s = 0.9), for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize_probe.py [cfg0|fc7|s3]"""
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
if which == "s3":  # round 2, session 3's kernels: K5 CTA pairs and RT = 2, half-warp direct rows, the LSTM step
    # on the direct kernel, 4-bit index runs (SpMV ring + direct, K4 passes)
    for M, K, N in ((9728, 1024, 40), (8192 + 64, 1536, 80)):  # pairs (S = 1); RT = 2 (S = 2, N > 64)
        W = synth.matrix(M, K, "f16", seed=11, device=dev)
        v4, i4, _ = bs.prune(W, 4, k=2)
        bs.spmm(bs.pack(v4, i4, K, 4, layout="sp24"), synth.vector(K, "f16", seed=12, n=N, device=dev))
    W = synth.matrix(6000, 3008, "f16", seed=13, device=dev)
    v, i, k = bs.prune(W, 32, sparsity=0.9)
    A = bs.pack(v, i, 3008, 32)
    x = synth.vector(3008, "f16", seed=14, device=dev)
    bs.spmv(A, x)                                    # half-warp rows
    bs.lstm_step(A, x, torch.zeros(1500, dtype=torch.float32, device=dev), bias=x[:0].new_zeros(6000))
    W = synth.matrix(512, 4096 + 128, "bf16", seed=15, device=dev)
    v, i, k = bs.prune(W, 16, k=3)
    A = bs.pack(v, i, 4096 + 128, 16)               # 4-bit index runs + tail
    bs.unpack(A)
    xb = synth.vector(4096 + 128, "bf16", seed=16, device=dev)
    bs.spmv(A, xb)                                   # direct kernel
    bs.spmv(A, xb, flags=bs.SPMV_PDL | bs.SPMV_RING)  # ring kernel
    bs.spmm(A, synth.vector(4096 + 128, "bf16", seed=17, n=11, device=dev))  # K4 passes
    torch.cuda.synchronize()
    sys.exit(0)
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
