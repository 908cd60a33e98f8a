"""Timing sweep of bs_spmv_ex on the paper's layer shapes (FLAGS = launch flags) on the GPU.

    python tools/spmv_sweep.py            # parent: runs each knob combination in a subprocess
Prints one JSON line per (knobs, shape, sparsity): microseconds and packed GB/s (CUDA events, rotating
copies so the working set exceeds L2)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [("big", 65536, 65536), ("fc6", 4096, 25088), ("fc7", 4096, 4096), ("ptb", 6000, 3008), ("ctc_ih", 4096, 2048), ("ctc_hh", 4096, 1024)]
SPARS = [0.5, 0.9, 0.97]


FLAGS = int(os.environ.get("FLAGS", "3"))  # bs_spmv_ex flags: 1 = PDL, 3 = PDL | W_STATIC


def child():
    import torch
    import paper_1811_00206_b200 as bs
    import synth
    if os.environ.get("BS_LIB"):  # A/B runs against another build of the same ABI
        bs.LIB_PATH = os.environ["BS_LIB"]
        bs._LIB = bs._load()
    dev = torch.device("cuda", 0)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    shapes = [s for s in SHAPES if s[0] in os.environ.get("SHAPES", "big,fc6,fc7,ptb,ctc_ih,ctc_hh").split(",")]
    for name, M, K in shapes:
        W = synth.matrix(M, K, "f16", seed=1, device=dev)
        x = synth.vector(K, "f16", seed=2, device=dev)
        for s in (SPARS if not name.startswith("ctc") else [0.875]):
            k = bs.k_from_sparsity(32, s)
            v, i, _ = bs.prune(W, 32, k=k)
            A = bs.pack(v, i, K, 32)
            del v, i
            C = max(1, -(-3 * l2 // A.nbytes))
            mats = [A] + [bs.BSMatrix(A.M, A.K, A.block, A.k, A.dtype, A.layout, A.packed.clone()) for _ in range(C - 1)]
            y = torch.empty(M, dtype=torch.float16, device=dev)
            iters = max(50, min(3000, int(3e10 / A.nbytes)))
            for j in range(10):
                bs.spmv(mats[j % C], x, out=y)
            torch.cuda.synchronize()
            # capture the launches in a CUDA graph so host launch overhead does not hide kernel time
            g = torch.cuda.CUDAGraph()
            s_ = torch.cuda.Stream()
            with torch.cuda.stream(s_):
                with torch.cuda.graph(g, stream=s_):
                    for j in range(min(iters, 200)):
                        bs.spmv(mats[j % C], x, out=y, flags=FLAGS)
            reps = max(1, iters // 200)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / (reps * min(iters, 200)) * 1e3
            pk = A.nbytes + K * 2 + M * 2
            print(json.dumps({
                              "shape": name, "s": s, "us": round(us, 2), "GBps": round(pk / us / 1e3, 1),
                              "copies": C, "flags": FLAGS, "lib": os.path.basename(os.environ.get("BS_LIB", "libbs.so"))}), flush=True)
            del mats, A


if __name__ == "__main__":
    if "--child" in sys.argv:
        child()
        sys.exit(0)
    for _ in (0,):
        env = dict(os.environ)
        subprocess.run([sys.executable, __file__, "--child"], env=env, check=False)
