"""Timeline of the SpMV kernel phases (debug build with -DBS_TRACE): python tools/trace_probe.py ptb 0.97"""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PKG = os.path.join(ROOT, "paper_1811_00206_b200")
LIB = os.path.join(ROOT, "probe_bin", "libbs_trace.so")


def build():
    import __graft_entry__
    b = __graft_entry__._build_module()
    objs = []
    os.makedirs(os.path.join(ROOT, "build", "trace"), exist_ok=True)
    for src in b.SOURCES:
        o = os.path.join(ROOT, "build", "trace", src + ".o")
        subprocess.check_call([b.NVCC, *b.ARCH, *b.FLAGS, "-DBS_TRACE", "-c", os.path.join(b.CSRC, src), "-o", o])
        objs.append(o)
    subprocess.check_call([b.NVCC, *b.ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs])


if __name__ == "__main__":
    if "--build" in sys.argv:
        build()
        sys.exit(0)
    import torch
    import paper_1811_00206_b200 as bs
    import synth
    SH = {"ptb": (6000, 3008), "fc7": (4096, 4096), "fc6": (4096, 25088), "big": (65536, 65536), "ctc_hh": (4096, 1024)}
    name, s = sys.argv[1], float(sys.argv[2])
    M, K = SH[name]
    bs.LIB_PATH = LIB  # swap in the traced library (same ABI)
    bs._LIB = bs._load()
    W = synth.matrix(M, K, "f16", seed=1, device="cuda")
    x = synth.vector(K, "f16", seed=2, device="cuda")
    v, i, k = bs.prune(W, 32, sparsity=s)
    A = bs.pack(v, i, K, 32)
    mats = [A] + [bs.BSMatrix(A.M, A.K, A.block, A.k, A.dtype, A.layout, A.packed.clone()) for _ in range(60)]
    y = torch.empty(M, dtype=torch.float16, device="cuda")
    for j in range(40):
        bs.spmv(mats[j % len(mats)], x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fl = int(os.environ.get("FLAGS", "1"))
    bs.spmv(mats[-2], x, out=y, flags=fl)  # the traced kernel follows another one, as in a layer chain
    bs.spmv(mats[-1], x, out=y, flags=fl)
    e1.record()
    torch.cuda.synchronize()
    n = 148 * 16 * 16
    buf = (ctypes.c_ulonglong * n)()
    bs.lib().bs_trace_read(ctypes.byref(buf), n)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(148, 16, 16).astype(np.int64)
    t0 = t[:, :, 0][t[:, :, 0] > 0].min()
    rel = np.where(t > 0, t - t0, -1)
    print(f"{name} s={s} event_us={e0.elapsed_time(e1)*1e3:.2f}")
    for ph, lab in [(0, "entry"), (5, "mbar init"), (7, "1st copy"), (1, "issued"), (6, "staged(warp)"), (2, "x staged"), (3, "first stage"), (4, "panels done"), (8, "end")]:
        col = rel[:, :, ph]
        col = col[col >= 0]
        if col.size:
            print(f"  {lab:12s} min {col.min()/1e3:7.2f} med {np.median(col)/1e3:7.2f} max {col.max()/1e3:7.2f} us")
