"""K6 phase timeline (library built with -DBS_TRACE_K6 into probe_bin/libbs_k6trace.so):
python tools/k6_trace_probe.py M K B k N. Prints, per phase mark, percentiles over CTAs of the time since the
earliest CTA start (us): 0 entry, 1 set-up done (after the PDL wait), 2 first chunk's stage full (decompress
group 0), 3 group 0's last chunk, 4 accumulator ready, 5 partial tile parked, 6 after the first cluster
barrier, 7 slice summed, 8 end."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_00206_b200 as bs  # noqa: E402
import synth  # noqa: E402

K5 = "--k5" in sys.argv  # the 2:4 kernel (libbs_k5trace.so, -DBS_TRACE_K5): marks 2 = first stage full
argv = [a for a in sys.argv[1:] if a != "--k5"]
bs.LIB_PATH = os.path.join(ROOT, "probe_bin", "libbs_k5trace.so" if K5 else "libbs_k6trace.so")
M, K, B, k, N = (int(v) for v in argv[:5])
W = synth.matrix(M, K, "f16", seed=3, device="cuda")
v, i, _ = bs.prune(W, B, k=k)
A = bs.pack(v, i, K, B, layout="sp24" if K5 else "spmm")
X = synth.vector(K, "f16", seed=4, n=N, device="cuda")
Y = torch.empty((N, M), dtype=torch.float16, device="cuda")
for _ in range(5):
    bs.spmm(A, X, out=Y)
torch.cuda.synchronize()
L = bs.lib()
rd = L.bs_k5_trace_read if K5 else L.bs_k6_trace_read
rd.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(4096 * 16, dtype=np.uint64)
rd(buf.ctypes.data, buf.size)
T = buf.reshape(4096, 16).astype(np.float64)
live = T[:, 0] > 0
T = T[live]
t0 = T[:, 0].min()
print(f"M={M} K={K} B={B} k={k} N={N}: {live.sum()} CTAs")
names = {9: "producer 0: cycles waiting for empty stages", 10: "MMA warp 0: cycles waiting for full stages",
         11: "MMA warp 0: cycles waiting for A tiles", 12: "MMA warp 0: cycles issuing (fence, MMAs, commits)",
         13: "decompress group 0: cycles waiting for free A tiles", 14: "decompress group 0: cycles waiting for stages",
         15: "decompress group 0: cycles decompressing"}
if not K5:
    for m, nm in names.items():
        col = buf.reshape(4096, 16)[live][:, m].astype(np.float64)
        print(f"  {nm}: p50 {np.percentile(col, 50):9.0f}  max {col.max():9.0f}")
for m in range(9):
    col = T[:, m]
    col = col[col > 0]
    if col.size:
        d = (col - t0) / 1e3
        print(f"  mark {m}: min {d.min():7.2f}  p50 {np.percentile(d, 50):7.2f}  p90 {np.percentile(d, 90):7.2f}  max {d.max():7.2f} us")
