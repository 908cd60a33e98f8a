"""SpMM sweep: bs_spmm vs cuBLAS dense GEMM on the same W_bs, CUDA-graph timed (rotating copies > L2).

    python tools/spmm_sweep.py [shape ...]   shapes: fc6 fc7 ctc_ih ctc_hh bench
One JSON line per (shape, s, N)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1811_00206_b200 as bs  # noqa: E402

LAYOUT = os.environ.get("LAYOUT", "spmv")
import synth  # noqa: E402
from bench import dense_from_canonical, graph_time_us  # noqa: E402

SHAPES = {"fc6": (4096, 25088, [0.9], [8, 32]), "fc7": (4096, 4096, [0.9], [8, 32]),
          "ctc_ih": (4096, 2048, [0.875], [1, 2, 4, 8, 16, 32, 64, 128, 256]),
          "ctc_hh": (4096, 1024, [0.875], [8, 64, 256]), "bench": (16384, 8192, [0.5, 0.9], [8]),
          "sq16k": (16384, 16384, [0.5, 0.9], [1, 8, 32, 128, 256, 1024])}


def main(names):
    dev = torch.device("cuda")
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    for name in names:
        M, K, sps, Ns = SHAPES[name]
        W = synth.matrix(M, K, "f16", seed=3, device=dev)
        B = 4 if LAYOUT == "sp24" else 32
        for s in ([0.5] if LAYOUT == "sp24" else sps):
            k = bs.k_from_sparsity(B, s)
            v, i, _ = bs.prune(W, B, k=k)
            A = bs.pack(v, i, K, B, layout=LAYOUT)
            Wd = dense_from_canonical(v, i, M, K, B)
            C = max(1, -(-3 * l2 // A.nbytes))
            mats = [A] + [bs.BSMatrix(A.M, A.K, A.block, A.k, A.dtype, A.layout, A.packed.clone()) for _ in range(C - 1)]
            Cd = max(1, -(-3 * l2 // (Wd.numel() * 2)))
            dens = [Wd] + [Wd.clone() for _ in range(Cd - 1)]
            for N in Ns:
                X = synth.vector(K, "f16", seed=4, n=N, device=dev)
                Y = torch.empty((N, M), dtype=torch.float16, device=dev)
                t = graph_time_us(lambda j: bs.spmm(mats[j % C], X, out=Y), max(2 * C, 20))
                td = graph_time_us(lambda j: torch.matmul(X, dens[j % Cd].t()), max(2 * Cd, 20))
                flops = 2.0 * A.nnz * N
                print(json.dumps({"layout": LAYOUT, "shape": name, "M": M, "K": K, "s": s, "k": k, "N": N, "us": round(t, 2),
                                  "cublas_us": round(td, 2), "speedup": round(td / t, 2),
                                  "TFLOPs_alg": round(flops / t / 1e6, 2), "packed_MB": round(A.nbytes / 1e6, 2)}),
                      flush=True)
            del mats, dens, A, Wd


if __name__ == "__main__":
    main(sys.argv[1:] or list(SHAPES))
