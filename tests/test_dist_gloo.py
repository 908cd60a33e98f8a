"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: row slices, padding, gather order, batch split.

The local product is injected (`local_fn`) with an fp64-oracle stand-in, because there is no GPU here. On the
GPU the same classes call the CUDA kernels and NCCL (bench.py --gpus N). Importing
paper_1811_00206_b200.dist does not load libbs.so (the package loads it on first use), so these tests
run on a checkout without the CUDA build."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

M, K, B, k = 37, 256, 32, 3   # 37 rows: uneven slices (19 + 18)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _Local:
    def __init__(self, r0, r1):
        W = synth.to_numpy(synth.matrix(r1 - r0, K, "f32", seed=5, row0=r0)) if r1 > r0 else None
        self.vi = oracle.prune(W, oracle.F32, B, k) if W is not None else None
        self.M = r1 - r0


def _spmv_oracle(local, x, out):
    v, i = local.vi
    y, _ = oracle.spmv(v, i, oracle.F32, local.M, K, B, k, x.numpy())
    out.copy_(torch.from_numpy(y.astype(np.float32)))
    return out


class _Full:
    M = M


def _spmm_oracle(A, X):
    W = synth.to_numpy(synth.matrix(M, K, "f32", seed=5))
    v, i = oracle.prune(W, oracle.F32, B, k)
    Y, _ = oracle.spmm(v, i, oracle.F32, M, K, B, k, np.ascontiguousarray(X.numpy()))
    return torch.from_numpy(Y.astype(np.float32))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_00206_b200.dist import BatchShardedBS, RowShardedBS, row_range
        r0, r1 = row_range(M, world, rank)
        layer = RowShardedBS(_Local(r0, r1), M, local_fn=_spmv_oracle)
        x = synth.vector(K, "f32", seed=6)
        y = layer(x)
        Xb = synth.vector(K, "f32", seed=7, n=5)
        Yb = BatchShardedBS(_Full(), local_fn=_spmm_oracle)(Xb, gather=True)
        q.put((rank, (r0, r1), y.numpy().copy(), Yb.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_row_and_batch_sharding_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    assert out[0][1] == (0, 19) and out[1][1] == (19, 37)
    W = synth.to_numpy(synth.matrix(M, K, "f32", seed=5))
    v, i = oracle.prune(W, oracle.F32, B, k)
    x = synth.to_numpy(synth.vector(K, "f32", seed=6))
    want, _ = oracle.spmv(v, i, oracle.F32, M, K, B, k, x)
    for _, _, y, Yb in out:
        np.testing.assert_array_equal(y, want.astype(np.float32))   # every rank holds the full y
        Xb = synth.to_numpy(synth.vector(K, "f32", seed=7, n=5))
        Yw, _ = oracle.spmm(v, i, oracle.F32, M, K, B, k, Xb)
        np.testing.assert_array_equal(Yb, Yw.astype(np.float32))


def test_row_range_cover():
    from paper_1811_00206_b200.dist import row_range
    for Mx in (1, 7, 64, 65536, 6000):
        for P in (1, 2, 3, 4, 8):
            spans = [row_range(Mx, P, r) for r in range(P)]
            assert spans[0][0] == 0 and spans[-1][1] == Mx
            for a, b in zip(spans, spans[1:]):
                assert a[1] == b[0]
