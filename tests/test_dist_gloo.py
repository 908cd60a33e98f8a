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


def test_cyclic_chunks_cover_and_gather_order():
    """Block-cyclic chunks: every row owned once; all ranks' chunk j are the contiguous rows [j·P·R, (j+1)·P·R),
    so the chunk-j all-gather lands in order (PipelinedRowShardedBS)."""
    from paper_1811_00206_b200.dist import cyclic_chunks
    for Mx, P, R in ((37, 2, 5), (65536, 8, 1024), (1000, 3, 64), (7, 4, 4)):
        owner = np.full(Mx, -1)
        chunks = [cyclic_chunks(Mx, P, r, R) for r in range(P)]
        assert len({len(c) for c in chunks}) == 1
        for r in range(P):
            for j, (a, b) in enumerate(chunks[r]):
                assert np.all(owner[a:b] == -1)
                owner[a:b] = r
                assert a == min((j * P + r) * R, Mx)
        assert np.all(owner >= 0)


def test_should_shard_policy():
    """shard iff t1 - t1/P > t_allgather."""
    from paper_1811_00206_b200.dist import should_shard
    assert should_shard(231.0, 8, 10.0)          # 65536^2 at 90%: 202 us saved vs ~10 us gather
    assert not should_shard(1.0, 8, 10.0)        # fc7 at 90%: ~1 us on one GPU
    assert not should_shard(100.0, 1, 0.0)
    assert should_shard(20.0, 2, 9.9) and not should_shard(20.0, 2, 10.0)


def _pipelined_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_00206_b200.dist import PipelinedRowShardedBS, cyclic_chunks
        R = 6
        locs = [_Local(a, b) if b > a else None for a, b in cyclic_chunks(M, world, rank, R)]
        layer = PipelinedRowShardedBS(locs, M, R, local_fn=_spmv_oracle)
        y = layer(synth.vector(K, "f32", seed=6))
        q.put((rank, y.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_pipelined_row_sharding_world2():
    """The block-cyclic pipelined path gathers the same y as the unsharded product (host logic, gloo)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipelined_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W = synth.to_numpy(synth.matrix(M, K, "f32", seed=5))
    v, i = oracle.prune(W, oracle.F32, B, k)
    want, _ = oracle.spmv(v, i, oracle.F32, M, K, B, k, synth.to_numpy(synth.vector(K, "f32", seed=6)))
    for _, y in out:
        np.testing.assert_array_equal(y, want.astype(np.float32))
