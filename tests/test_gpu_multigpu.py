"""T3: the multi-GPU paths on real GPUs over NCCL (skipped unless >= 2 GPUs are visible; every gpurun box of
this build has one, so the single-GPU simulations in test_gpu_dist.py carry the fused protocol there).

World = min(4, GPUs) ranks, one per GPU, NCCL backend on 127.0.0.1. Each rank prunes and packs its own row
slice of the same seeded layer (synth regenerates any row slice byte-identically); the test then requires,
bit for bit against the 1-GPU product computed on cuda:0:
  - RowShardedBS (local bs_spmv + NCCL all_gather_into_tensor): every rank's full y;
  - FusedRowShardedBS (bs_spmv_allgather over CUDA-IPC peer mappings + bs_allgather_wait): every rank's y,
    over three epochs (the two y buffers alternate);
  - BatchShardedBS (replicated W, split batch, gather=True): every rank's full Y.
Row sharding is bit-identical because the summation order depends on (K, B, dtype) only (A10)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs >= 2 GPUs (NCCL)")]

M, K, B, k, N = 4096 + 37, 8192, 32, 3, 10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        import paper_1811_00206_b200 as bs
        from paper_1811_00206_b200.dist import BatchShardedBS, FusedRowShardedBS, RowShardedBS, row_range
        r0, r1 = row_range(M, world, rank)
        Wl = synth.matrix(r1 - r0, K, "f16", seed=synth.seed_for(50, 0), row0=r0, device=dev)
        v, i, _ = bs.prune(Wl, B, k=k)
        Al = bs.pack(v, i, K, B)
        x = synth.vector(K, "f16", seed=synth.seed_for(50, 1), device=dev)
        y_nccl = RowShardedBS(Al, M)(x).clone()
        fused = FusedRowShardedBS(Al, M, torch.float16, dev)
        y_fused = [fused(x).clone() for _ in range(3)]
        torch.cuda.synchronize(dev)
        dist.barrier()
        fused.close()
        W = synth.matrix(M, K, "f16", seed=synth.seed_for(50, 0), device=dev)
        vf, i_f, _ = bs.prune(W, B, k=k)
        X = synth.vector(K, "f16", seed=synth.seed_for(50, 2), n=N, device=dev)
        Y = BatchShardedBS(bs.pack(vf, i_f, K, B))(X, gather=True)
        torch.cuda.synchronize(dev)
        q.put((rank, y_nccl.cpu(), [y.cpu() for y in y_fused], Y.cpu()))
    except Exception as e:  # report instead of hanging the parent on the queue
        q.put((rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


def test_nccl_row_fused_batch_bit_identical():
    import paper_1811_00206_b200 as bs
    world = min(4, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    for rank, y_nccl, _, _ in out:
        assert not isinstance(y_nccl, str), f"rank {rank}: {y_nccl}"
    dev = torch.device("cuda", 0)
    W = synth.matrix(M, K, "f16", seed=synth.seed_for(50, 0), device=dev)
    v, i, _ = bs.prune(W, B, k=k)
    A = bs.pack(v, i, K, B)
    y1 = bs.spmv(A, synth.vector(K, "f16", seed=synth.seed_for(50, 1), device=dev)).cpu()
    Y1 = bs.spmm(A, synth.vector(K, "f16", seed=synth.seed_for(50, 2), n=N, device=dev)).cpu()
    for rank, y_nccl, y_fused, Y in out:
        assert torch.equal(y_nccl, y1), rank
        for e, yf in enumerate(y_fused):
            assert torch.equal(yf, y1), (rank, e)
        assert torch.equal(Y, Y1), rank
    for p in procs:
        assert p.exitcode == 0
