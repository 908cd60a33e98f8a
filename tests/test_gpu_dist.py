"""The fused all-gather (bs_spmv_allgather + bs_allgather_wait) and the pipelined
NCCL path, checked on ONE GPU by simulating P ranks: each simulated rank has its own full y buffers, flags
and counter on the device, and its shard's SpMV kernel stores into all of them exactly as it would through
peer-mapped NVLink pointers. Bar: every rank's y is bit-identical to the unsharded SpMV (O-9), epoch after
epoch (buffer parity, monotonic counters, flag protocol)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bs():
    import paper_1811_00206_b200 as bs
    return bs


@pytest.mark.parametrize("M,K,P,dname", [(1000, 25088, 2, "f16"), (4099, 4096, 3, "bf16"), (8192, 8192, 8, "f16"),
                                         (333, 3008, 8, "f32")])
def test_fused_allgather_simulated_ranks(bs, M, K, P, dname):
    from paper_1811_00206_b200.dist import FusedRowShardedBS, row_range
    B, k = 32, 3
    dev = torch.device("cuda")
    W = synth.matrix(M, K, dname, seed=synth.seed_for(60, M)).to(dev)
    vals, idx, _ = bs.prune(W, B, k=k)
    A = bs.pack(vals, idx, K, B)
    peers = FusedRowShardedBS.make_peers(P, M, W.dtype, dev)
    layers = []
    for r in range(P):
        r0, r1 = row_range(M, P, r)
        v, i, _ = bs.prune(W[r0:r1].contiguous(), B, k=k)
        layers.append(FusedRowShardedBS(bs.pack(v, i, K, B), M, W.dtype, dev, rank=r, world=P, peers=peers))
    for epoch in range(1, 6):
        x = synth.vector(K, dname, seed=synth.seed_for(60, 100 + epoch)).to(dev)
        ref = bs.spmv(A, x)
        outs = [layer.launch(x) for layer in layers]   # every rank's SpMV (stores into all ranks' y)
        for layer in layers:
            layer.wait()
        torch.cuda.synchronize()
        for r, y in enumerate(outs):
            assert torch.equal(y, ref), (epoch, r)
            assert y.data_ptr() == peers["y"][r][epoch % 2].data_ptr()
        for r in range(P):
            assert torch.all(peers["flags"][r] == epoch)
    for r in range(P):
        c = int(peers["counter"][r].item())
        assert c % 5 == 0 and c > 0


def test_fused_allgather_epilogue_and_errors(bs):
    """bias + ReLU fused with the all-gather equals bs_spmv_fused; a bad bs_allgather is rejected."""
    from paper_1811_00206_b200 import _AllGather
    from paper_1811_00206_b200.dist import FusedRowShardedBS, row_range
    M, K, B, k, P = 700, 4096, 32, 4, 4
    dev = torch.device("cuda")
    W = synth.matrix(M, K, "f16", seed=61).to(dev)
    x = synth.vector(K, "f16", seed=62).to(dev)
    bias = synth.vector(M, "f16", seed=63).to(dev)
    vals, idx, _ = bs.prune(W, B, k=k)
    ref = bs.spmv(bs.pack(vals, idx, K, B), x, bias=bias, act="relu")
    peers = FusedRowShardedBS.make_peers(P, M, W.dtype, dev)
    layers = []
    for r in range(P):
        r0, r1 = row_range(M, P, r)
        v, i, _ = bs.prune(W[r0:r1].contiguous(), B, k=k)
        layers.append(FusedRowShardedBS(bs.pack(v, i, K, B), M, W.dtype, dev, rank=r, world=P, peers=peers))
    outs = []
    for r, layer in enumerate(layers):
        r0, r1 = row_range(M, P, r)
        outs.append(layer.launch(x, bias=bias[r0:r1].contiguous(), act="relu"))
    for layer in layers:
        layer.wait()
    for y in outs:
        assert torch.equal(y, ref)
    ag = _AllGather()
    ag.nranks, ag.rank, ag.epoch = 9, 0, 1
    with pytest.raises(bs.BSError):
        bs.spmv_allgather(layers[0].local, x, ag)
    ag2 = layers[0]._ag()
    ag2.epoch = 0
    with pytest.raises(bs.BSError):
        bs.allgather_wait(ag2, dev)


def test_peer_export_roundtrip(bs):
    """bs_peer_export finds the allocation base and offset of a pointer inside a torch tensor (the import
    side needs a second process; it is exercised by FusedRowShardedBS under torchrun)."""
    import ctypes
    t = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    assert bs.lib().bs_peer_export(ctypes.c_void_p(t.data_ptr() + 4096), h, ctypes.byref(off)) == 0
    assert off.value >= 4096 and any(h.raw)
