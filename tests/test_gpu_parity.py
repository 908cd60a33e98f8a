"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle, on the same seeded inputs.

Bar (BASELINE.json north_star):
  - pruning masks (canonical idx and value bits) and packed bytes: bit-exact;
  - y: |y_gpu - y_ref| <= tau * sum|w||x| per element, tau = 1e-4 (f32), 1e-2 (f16/bf16);
  - integer-exact inputs and row sharding: bit-identical.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

DT = {"f32": oracle.F32, "f16": oracle.F16, "bf16": oracle.BF16}


@pytest.fixture(scope="module")
def bs():
    import paper_1811_00206_b200 as bs
    return bs


def _idx_np(idx: torch.Tensor) -> np.ndarray:
    return idx.cpu().numpy().view(np.uint16)


def _raw(t: torch.Tensor) -> np.ndarray:
    a = synth.to_numpy(t)
    return a.view(np.uint32 if a.itemsize == 4 else np.uint16)


def _prune_parity(bs, W: torch.Tensor, dname: str, B: int, k: int):
    vals, idx, k2 = bs.prune(W.cuda(), B, k=k)
    assert k2 == k
    Wn = synth.to_numpy(W)
    ov, oi = oracle.prune(Wn, DT[dname], B, k)
    np.testing.assert_array_equal(_idx_np(idx), oi)
    np.testing.assert_array_equal(_raw(vals), ov.view(np.uint32 if ov.itemsize == 4 else np.uint16))
    return vals, idx, ov, oi


# (M, K, B, k, dtype, family): small shapes that span several panels, a ragged tail, NB < 32,
# B > 256 (u16 indices), odd B, the 2:4 shape and every dtype.
SMALL = [
    (64, 64, 16, 8, "f32", "gaussian"),        # cfg0 tiny (BJ.configs[0])
    (96, 3008, 32, 3, "f16", "gaussian"),      # PTB row width (NB = 94 < 256: tail only)
    (70, 25088, 32, 3, "f16", "gaussian"),     # fc6 row width: 3 panels + 16-block tail
    (33, 25088, 32, 1, "bf16", "gaussian"),
    (50, 4096, 32, 16, "f32", "gaussian"),     # fc7 width, f32: V = 4
    (40, 8192, 32, 2, "bf16", "ties"),
    (48, 2048, 4, 2, "f16", "gaussian"),       # 2:4 shape on the generic path
    (31, 1024, 32, 4, "f16", "sameoffset"),    # CTC W_hh width, NB = 32
    (29, 2048, 512, 9, "f16", "gaussian"),     # B > 256: u16 indices
    (17, 1000, 25, 8, "f32", "ties"),          # odd B (Table brange balance range 25)
    (65, 640, 20, 0, "f16", "gaussian"),       # k = 0
    (8, 256, 16, 16, "bf16", "gaussian"),      # k = B (dense)
    (3, 96, 1, 1, "f16", "gaussian"),          # B = 1
    (40, 4096 + 16 * 40, 16, 4, "f16", "gaussian"),  # 4-bit index runs (B = 16, NB = 296): a panel + a 40-block tail
    (33, 16 * 512, 16, 3, "bf16", "ties"),     # 4-bit runs, two panels, no tail
    (20, 8 * 300, 8, 2, "f16", "sameoffset"),  # 4-bit runs, B = 8
]


@pytest.mark.parametrize("M,K,B,k,dname,family", SMALL)
def test_prune_pack_spmv_small(bs, M, K, B, k, dname, family):
    W = synth.matrix(M, K, dname, family=family, seed=synth.seed_for(0, M + K + B), B=B)
    vals, idx, ov, oi = _prune_parity(bs, W, dname, B, k)
    x = synth.vector(K, dname, seed=synth.seed_for(0, 7))
    for layout, olay in (("spmv", oracle.SPMV), ("spmm", oracle.SPMM)):
        A = bs.pack(vals, idx, K, B, layout=layout)
        assert A.nbytes == oracle.packed_bytes(M, K, B, k, DT[dname], olay)
        np.testing.assert_array_equal(A.packed.cpu().numpy(), oracle.pack(ov, oi, M, K, B, k, DT[dname], olay))
        uv, ui = bs.unpack(A)
        np.testing.assert_array_equal(_raw(uv), _raw(vals))
        np.testing.assert_array_equal(_idx_np(ui), oi)
        if layout == "spmm":  # the tile layout feeds bs_spmm; check it on a 3-column batch
            X3 = synth.vector(K, dname, seed=synth.seed_for(0, 8), n=3)
            Y3 = bs.spmm(A, X3.cuda())
            Yr, bY = oracle.spmm(ov, oi, DT[dname], M, K, B, k, synth.to_numpy(X3))
            ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(Y3), DT[dname]), Yr, bY, oracle.TAU[DT[dname]])
            assert ok, f"spmm: worst |err|/bound = {worst}"
            continue
        y = bs.spmv(A, x.cuda())
        torch.cuda.synchronize()
        yr, bound = oracle.spmv(ov, oi, DT[dname], M, K, B, k, synth.to_numpy(x))
        ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(y), DT[dname]), yr, bound, oracle.TAU[DT[dname]])
        assert ok, f"{layout}: worst |err|/bound = {worst}"


def test_prune_special_values(bs):
    for dname in ("f32", "f16", "bf16"):
        W = synth.special_block_matrix(dname)
        for k in range(0, 17):
            if k == 0:
                continue
            _prune_parity(bs, W, dname, 16, k)


@pytest.mark.parametrize("dname", ["f16", "bf16", "f32"])
def test_spmv_integer_exact_bit_identical(bs, dname):
    """W, x in {-1,0,1}: every partial sum is an exact integer, so y must equal the oracle bit for bit."""
    M, K, B, k = 300, 6144, 32, 5
    W = synth.matrix(M, K, dname, family="intexact", seed=41)
    x = synth.vector(K, dname, family="intexact", seed=42)
    vals, idx, ov, oi = _prune_parity(bs, W, dname, B, k)
    A = bs.pack(vals, idx, K, B)
    y = bs.spmv(A, x.cuda())
    yr, _ = oracle.spmv(ov, oi, DT[dname], M, K, B, k, synth.to_numpy(x))
    assert np.all(np.abs(yr) <= 256)  # representable in every D
    np.testing.assert_array_equal(oracle.to_double(synth.to_numpy(y), DT[dname]), yr)


def test_spmv_unit_vectors(bs):
    """x = e_j returns column j of W_bs exactly (catches wrong offsets, banks or transposes)."""
    M, K, B, k = 40, 8192 + 512, 32, 3
    W = synth.matrix(M, K, "f16", seed=43)
    vals, idx, ov, oi = _prune_parity(bs, W, "f16", B, k)
    A = bs.pack(vals, idx, K, B)
    Wd = oracle.decode(ov, oi, oracle.F16, M, K, B, k)
    for j in (0, 1, 31, 32, 33, 1023, 1024, 8191, 8192, K - 1):
        x = torch.zeros(K, dtype=torch.float16)
        x[j] = 1
        y = bs.spmv(A, x.cuda())
        np.testing.assert_array_equal(oracle.to_double(synth.to_numpy(y), oracle.F16), Wd[:, j])


def test_row_sharding_bit_identical(bs):
    """Rows packed and multiplied in P slices concatenate to the unsharded y bit for bit (O-9)."""
    M, K, B, k = 1000, 25088, 32, 3
    W = synth.matrix(M, K, "f16", seed=44).cuda()
    x = synth.vector(K, "f16", seed=45).cuda()
    vals, idx, _ = bs.prune(W, B, k=k)
    y1 = bs.spmv(bs.pack(vals, idx, K, B), x)
    from paper_1811_00206_b200.dist import row_range
    for P in (2, 3, 8):
        parts = []
        for r in range(P):
            r0, r1 = row_range(M, P, r)
            Ws = synth.matrix(r1 - r0, K, "f16", seed=44, row0=r0).cuda()  # regenerated slice
            v, i, _ = bs.prune(Ws, B, k=k)
            parts.append(bs.spmv(bs.pack(v, i, K, B), x))
        assert torch.equal(torch.cat(parts), y1)


def test_spmv_launch_modes_and_dependencies(bs):
    """bs_spmv_ex flags (plain / PDL / PDL + static weights) give bit-identical y, and the PDL waits hold:
    a chain of layers where each x is the previous kernel's y, with ping-pong y buffers (a WAR hazard if
    y were written before the wait), and a pack immediately followed by a PDL SpMV that reads its output."""
    K, B, k = 4096, 32, 3
    dev = torch.device("cuda")
    mats = []
    for j in range(6):
        W = synth.matrix(K, K, "f16", seed=synth.seed_for(9, j), device=dev)
        v, i, _ = bs.prune(W, B, k=k)
        mats.append(bs.pack(v, i, K, B))
    x0 = synth.vector(K, "f16", seed=synth.seed_for(9, 99), device=dev)
    modes = (0, bs.SPMV_PDL, bs.SPMV_PDL | bs.SPMV_W_STATIC)
    outs = []
    for f in modes:
        ping, pong = torch.empty(K, dtype=torch.float16, device=dev), torch.empty(K, dtype=torch.float16, device=dev)
        cur = x0.clone()
        for rep in range(3):
            for j, A in enumerate(mats):
                dst = ping if (rep * len(mats) + j) % 2 == 0 else pong
                bs.spmv(A, cur, out=dst, flags=f)
                cur = dst
                cur.mul_(1.0 / 16)  # a torch kernel between layers (writes x of the next SpMV)
        torch.cuda.synchronize()
        outs.append(cur.clone())
    assert torch.isfinite(outs[0].float()).all()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    # pack -> PDL SpMV (the SpMV's W reads must wait for the pack kernel)
    W = synth.matrix(700, K, "f16", seed=synth.seed_for(9, 50), device=dev)
    v, i, _ = bs.prune(W, B, k=k)
    ref = bs.spmv(bs.pack(v, i, K, B), x0, flags=0)
    for _ in range(3):
        A = bs.pack(v, i, K, B)
        assert torch.equal(bs.spmv(A, x0), ref)
    with pytest.raises(bs.BSError):
        bs.spmv(mats[0], x0, flags=8)


@pytest.mark.parametrize("act", ["none", "relu", "sigmoid", "tanh"])
@pytest.mark.parametrize("M,K,dname", [(300, 25088, "f16"), (257, 3008, "bf16"), (130, 4096, "f32"), (64, 64, "f32")])
def test_spmv_fused_epilogue(bs, M, K, dname, act):
    """bs_spmv_fused: y = act(W_bs·x + bias) against the fp64 oracle (Eq. 1 with its +B). Tolerance: the
    north-star tau times (sum|w||x| + |bias|) (every activation is 1-Lipschitz), plus one unit in the last
    place of D for the final rounding of a value that the bound does not scale (e.g. sigmoid(0) = 0.5)."""
    B = 32 if K % 32 == 0 and K > 64 else 16
    k = 3 if B == 32 else 8
    W = synth.matrix(M, K, dname, seed=synth.seed_for(8, M + K))
    vals, idx, ov, oi = _prune_parity(bs, W, dname, B, k)
    A = bs.pack(vals, idx, K, B)
    x = synth.vector(K, dname, seed=synth.seed_for(8, 1))
    bias = synth.vector(M, dname, seed=synth.seed_for(8, 2))
    y = bs.spmv(A, x.cuda(), bias=bias.cuda(), act=act)
    yr, bound = oracle.spmv_act(ov, oi, DT[dname], M, K, B, k, synth.to_numpy(x), synth.to_numpy(bias), act)
    ulp = {"f32": 2.0 ** -23, "f16": 2.0 ** -10, "bf16": 2.0 ** -7}[dname]
    err = np.abs(oracle.to_double(synth.to_numpy(y), DT[dname]) - yr)
    tol = oracle.TAU[DT[dname]] * bound + ulp * np.abs(yr) + 1e-6
    assert np.all(err <= tol), f"worst err/tol {float(np.max(err / tol)):.3g}"
    if act == "relu":
        assert (synth.to_numpy(y).astype(np.float32) >= 0).all()
    # no bias, no activation: bit-identical to bs_spmv; bias only: the same as act = none
    y0 = bs.spmv(A, x.cuda())
    y1 = bs.spmv(A, x.cuda(), act="none")
    assert torch.equal(y0, y1)


def test_spmv_fused_k0_and_errors(bs):
    """k = 0: W_bs = 0, so y = act(bias); SP24 has no fused epilogue; unknown activations are rejected."""
    M, K, B = 100, 640, 32
    W = synth.matrix(M, K, "f16", seed=71).cuda()
    v, i, _ = bs.prune(W, B, k=0)
    A = bs.pack(v, i, K, B)
    x = synth.vector(K, "f16", seed=72).cuda()
    bias = synth.vector(M, "f16", seed=73).cuda()
    y = bs.spmv(A, x, bias=bias, act="tanh")
    ref = torch.tanh(bias.float())
    assert torch.allclose(y.float(), ref, atol=2e-3, rtol=0)
    W4 = synth.matrix(64, 256, "f16", seed=74).cuda()
    v4, i4, _ = bs.prune(W4, 4, k=2)
    A4 = bs.pack(v4, i4, 256, 4, layout="sp24")
    with pytest.raises(bs.BSError):
        bs.spmv(A4, synth.vector(256, "f16", seed=75).cuda(), act="relu")
    with pytest.raises(ValueError):
        bs.spmv(A, x, act="gelu")


@pytest.mark.parametrize("N", [1, 2, 3, 8, 13, 32, 64])
@pytest.mark.parametrize("dname", ["f16", "bf16", "f32"])
def test_spmm_small(bs, N, dname):
    M, K, B, k = 77, 3072 + 96, 32, 4
    W = synth.matrix(M, K, dname, seed=46)
    X = synth.vector(K, dname, seed=47, n=N)
    vals, idx, ov, oi = _prune_parity(bs, W, dname, B, k)
    for layout in ("spmm", "spmv"):
        A = bs.pack(vals, idx, K, B, layout=layout)
        Y = bs.spmm(A, X.cuda())
        Yr, bound = oracle.spmm(ov, oi, DT[dname], M, K, B, k, synth.to_numpy(X))
        ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(Y), DT[dname]), Yr, bound, oracle.TAU[DT[dname]])
        assert ok, f"{layout} N={N}: worst {worst}"


def test_spmm_column_independence(bs):
    """Column n of Y does not depend on N (batch sharding is bit-identical)."""
    M, K, B, k = 200, 4096, 32, 4
    W = synth.matrix(M, K, "f16", seed=48).cuda()
    X = synth.vector(K, "f16", seed=49, n=64).cuda()
    vals, idx, _ = bs.prune(W, B, k=k)
    A = bs.pack(vals, idx, K, B, layout="spmm")
    Y64 = bs.spmm(A, X)
    for n0, n1 in ((0, 1), (5, 13), (8, 40), (63, 64)):
        assert torch.equal(bs.spmm(A, X[n0:n1].contiguous()), Y64[n0:n1])


@pytest.mark.parametrize("K,N", [(2048, 16), (1024, 13), (3008, 12), (2048, 40)])
def test_spmm_spmv_layout_sixteen_wide(bs, K, N):
    """Passes of 16 columns (32-byte x slots, CTC-sized K) give the same columns bit for bit as passes of
    8 and 1, and match the oracle."""
    M, B, k = 333, 32, 4
    W = synth.matrix(M, K, "bf16", seed=synth.seed_for(9, 400 + K))
    X = synth.vector(K, "bf16", seed=synth.seed_for(9, 401), n=N)
    vals, idx, ov, oi = _prune_parity(bs, W, "bf16", B, k)
    A = bs.pack(vals, idx, K, B, layout="spmv")
    Xd = X.cuda()
    Y = bs.spmm(A, Xd)
    for n0, n1 in ((0, 8), (8, N), (N - 1, N)):
        assert torch.equal(bs.spmm(A, Xd[n0:n1].contiguous()), Y[n0:n1]), (n0, n1)
    Yr, bound = oracle.spmm(ov, oi, oracle.BF16, M, K, B, k, synth.to_numpy(X))
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(Y), oracle.BF16), Yr, bound, oracle.TAU[oracle.BF16])
    assert ok, worst


def test_spmm_spmv_layout_pass_widths(bs):
    """SPMV-layout SpMM: passes of 1..8 columns (x slots NV = 2, 4, 8) share one K-chunking, so column
    n is bit-identical for every N (K spans several x chunks plus a tail), and matches the oracle."""
    M, K, B, k = 150, 16384 + 32 * 40, 32, 3
    W = synth.matrix(M, K, "f16", seed=64)
    X = synth.vector(K, "f16", seed=65, n=13)
    vals, idx, ov, oi = _prune_parity(bs, W, "f16", B, k)
    A = bs.pack(vals, idx, K, B, layout="spmv")
    Xd = X.cuda()
    Y13 = bs.spmm(A, Xd)
    for n0, n1 in ((0, 1), (3, 5), (5, 9), (9, 12), (12, 13), (0, 8)):
        assert torch.equal(bs.spmm(A, Xd[n0:n1].contiguous()), Y13[n0:n1]), (n0, n1)
    Yr, bound = oracle.spmm(ov, oi, oracle.F16, M, K, B, k, synth.to_numpy(X))
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(Y13), oracle.F16), Yr, bound, oracle.TAU[oracle.F16])
    assert ok, worst


@pytest.mark.parametrize("M", [77, 700, 4096 + 33, 9800])
def test_spmm_tc_split_k(bs, M):
    """K6 split-K over a cluster: S = min(8, SMs / tiles, chunks / 6) (1 tile -> 5, 6 -> 5, 33 -> 4,
    77 -> 1 on 148 SMs with 33 chunks); every S matches the oracle, and columns stay independent of N."""
    K, B, k, N = 2048 + 32, 32, 4, 24
    W = synth.matrix(M, K, "bf16", seed=66)
    X = synth.vector(K, "bf16", seed=67, n=N)
    vals, idx, ov, oi = _prune_parity(bs, W, "bf16", B, k)
    A = bs.pack(vals, idx, K, B, layout="spmm")
    Xd = X.cuda()
    Y = bs.spmm(A, Xd)
    Yr, bound = oracle.spmm(ov, oi, oracle.BF16, M, K, B, k, synth.to_numpy(X))
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(Y), oracle.BF16), Yr, bound, oracle.TAU[oracle.BF16])
    assert ok, worst
    assert torch.equal(bs.spmm(A, Xd[7:8].contiguous()), Y[7:8])


def test_spmv_host_e2e(bs):
    M, K, B, k = 512, 4096, 32, 3
    W = synth.matrix(M, K, "f16", seed=50)
    x = synth.vector(K, "f16", seed=51)
    vals, idx, ov, oi = _prune_parity(bs, W, "f16", B, k)
    A = bs.pack(vals, idx, K, B)
    xh = x.pin_memory()
    yh = torch.empty(M, dtype=torch.float16).pin_memory()
    xd = torch.empty(K, dtype=torch.float16, device="cuda")
    yd = torch.empty(M, dtype=torch.float16, device="cuda")
    bs.spmv_host(A, xh, yh, xd, yd)
    torch.cuda.synchronize()
    assert torch.equal(yh, bs.spmv(A, x.cuda()).cpu())


def test_errors(bs):
    W = torch.zeros((4, 30), dtype=torch.float16, device="cuda")
    with pytest.raises(bs.BSError) as e:
        bs.prune(W, 16, k=4)
    assert e.value.status == bs.BS_ERR_SHAPE
    with pytest.raises(bs.BSError) as e:
        bs.prune(torch.zeros((4, 32), dtype=torch.float16, device="cuda"), 16, k=17)
    assert e.value.status == bs.BS_ERR_ARG
    v, i, _ = bs.prune(torch.zeros((4, 32), dtype=torch.float16, device="cuda"), 8, k=2)
    with pytest.raises(bs.BSError) as e:
        bs.pack(v, i, 32, 8, layout="sp24")
    assert e.value.status == bs.BS_ERR_UNSUPPORTED


# ---------------------------------------------------------------- full-size configs (BASELINE configs)

FULL = [
    ("ptb", 6000, 3008, 32, 3, "f16"),      # configs[1]: 6000x3000 padded to 3008 (A5)
    ("fc6", 4096, 25088, 32, 3, "f16"),     # configs[2]
    ("fc7", 4096, 4096, 32, 1, "bf16"),
    ("fc7f32", 4096, 4096, 32, 16, "f32"),
    ("ctc_ih", 4096, 2048, 32, 4, "f16"),   # configs[3], 87.5%
    ("ctc_hh", 4096, 1024, 32, 4, "f16"),
]


@pytest.mark.parametrize("name,M,K,B,k,dname", FULL)
def test_full_configs(bs, name, M, K, B, k, dname):
    W = synth.matrix(M, K, dname, seed=synth.seed_for(2, 0))
    x = synth.vector(K, dname, seed=synth.seed_for(2, 1))
    vals, idx, ov, oi = _prune_parity(bs, W, dname, B, k)
    A = bs.pack(vals, idx, K, B)
    np.testing.assert_array_equal(A.packed.cpu().numpy(), oracle.pack(ov, oi, M, K, B, k, DT[dname], oracle.SPMV))
    y = bs.spmv(A, x.cuda())
    yr, bound = oracle.spmv(ov, oi, DT[dname], M, K, B, k, synth.to_numpy(x))
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(y), DT[dname]), yr, bound, oracle.TAU[DT[dname]])
    assert ok, worst


def test_full_fc6_spmm32(bs):
    M, K, B, k, N = 4096, 25088, 32, 3, 32
    W = synth.matrix(M, K, "f16", seed=synth.seed_for(2, 2))
    X = synth.vector(K, "f16", seed=synth.seed_for(2, 3), n=N)
    vals, idx, _ = bs.prune(W.cuda(), B, k=k)
    A = bs.pack(vals, idx, K, B, layout="spmm")
    Y = bs.spmm(A, X.cuda())
    rows = np.random.default_rng(0).choice(M, 256, replace=False).astype(np.int64)
    ov, oi = synth.to_numpy(vals), _idx_np(idx)
    Yr, bound = oracle.spmm(ov, oi, oracle.F16, M, K, B, k, synth.to_numpy(X), rows=rows)
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(Y[:, rows].contiguous()), oracle.F16), Yr, bound, 1e-2)
    assert ok, worst


@pytest.mark.slow
def test_big_65536_sampled_rows(bs):
    """configs[4]: 65536x65536 at 90% (k = 3 of 32), exactly as bench.py runs it; checked on sampled rows."""
    M = K = 65536
    B, k = 32, 3
    W = synth.matrix(M, K, "f16", seed=synth.seed_for(4, 0), device="cuda")
    x = synth.vector(K, "f16", seed=synth.seed_for(4, 1), device="cuda")
    vals, idx, _ = bs.prune(W, B, k=k)
    A = bs.pack(vals, idx, K, B)
    y = bs.spmv(A, x)
    rng = np.random.default_rng(1)
    rows = np.unique(np.concatenate([rng.choice(M, 2048, replace=False), [0, M - 1, 8191, 8192, 32767, 32768]]))
    rt = torch.from_numpy(rows).cuda()
    Wr = synth.to_numpy(W[rt])
    ov, oi = oracle.prune(Wr, oracle.F16, B, k)
    np.testing.assert_array_equal(_idx_np(idx[rt]), oi)
    np.testing.assert_array_equal(_raw(vals[rt]), ov.view(np.uint16))
    yr, bound = oracle.spmv_rowslice(ov, oi, oracle.F16, K, B, k, synth.to_numpy(x))
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(y[rt]), oracle.F16), yr, bound, 1e-2)
    assert ok, worst


def test_big_fused_epilogue_sampled_rows(bs):
    """The fused layer at scale: 320000 x 4096 (2163 rows per CTA, more than the 4 bias rows per thread the
    kernel prefetches in registers), bias + ReLU, W_STATIC launch; checked on sampled rows against the
    oracle's SpMV plus the bias and the activation from their definitions."""
    M, K, B, k = 320000, 4096, 32, 3
    W = synth.matrix(M, K, "bf16", seed=synth.seed_for(7, 0), device="cuda")
    x = synth.vector(K, "bf16", seed=synth.seed_for(7, 1), device="cuda")
    b = synth.vector(M, "bf16", seed=synth.seed_for(7, 2), device="cuda")
    vals, idx, _ = bs.prune(W, B, k=k)
    A = bs.pack(vals, idx, K, B)
    y = bs.spmv(A, x, bias=b, act="relu", flags=bs.SPMV_PDL | bs.SPMV_W_STATIC)
    rng = np.random.default_rng(2)
    rows = np.unique(np.concatenate([rng.choice(M, 1500, replace=False), [0, 2162, 2163, 2164, M - 1]]))
    rt = torch.from_numpy(rows).cuda()
    ov, oi = oracle.prune(synth.to_numpy(W[rt]), oracle.BF16, B, k)
    s_, bound = oracle.spmv_rowslice(ov, oi, oracle.BF16, K, B, k, synth.to_numpy(x))
    bb = oracle.to_double(synth.to_numpy(b[rt]), oracle.BF16)
    yr = np.array([oracle.act(v, "relu") for v in s_ + bb])
    err = np.abs(oracle.to_double(synth.to_numpy(y[rt]), oracle.BF16) - yr)
    assert np.all(err <= 1e-2 * (bound + np.abs(bb)) + 2.0 ** -7 * np.abs(yr) + 1e-6)


@pytest.mark.parametrize("case", range(24))
def test_random_shapes(bs, case):
    """Seeded random shapes across the parameter space (M, K = NB·B, B, k, dtype, family): prune masks and
    packed bytes bit-exact, SpMV and a small-batch SpMM within the north-star tolerance."""
    rng = np.random.default_rng(1000 + case)
    B = int(rng.choice([2, 4, 8, 16, 20, 25, 32, 64, 100, 300]))
    NB = int(rng.integers(1, 600)) if B <= 64 else int(rng.integers(1, 40))
    K, M = NB * B, int(rng.integers(1, 700))
    k = int(rng.integers(0, B + 1)) if case % 4 == 0 else int(rng.integers(1, max(2, B // 4 + 1)))
    dname = ["f16", "bf16", "f32"][case % 3]
    family = ["gaussian", "ties", "sameoffset"][case % 3 if B <= 64 else 0]
    W = synth.matrix(M, K, dname, family=family, seed=synth.seed_for(6, case), B=B)
    vals, idx, ov, oi = _prune_parity(bs, W, dname, B, k)
    A = bs.pack(vals, idx, K, B)
    np.testing.assert_array_equal(A.packed.cpu().numpy(), oracle.pack(ov, oi, M, K, B, k, DT[dname], oracle.SPMV))
    x = synth.vector(K, dname, seed=synth.seed_for(6, 100 + case))
    y = bs.spmv(A, x.cuda())
    yr, bound = oracle.spmv(ov, oi, DT[dname], M, K, B, k, synth.to_numpy(x))
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(y), DT[dname]), yr, bound, oracle.TAU[DT[dname]])
    assert ok, f"spmv worst {worst}"
    N = int(rng.integers(2, 12))
    X = synth.vector(K, dname, seed=synth.seed_for(6, 200 + case), n=N)
    Y = bs.spmm(A, X.cuda())
    Yr, Yb = oracle.spmm(ov, oi, DT[dname], M, K, B, k, synth.to_numpy(X))
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(Y), DT[dname]), Yr, Yb, oracle.TAU[DT[dname]])
    assert ok, f"spmm worst {worst}"


@pytest.mark.parametrize("B,k,N", [(32, 3, 1), (32, 3, 8), (32, 3, 32), (4, 2, 1), (4, 2, 48)])
def test_spmm_auto_layout(bs, B, k, N):
    """pack(layout="auto", batch=N) (bs_choose_layout) followed by bs_spmm, against the oracle."""
    M, K = 300, 2048
    W = synth.matrix(M, K, "f16", seed=synth.seed_for(9, 300 + N + B))
    vals, idx, ov, oi = _prune_parity(bs, W, "f16", B, k)
    A = bs.pack(vals, idx, K, B, layout="auto", batch=N)
    assert A.layout == bs.choose_layout(M, K, B, k, torch.float16, N)
    X = synth.vector(K, "f16", seed=synth.seed_for(9, 301), n=N)
    Y = bs.spmm(A, X.cuda())
    Yr, Yb = oracle.spmm(ov, oi, oracle.F16, M, K, B, k, synth.to_numpy(X))
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(Y), oracle.F16), Yr, Yb, 1e-2)
    assert ok, worst


@pytest.mark.parametrize("B,dname,family", [(32, "f16", "gaussian"), (16, "bf16", "ties"), (8, "f32", "gaussian"),
                                             (4, "f16", "ties"), (32, "f32", "ties"), (2, "bf16", "gaussian")])
def test_block_rank(bs, B, dname, family):
    """bs_block_rank equals the oracle's sort positions bit for bit, and rank < k is bs_prune's mask for a
    whole schedule of k (Alg. 1's gradual sparsity without retraining)."""
    M, K = 257, 64 * B
    W = synth.matrix(M, K, dname, family=family, seed=synth.seed_for(9, 500 + B), B=B)
    R = bs.block_rank(W.cuda(), B)
    np.testing.assert_array_equal(R.cpu().numpy(), oracle.block_rank(synth.to_numpy(W), DT[dname], B))
    for k in sorted({1, B // 4, B // 2, B - 1} - {0}):
        _, idx, _ = bs.prune(W.cuda(), B, k=k)
        mask = torch.zeros((M, K // B, B), dtype=torch.bool, device="cuda")
        mask.scatter_(2, idx.to(torch.int64), True)
        assert torch.equal(R.view(M, K // B, B) < k, mask)


def test_block_rank_special_values(bs):
    for dname in ("f32", "f16", "bf16"):
        W = synth.special_block_matrix(dname)
        R = bs.block_rank(W.cuda(), 16)
        np.testing.assert_array_equal(R.cpu().numpy(), oracle.block_rank(synth.to_numpy(W), DT[dname], 16))


# ---------------------------------------------------------------- 2:4 (B = 4, k = 2): SP24 layout

@pytest.mark.parametrize("N", [1, 2, 8, 16, 64, 200])
@pytest.mark.parametrize("dname", ["f16", "bf16"])
def test_sp24_spmm(bs, N, dname):
    """2:4 on the sparse tensor cores (N >= 2) and the CUDA-core path (N = 1) vs the oracle."""
    M, K = 300, 1024  # 3 row tiles (the last one partial), 8 chunks of 128 columns
    W = synth.matrix(M, K, dname, seed=60 + N)
    X = synth.vector(K, dname, seed=61, n=N)
    vals, idx, ov, oi = _prune_parity(bs, W, dname, 4, 2)
    A = bs.pack(vals, idx, K, 4, layout="sp24")
    np.testing.assert_array_equal(A.packed.cpu().numpy(), oracle.pack(ov, oi, M, K, 4, 2, DT[dname], oracle.SP24))
    Y = bs.spmm(A, X.cuda())
    Yr, bound = oracle.spmm(ov, oi, DT[dname], M, K, 4, 2, synth.to_numpy(X))
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(Y), DT[dname]), Yr, bound, 1e-2)
    assert ok, f"sp24 N={N}: worst {worst}"


@pytest.mark.parametrize("M", [130, 4096, 9600])
def test_sp24_split_k(bs, M):
    """K5 split-K clusters (33 chunks): S = 5 (2 tiles), 4 (32 tiles), 1 (75 tiles); oracle parity and
    N-independence."""
    K, N = 4096 + 128, 40
    W = synth.matrix(M, K, "f16", seed=68)
    X = synth.vector(K, "f16", seed=69, n=N)
    vals, idx, ov, oi = _prune_parity(bs, W, "f16", 4, 2)
    A = bs.pack(vals, idx, K, 4, layout="sp24")
    Xd = X.cuda()
    Y = bs.spmm(A, Xd)
    Yr, bound = oracle.spmm(ov, oi, oracle.F16, M, K, 4, 2, synth.to_numpy(X))
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(Y), oracle.F16), Yr, bound, 1e-2)
    assert ok, worst
    assert torch.equal(bs.spmm(A, Xd[3:5].contiguous()), Y[3:5])


def test_sp24_spmv_and_integer_exact(bs):
    M, K = 257, 2048
    W = synth.matrix(M, K, "f16", family="intexact", seed=62)
    X = synth.vector(K, "f16", family="intexact", seed=63, n=16)
    vals, idx, ov, oi = _prune_parity(bs, W, "f16", 4, 2)
    A = bs.pack(vals, idx, K, 4, layout="sp24")
    y = bs.spmv(A, X[0].contiguous().cuda())
    yr, _ = oracle.spmv(ov, oi, oracle.F16, M, K, 4, 2, synth.to_numpy(X[0].contiguous()))
    np.testing.assert_array_equal(oracle.to_double(synth.to_numpy(y), oracle.F16), yr)
    Y = bs.spmm(A, X.cuda())  # tensor cores, integer-exact: bit-identical
    Yr, _ = oracle.spmm(ov, oi, oracle.F16, M, K, 4, 2, synth.to_numpy(X))
    np.testing.assert_array_equal(oracle.to_double(synth.to_numpy(Y), oracle.F16), Yr)
