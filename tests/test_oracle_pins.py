"""Pins for the fp64 oracle (oracle/oracle.c) against what the paper and the mathematics fix.

These are CPU-only tests. Each pin is chosen so that a plausible mistake in the oracle fails at
least one of them: a dropped term, a wrong sign or index, a transposed operand, the wrong tie-break
or the wrong rounding. Citations: P:n = PAPER.md line, S:n = SPEC.md line.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _key(v: float):
    """Magnitude key of docs/layout.md: NaN above everything (all NaNs equal), else |v|."""
    return (1, 0.0) if math.isnan(v) else (0, abs(v))


# ------------------------------------------------------------------ k (A1)

def test_k_paper_instances():
    for B, s, k, cite in _gold("paper_k.json")["cases"]:
        assert oracle.k_from_sparsity(B, s) == k, cite


def test_k_invalid():
    assert oracle.k_from_sparsity(32, 1.0) == -1
    assert oracle.k_from_sparsity(32, -0.1) == -1
    assert oracle.k_from_sparsity(0, 0.5) == -1
    assert oracle.k_from_sparsity(32, float("nan")) == -1
    assert oracle.k_from_sparsity(32, 0.0) == 32


# ------------------------------------------------------------------ prune (Alg. 1 step)

def test_prune_spec_example_S143():
    g = _gold("spec_examples.json")["prune_S143"]
    W = np.array([g["row"]], dtype=np.float32)
    k = oracle.k_from_sparsity(g["block"], g["sparsity"])
    vals, idx = oracle.prune(W, oracle.F32, g["block"], k)
    assert idx[0].tolist() == g["kept_idx"]
    np.testing.assert_array_equal(vals[0], np.array(g["kept_vals"], dtype=np.float32))


def test_encode_example_S59():
    g = _gold("spec_examples.json")["encode_S59"]
    W = np.array([g["row"]], dtype=np.float32)
    vals, idx = oracle.prune(W, oracle.F32, g["block"], g["k"])
    assert idx[0].tolist() == g["idx"]
    assert vals[0].tolist() == g["vals"]


def test_prune_fig2_shape():
    """a 16-wide row in 4 blocks of 4 at 50% leaves 2 per block, and the same split applies to every row."""
    W = synth.to_numpy(synth.matrix(3, 16, "f32", seed=5))
    vals, idx = oracle.prune(W, oracle.F32, 4, 2)
    assert vals.shape == (3, 4, 2) and idx.shape == (3, 4, 2)
    assert np.all(idx[..., 0] < idx[..., 1])


def _brute_force_keep(block_vals, k):
    """The unique k-subset S with: for kept i and dropped j, key_i > key_j, or key_i == key_j and i < j.
    Enumerates all C(B, k) subsets (SURVEY §8(c) selection pin (i))."""
    B = len(block_vals)
    keys = [_key(float(v)) for v in block_vals]
    winners = []
    for S in itertools.combinations(range(B), k):
        Sset = set(S)
        ok = True
        for i in S:
            for j in range(B):
                if j in Sset:
                    continue
                if keys[i] > keys[j] or (keys[i] == keys[j] and i < j):
                    continue
                ok = False
                break
            if not ok:
                break
        if ok:
            winners.append(S)
    assert len(winners) == 1, "exactly one subset must satisfy the ordering"
    return list(winners[0])


@pytest.mark.parametrize("B", [4, 6, 8, 12, 16])
@pytest.mark.parametrize("family", ["gaussian", "ties"])
def test_prune_brute_force(B, family):
    K = 2 * B
    Wt = synth.matrix(3, K, "f16", family=family, seed=100 + B, B=B)
    W = synth.to_numpy(Wt)
    Wd = W.astype(np.float64)
    for k in range(0, B + 1):
        vals, idx = oracle.prune(W, oracle.F16, B, k)
        for r in range(3):
            for b in range(K // B):
                want = _brute_force_keep(Wd[r, b * B:(b + 1) * B], k)
                assert idx[r, b].tolist() == want
                np.testing.assert_array_equal(vals[r, b].view(np.uint16), W[r, b * B + np.array(want, dtype=int)].view(np.uint16))


def _rank_count_keep(W: np.ndarray, B: int, k: int) -> np.ndarray:
    """Independent vectorised rank count: keep j iff #{i: key_i > key_j} + #{i < j: key_i == key_j} < k.
    Returns a boolean mask. This is the second oracle of SURVEY §8(c) O-3."""
    M, K = W.shape
    x = W.astype(np.float64).reshape(M, K // B, B)
    nan = np.isnan(x)
    mag = np.where(nan, np.inf, np.abs(x))
    tier = nan.astype(np.int8)
    gt = (tier[..., :, None] > tier[..., None, :]) | ((tier[..., :, None] == tier[..., None, :]) & (mag[..., :, None] > mag[..., None, :]))
    eq = (tier[..., :, None] == tier[..., None, :]) & ((mag[..., :, None] == mag[..., None, :]) | (nan[..., :, None] & nan[..., None, :]))
    lower = np.arange(B)[:, None] < np.arange(B)[None, :]  # [i, j]: i < j
    rank = gt.sum(axis=-2) + (eq & lower).sum(axis=-2)  # count over i for each j
    return (rank < k).reshape(M, K)


def _mask_from_canonical(idx, M, K, B):
    mask = np.zeros((M, K), dtype=bool)
    NB = K // B
    for b in range(NB):
        cols = b * B + idx[:, b, :].astype(np.int64)
        np.put_along_axis(mask, cols, True, axis=1) if cols.size else None
    return mask


@pytest.mark.parametrize("dt,dname", [(oracle.F32, "f32"), (oracle.F16, "f16"), (oracle.BF16, "bf16")])
@pytest.mark.parametrize("B,k", [(16, 8), (32, 3), (32, 1), (32, 16), (4, 2), (25, 8), (64, 7)])
@pytest.mark.parametrize("family", ["gaussian", "ties"])
def test_prune_rank_count_agreement(dt, dname, B, k, family):
    M, K = 24, B * 6
    W = synth.to_numpy(synth.matrix(M, K, dname, family=family, seed=7 + B + k, B=B))
    vals, idx = oracle.prune(W, dt, B, k)
    want = _rank_count_keep(oracle.to_double(W, dt) if dt == oracle.BF16 else W, B, k)
    got = _mask_from_canonical(idx, M, K, B)
    np.testing.assert_array_equal(got, want)


def test_prune_special_values():
    """NaN ranks above +Inf, all NaNs tie (lower offset wins), ±0 tie, ±Inf tie."""
    W = synth.to_numpy(synth.special_block_matrix("f32"))
    vals, idx = oracle.prune(W, oracle.F32, 16, 4)
    want = _rank_count_keep(W, 16, 4)
    np.testing.assert_array_equal(_mask_from_canonical(idx, 4, 32, 16), want)
    # hand-derived: block (0,0) = [0,-0,1,-1,1,2,-2,.5,-.5,3,nan,.25,-inf,inf,0,1]
    assert idx[0, 0].tolist() == [9, 10, 12, 13]  # nan, -inf, inf, then 3.0
    # block (0,1) = [nan,nan,1,nan,-nan,0,0,5,-5,5,inf,-inf,inf,.1,.2,.3] -> the four NaNs
    assert idx[0, 1].tolist() == [0, 1, 3, 4]
    # all-equal block keeps offsets 0..k-1 (pin (vii))
    assert idx[1, 0].tolist() == [0, 1, 2, 3]
    # ±0 block: all tie -> 0..3
    assert idx[1, 1].tolist() == [0, 1, 2, 3]


def test_prune_rowwise_reduction():
    """B = K reduces balanced pruning to row-wise magnitude pruning with the same k (BJ.north_star; A8)."""
    M, K = 16, 96
    W = synth.to_numpy(synth.matrix(M, K, "f32", seed=11))
    for s in (0.5, 0.75, 0.9):
        k = oracle.k_from_sparsity(K, s)
        vals, idx = oracle.prune(W, oracle.F32, K, k)
        order = np.argsort(-np.abs(W.astype(np.float64)), axis=1, kind="stable")[:, :k]
        np.testing.assert_array_equal(idx[:, 0, :], np.sort(order, axis=1))


def test_prune_invariants_and_nesting():
    """Exactly k per block, strictly ascending offsets, nnz = M·NB·k, achieved sparsity = 1 - k/B (A7),
    per-block optimality, and nesting: kept(k') ⊆ kept(k) for k' ≤ k."""
    M, K, B = 20, 128, 32
    W = synth.to_numpy(synth.matrix(M, K, "f16", seed=13))
    masks = {}
    for k in range(B + 1):
        vals, idx = oracle.prune(W, oracle.F16, B, k)
        assert idx.shape == (M, K // B, k)
        if k > 1:
            assert np.all(np.diff(idx.astype(np.int64), axis=-1) > 0)
        m = _mask_from_canonical(idx, M, K, B)
        assert m.sum() == M * (K // B) * k
        assert 1 - m.sum() / (M * K) == pytest.approx(1 - k / B)
        # optimality: min kept |w| >= max dropped |w| in every block
        a = np.abs(W.astype(np.float64)).reshape(M, K // B, B)
        mb = m.reshape(M, K // B, B)
        if 0 < k < B:
            assert np.all(np.where(mb, a, np.inf).min(-1) >= np.where(mb, -np.inf, a).max(-1))
        masks[k] = m
    for k in range(B):
        assert np.all(masks[k] <= masks[k + 1])


def test_prune_sign_invariance():
    M, K, B = 8, 64, 16
    W = synth.to_numpy(synth.matrix(M, K, "f32", seed=17))
    v1, i1 = oracle.prune(W, oracle.F32, B, 5)
    v2, i2 = oracle.prune(-W, oracle.F32, B, 5)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(v1, -v2)


def test_prune_rejects_bad_shapes():
    W = np.zeros((2, 30), dtype=np.float32)
    with pytest.raises(ValueError):
        oracle.prune(W, oracle.F32, 16, 4)  # 30 mod 16 != 0
    with pytest.raises(ValueError):
        oracle.prune(np.zeros((2, 32), np.float32), oracle.F32, 16, 17)


# ------------------------------------------------------------------ element decoding

def test_half_decoder_all_patterns():
    """The oracle's own binary16 decoder agrees with numpy on all 65536 bit patterns (NaN as NaN)."""
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    want = bits.view(np.float16).astype(np.float64)
    got = oracle.to_double(bits.view(np.float16), oracle.F16)
    both_nan = np.isnan(want) & np.isnan(got)
    assert np.all(both_nan | (want == got))
    assert np.all(np.signbit(want[~np.isnan(want)]) == np.signbit(got[~np.isnan(want)]))


def test_bf16_decoder_sample():
    bits = np.arange(0, 65536, 7, dtype=np.uint32).astype(np.uint16)
    want = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()
    got = oracle.to_double(bits, oracle.BF16)
    assert np.all((np.isnan(want) & np.isnan(got)) | (want == got))


# ------------------------------------------------------------------ pack (docs/layout.md)

def test_packed_bytes_closed_form():
    """fc6 4096x25088, f16, B=32, k=3: NB = 784 = 3 panels of 256 blocks + a 16-block tail. Panel entries
    cost 2 + 5/8 bytes (5-bit index runs, docs/layout.md), tail entries 2 + 1; every region is 256-aligned.
    That is the algorithmic 2.625 B per nonzero of SURVEY §8(d) on the panels."""
    nnz = 4096 * 784 * 3
    panel, tail = 4096 * 768 * 3, 4096 * 16 * 3
    assert panel + tail == nnz
    assert oracle.packed_bytes(4096, 25088, 32, 3, oracle.F16, oracle.SPMV) == panel * 21 // 8 + 3 * tail == 25362432
    assert oracle.packed_bytes(4096, 25088, 32, 3, oracle.F32, oracle.SPMV) == 5 * nnz  # f32: V = 4, u8 indices
    # 65536², 90%: 402,653,184 nnz, all in panels -> 2.625 B each = 1,056,964,608 bytes
    assert oracle.packed_bytes(65536, 65536, 32, 3, oracle.F16, oracle.SPMV) == 65536 * 2048 * 3 * 21 // 8 == 1056964608
    # fc7 (NB = 128 -> V = 4): u8 indices, 3 B per nonzero
    assert oracle.packed_bytes(4096, 4096, 32, 3, oracle.F16, oracle.SPMV) == 3 * 4096 * 128 * 3
    # B <= 16 with NB >= 256 (V = 8) -> 4-bit index runs: 2.5 B per panel nonzero; NB = 128 (V = 4) -> u8
    assert oracle.packed_bytes(64, 4096, 16, 4, oracle.F16, oracle.SPMV) == 64 * 256 * 4 * 5 // 2
    assert oracle.packed_bytes(64, 2048, 8, 2, oracle.F16, oracle.SPMV) == 64 * 256 * 2 * 5 // 2
    assert oracle.packed_bytes(64, 2048, 16, 4, oracle.F16, oracle.SPMV) == 64 * 128 * 4 * 3
    # B > 256 -> u16 indices: 4 B per nnz at f16
    assert oracle.packed_bytes(64, 1024, 512, 8, oracle.F16, oracle.SPMV) == 4 * 64 * 2 * 8
    # SP24: K/2 values + K/8 metadata bytes per row
    assert oracle.packed_bytes(4096, 2048, 4, 2, oracle.F16, oracle.SP24) == 4096 * 1024 * 2 + 4096 * 256
    assert oracle.packed_bytes(4, 30, 4, 2, oracle.F16, oracle.SPMV) == 0  # 30 mod 4 != 0
    assert oracle.packed_bytes(4, 32, 8, 2, oracle.F16, oracle.SP24) == 0  # SP24 needs B=4,k=2


def test_pack_spmv_transpose_closed_form():
    """B=1, k=1, K=96, f16: NB=96 -> V=2, P=64, one full panel + a 32-block tail. The panel is the
    32×2 transpose of blocks 0..63 (lane l holds blocks l and 32+l); the tail is blocks 64..95 in order."""
    K = 96
    vals = np.arange(K, dtype=np.float16).reshape(1, K, 1)
    idx = np.zeros((1, K, 1), dtype=np.uint16)
    buf = oracle.pack(vals, idx, 1, K, 1, 1, oracle.F16, oracle.SPMV)
    va = buf[:128].view(np.float16)
    np.testing.assert_array_equal(va, np.arange(64, dtype=np.float16).reshape(2, 32).T.reshape(-1))
    vb = buf[256:256 + 64].view(np.float16)
    np.testing.assert_array_equal(vb, np.arange(64, 96, dtype=np.float16))


def test_pack_spmv_steps_closed_form():
    """f32, B=2, k=2 (dense), K=256: NB=128 -> V=4, P=128, one panel, T=0. The step t holds the t-th entry of
    every block, with lane l owning blocks l, 32+l, 64+l, 96+l (a 4×32 -> 32×4 transpose)."""
    K, B, k = 256, 2, 2
    blk = np.arange(128)
    vals = np.stack([blk * 10 + 0, blk * 10 + 1], axis=-1).astype(np.float32).reshape(1, 128, 2)
    idx = np.tile(np.array([0, 1], dtype=np.uint16), (1, 128, 1))
    buf = oracle.pack(vals, idx, 1, K, B, k, oracle.F32, oracle.SPMV)
    assert buf.size == 1280  # 2 steps x (128 values x 4 B + 128 indices x 1 B), 256-aligned
    for t in range(2):
        step = buf[t * 640:(t + 1) * 640]  # a step = its 128 values, then its 128 indices
        want = (blk.reshape(4, 32).T.reshape(-1) * 10 + t).astype(np.float32)
        np.testing.assert_array_equal(step[:512].view(np.float32), want)
        np.testing.assert_array_equal(step[512:], np.full(128, t, dtype=np.uint8))


def test_pack_spmv_four_bit_runs_closed_form():
    """B=16, f16, K=4096: NB=256 -> V=8, one panel, k=1. Block b keeps offset (5b+3) mod 16 with value b.
    The step is 256 values (lane-major transpose), then lane l's 32-bit word sum_v idx(v*32+l) << 4v as
    32 little-endian u32 words (docs/layout.md), 640 bytes in all, padded to 768."""
    K, B, NB = 4096, 16, 256
    blk = np.arange(NB)
    vals = blk.astype(np.float16).reshape(1, NB, 1)
    offs = (5 * blk + 3) % 16
    buf = oracle.pack(vals, offs.astype(np.uint16).reshape(1, NB, 1), 1, K, B, 1, oracle.F16, oracle.SPMV)
    assert buf.size == 768
    np.testing.assert_array_equal(buf[:512].view(np.float16), blk.reshape(8, 32).T.reshape(-1).astype(np.float16))
    words = buf[512:640].view("<u4")
    for l in range(32):
        want = sum(int(offs[v * 32 + l]) << (4 * v) for v in range(8))
        assert int(words[l]) == want, l
    assert not buf[640:].any()


def test_pack_spmv_five_bit_runs_closed_form():
    """B=32, f16, K=8192: NB=256 -> V=8, one panel, k=1. Block b keeps offset (7b+3) mod 32 with value b.
    The step is 256 values (lane-major transpose), then lane l's 40-bit field sum_v idx(v*32+l) << 5v as
    32 u32 words and 32 bytes (docs/layout.md), 672 bytes in all, padded to 768."""
    K, B, NB = 8192, 32, 256
    blk = np.arange(NB)
    vals = blk.astype(np.float16).reshape(1, NB, 1)
    offs = (7 * blk + 3) % 32
    idx = offs.astype(np.uint16).reshape(1, NB, 1)
    buf = oracle.pack(vals, idx, 1, K, B, 1, oracle.F16, oracle.SPMV)
    assert buf.size == 768
    np.testing.assert_array_equal(buf[:512].view(np.float16), blk.reshape(8, 32).T.reshape(-1).astype(np.float16))
    words = buf[512:640].view("<u4")
    tops = buf[640:672]
    for lane in range(32):
        F = 0
        for v in range(8):
            F |= int(offs[v * 32 + lane]) << (5 * v)
        assert int(words[lane]) == F & 0xFFFFFFFF
        assert int(tops[lane]) == F >> 32
    assert not buf[672:].any()


def test_pack_spmm_blob_closed_form():
    """SPMM layout: M=130 rows -> tiles of 128 and 2; K=96, B=32 -> CB=2 blocks per chunk -> chunks of 2 and 1 blocks.
    Each blob lists (row, block, entry) values row-major, 16-byte padded, then the indices."""
    M, K, B, k = 130, 96, 32, 1
    NB = 3
    vals = np.arange(M * NB * k, dtype=np.float16).reshape(M, NB, k)
    idx = (np.arange(M * NB * k) % 32).astype(np.uint16).reshape(M, NB, k)
    buf = oracle.pack(vals, idx, M, K, B, k, oracle.F16, oracle.SPMM)
    p16 = lambda n: (n + 15) // 16 * 16
    blob = lambda mt, cb: p16(mt * cb * k * 2) + p16(mt * cb * k)
    tb = blob(128, 2) + blob(128, 1)
    assert buf.size == (tb + blob(2, 2) + blob(2, 1) + 255) // 256 * 256
    # tile 0, chunk 0: rows 0..127, blocks 0..1
    b00 = buf[:blob(128, 2)]
    np.testing.assert_array_equal(b00[:512].view(np.float16), vals[:128, 0:2, 0].reshape(-1))
    np.testing.assert_array_equal(b00[512:768], idx[:128, 0:2, 0].reshape(-1).astype(np.uint8))
    # tile 0, chunk 1: block 2 only
    b01 = buf[blob(128, 2):tb]
    np.testing.assert_array_equal(b01[:256].view(np.float16), vals[:128, 2, 0])
    # tile 1 (rows 128..129), chunk 1 (block 2): values then indices, each padded to 16 bytes
    b11 = buf[tb + blob(2, 2):tb + blob(2, 2) + blob(2, 1)]
    np.testing.assert_array_equal(b11[:4].view(np.float16), vals[128:, 2, 0])
    np.testing.assert_array_equal(b11[16:18], idx[128:, 2, 0].astype(np.uint8))


@pytest.mark.parametrize("layout", [oracle.SPMV, oracle.SPMM])
@pytest.mark.parametrize("M,K,B,k,dt,dname", [(5, 3008, 32, 3, oracle.F16, "f16"), (3, 1024, 16, 8, oracle.F32, "f32"),
                                               (2, 2048, 512, 9, oracle.BF16, "bf16"), (4, 64, 4, 2, oracle.F16, "f16"),
                                               (3, 8192 + 1024, 32, 3, oracle.BF16, "bf16"),
                                               (3, 4096 + 512, 16, 5, oracle.F16, "f16"),     # 4-bit runs + tail
                                               (2, 2048 + 64, 8, 3, oracle.BF16, "bf16")])    # 4-bit runs, B = 8
def test_pack_is_a_permutation(layout, M, K, B, k, dt, dname):
    """The packed value+index pairs are exactly the canonical multiset (no entry lost or duplicated)."""
    W = synth.to_numpy(synth.matrix(M, K, dname, seed=21))
    vals, idx = oracle.prune(W, dt, B, k)
    buf = oracle.pack(vals, idx, M, K, B, k, dt, layout)
    es = 4 if dt == oracle.F32 else 2
    isz = 1 if B <= 256 else 2
    n = M * (K // B) * k
    NB = K // B
    cv = vals.reshape(-1).view(np.uint32 if es == 4 else np.uint16).astype(np.uint64)
    ci = idx.reshape(-1).astype(np.uint64)
    if layout == oracle.SPMM:  # walk the blobs (all M < 128 here: one row tile)
        CB = -(-64 // B) if B <= 64 else 1
        p16 = lambda x: (x + 15) // 16 * 16
        off, vs, is_ = 0, [], []
        for c in range(-(-NB // CB)):
            cb = min(CB, NB - CB * c)
            nv = M * cb * k
            vs.append(buf[off:off + nv * es])
            is_.append(buf[off + p16(nv * es):off + p16(nv * es) + nv * isz])
            off += p16(nv * es) + p16(nv * isz)
        pv = np.concatenate(vs).view(np.uint32 if es == 4 else np.uint16).astype(np.uint64)
        pi = np.concatenate(is_).view(np.uint8 if isz == 1 else np.uint16).astype(np.uint64)
        np.testing.assert_array_equal(np.sort(pv << 16 | pi), np.sort(cv << 16 | ci))
        return
    vmax = 16 // es
    V = 1
    while V * 2 <= vmax and 64 * V <= NB:
        V *= 2
    P = 32 * V
    nA = M * (NB // P) * P * k
    nB = n - nA
    T = NB - (NB // P) * P
    a = lambda x: (x + 255) // 256 * 256
    five = B == 32 and V == 8
    four = B <= 16 and V == 8
    ri = 160 if five else 128 if four else P * isz                  # index run bytes per step
    nsteps = nA // P
    A = buf[:nsteps * (P * es + ri)].reshape(-1, P * es + ri)         # steps: P values then the index run
    offB = a(nsteps * (P * es + ri))
    offC = offB + a(nB * es)
    assert buf.size == offC + a(nB * isz)
    vraw = np.concatenate([A[:, :P * es].reshape(-1), buf[offB:offB + nB * es]])   # tail values (region B)
    assert T * M * k == nB
    pv = vraw.view(np.uint32 if es == 4 else np.uint16).astype(np.uint64)
    if five:  # 40-bit lane fields: u32 plane + byte plane; index v of lane l is bits 5v..5v+4
        F = A[:, P * es:P * es + 128].copy().view("<u4").astype(np.uint64) | (A[:, P * es + 128:].astype(np.uint64) << 32)
        ia = np.stack([(F >> (5 * v)) & 31 for v in range(8)], axis=-1).reshape(-1)  # (step, lane, v) = position l*V + v
        pi = np.concatenate([ia, buf[offC:offC + nB].astype(np.uint64)])
    elif four:  # 32-bit lane words; index v of lane l is bits 4v..4v+3
        G = A[:, P * es:].copy().view("<u4").astype(np.uint64)
        ia = np.stack([(G >> (4 * v)) & 15 for v in range(8)], axis=-1).reshape(-1)
        pi = np.concatenate([ia, buf[offC:offC + nB].astype(np.uint64)])
    else:
        iraw = np.concatenate([A[:, P * es:].reshape(-1), buf[offC:offC + nB * isz]])  # tail indices (region C)
        pi = iraw.view(np.uint8 if isz == 1 else np.uint16).astype(np.uint64)
    cv = vals.reshape(-1).view(np.uint32 if es == 4 else np.uint16).astype(np.uint64)
    ci = idx.reshape(-1).astype(np.uint64)
    np.testing.assert_array_equal(np.sort(pv << 16 | pi), np.sort(cv << 16 | ci))


def test_pack_sp24_metadata():
    """SP24 (B=4, k=2): values in canonical order; each nibble is idx0 | idx1<<2 with idx0 < idx1 (6 legal patterns)."""
    M, K = 6, 64
    W = synth.to_numpy(synth.matrix(M, K, "f16", seed=23))
    vals, idx = oracle.prune(W, oracle.F16, 4, 2)
    buf = oracle.pack(vals, idx, M, K, 4, 2, oracle.F16, oracle.SP24)
    np.testing.assert_array_equal(buf[:M * K].view(np.float16).reshape(vals.shape), vals)
    meta = buf[256 * ((M * K + 255) // 256):][:M * K // 8]
    nib = np.stack([meta & 0xF, meta >> 4], axis=-1).reshape(M, K // 4)
    legal = {0 | 1 << 2, 0 | 2 << 2, 0 | 3 << 2, 1 | 2 << 2, 1 | 3 << 2, 2 | 3 << 2}
    assert set(np.unique(nib).tolist()) <= legal
    np.testing.assert_array_equal(nib & 3, idx[..., 0])
    np.testing.assert_array_equal(nib >> 2, idx[..., 1])


# ------------------------------------------------------------------ products (Eq. 1)

def test_spmv_spec_example_S249():
    g = _gold("spec_examples.json")["spmv_S249"]
    W = np.array([g["row"]], dtype=np.float32)
    vals, idx = oracle.prune(W, oracle.F32, g["block"], g["k"])
    y, bound = oracle.spmv(vals, idx, oracle.F32, 1, 8, g["block"], g["k"], np.array(g["x"], dtype=np.float32))
    assert y[0] == g["y"] and bound[0] == 2 * 2 + 1 * 7


def test_spmv_k0_is_zero():
    """k = 0 gives W_bs = 0 and y = 0."""
    W = synth.to_numpy(synth.matrix(4, 64, "f32"))
    vals, idx = oracle.prune(W, oracle.F32, 16, 0)
    y, bound = oracle.spmv(vals, idx, oracle.F32, 4, 64, 16, 0, np.ones(64, np.float32))
    assert np.all(y == 0) and np.all(bound == 0)


def test_spmv_dense_case_equals_gemv():
    """k = B (s = 0) leaves W unchanged, so y is the dense GEMV. Compared with numpy's fp64 matmul."""
    M, K = 12, 96
    W = synth.to_numpy(synth.matrix(M, K, "f32", seed=3))
    x = synth.to_numpy(synth.vector(K, "f32", seed=4))
    vals, idx = oracle.prune(W, oracle.F32, 32, 32)
    y, _ = oracle.spmv(vals, idx, oracle.F32, M, K, 32, 32, x)
    np.testing.assert_allclose(y, W.astype(np.float64) @ x.astype(np.float64), rtol=1e-13, atol=1e-15)


def test_spmv_unit_vector_extracts_column():
    """x = e_j gives y = column j of W_bs exactly (pin (iii)); it catches transposed operands and wrong offsets."""
    M, K, B, k = 10, 64, 16, 5
    W = synth.to_numpy(synth.matrix(M, K, "f16", seed=8))
    vals, idx = oracle.prune(W, oracle.F16, B, k)
    Wd = oracle.decode(vals, idx, oracle.F16, M, K, B, k)
    for j in (0, 1, 15, 16, 37, 63):
        x = np.zeros(K, np.float16)
        x[j] = 1
        y, _ = oracle.spmv(vals, idx, oracle.F16, M, K, B, k, x)
        np.testing.assert_array_equal(y, Wd[:, j])
        kept = np.zeros(M, bool)
        for r in range(M):
            kept[r] = (j % B) in idx[r, j // B].tolist()
        np.testing.assert_array_equal(y != 0, kept & (W[:, j] != 0))


def test_spmv_integer_exact():
    """W, x in {-1,0,1}: y is an exact integer, checked against Python-int arithmetic on the mask (pin (ii))."""
    M, K, B, k = 16, 256, 32, 7
    W = synth.to_numpy(synth.matrix(M, K, "f16", family="intexact", seed=9))
    x = synth.to_numpy(synth.vector(K, "f16", family="intexact", seed=10))
    vals, idx = oracle.prune(W, oracle.F16, B, k)
    y, _ = oracle.spmv(vals, idx, oracle.F16, M, K, B, k, x)
    mask = _rank_count_keep(W, B, k)
    Wi = W.astype(np.int64) * mask
    want = [sum(int(Wi[r, c]) * int(x[c]) for c in range(K)) for r in range(M)]
    assert y.tolist() == [float(v) for v in want]


def test_spmv_sparse_form_equals_dense_masked():
    """Sum over canonical entries == dense-masked W_bs·x (O-7), up to fp64 rounding."""
    M, K, B, k = 32, 512, 32, 3
    W = synth.to_numpy(synth.matrix(M, K, "bf16", seed=12))
    x = synth.to_numpy(synth.vector(K, "bf16", seed=13))
    vals, idx = oracle.prune(W, oracle.BF16, B, k)
    y, bound = oracle.spmv(vals, idx, oracle.BF16, M, K, B, k, x)
    Wd = oracle.decode(vals, idx, oracle.BF16, M, K, B, k)
    yd = oracle.gemv_dense(Wd, oracle.to_double(x, oracle.BF16))
    assert np.all(np.abs(y - yd) <= 1e-12 * bound)
    assert np.all(bound >= np.abs(y))


def test_spmv_row_sampling():
    M, K, B, k = 40, 256, 32, 4
    W = synth.to_numpy(synth.matrix(M, K, "f16", seed=14))
    x = synth.to_numpy(synth.vector(K, "f16", seed=15))
    vals, idx = oracle.prune(W, oracle.F16, B, k)
    y, b = oracle.spmv(vals, idx, oracle.F16, M, K, B, k, x)
    rows = np.array([39, 0, 17], dtype=np.int64)
    ys, bs = oracle.spmv(vals, idx, oracle.F16, M, K, B, k, x, rows=rows)
    np.testing.assert_array_equal(ys, y[rows])
    y2, _ = oracle.spmv_rowslice(vals[rows], idx[rows], oracle.F16, K, B, k, x)
    np.testing.assert_array_equal(y2, y[rows])


def test_spmm_identity_and_columns():
    """X = I gives Y[n][r] = W_bs[r][n], and every column equals SpMV of that column."""
    M, K, B, k = 9, 32, 8, 3
    W = synth.to_numpy(synth.matrix(M, K, "f32", seed=16))
    vals, idx = oracle.prune(W, oracle.F32, B, k)
    Wd = oracle.decode(vals, idx, oracle.F32, M, K, B, k)
    Y, _ = oracle.spmm(vals, idx, oracle.F32, M, K, B, k, np.eye(K, dtype=np.float32))
    np.testing.assert_array_equal(Y, Wd.T)
    X = synth.to_numpy(synth.vector(K, "f32", n=5, seed=17))
    Y, _ = oracle.spmm(vals, idx, oracle.F32, M, K, B, k, X)
    for n in range(5):
        y, _ = oracle.spmv(vals, idx, oracle.F32, M, K, B, k, np.ascontiguousarray(X[n]))
        np.testing.assert_array_equal(Y[n], y)
    rows = np.array([8, 2], dtype=np.int64)
    Yr, _ = oracle.spmm(vals, idx, oracle.F32, M, K, B, k, X, rows=rows)
    np.testing.assert_array_equal(Yr, Y[:, rows])


def test_ideal_time_S531():
    g = _gold("spec_examples.json")["ideal_time_S531"]
    assert oracle.ideal_time(g["d_time"], g["o_time"], g["sparsity"]) == pytest.approx(g["i_time"], abs=1e-12)
    assert oracle.ideal_time(50.0, 10.0, 0.0) == 50.0  # s = 0 -> dense time


# ------------------------------------------------------------------ layer epilogue (Eq. 1's +B, NEXT-2)

def test_act_closed_forms():
    """The activations at points where they have exact closed forms: sigmoid(0) = 1/2, sigmoid(ln 3) = 3/4,
    tanh(ln 2) = 3/5, tanh(-ln 3) = -4/5, ReLU on both signs; tanh is odd; sigmoid(v) + sigmoid(-v) = 1."""
    import math
    assert oracle.act(0.0, "sigmoid") == 0.5
    assert abs(oracle.act(math.log(3.0), "sigmoid") - 0.75) < 1e-15
    assert abs(oracle.act(math.log(2.0), "tanh") - 0.6) < 1e-15
    assert abs(oracle.act(-math.log(3.0), "tanh") + 0.8) < 1e-15
    assert oracle.act(-2.5, "relu") == 0.0 and oracle.act(2.5, "relu") == 2.5 and oracle.act(0.0, "relu") == 0.0
    assert oracle.act(-7.25, "none") == -7.25
    for v in (0.1, 1.7, 5.0, 30.0):
        assert oracle.act(-v, "tanh") == -oracle.act(v, "tanh")
        assert abs(oracle.act(v, "sigmoid") + oracle.act(-v, "sigmoid") - 1.0) < 1e-15
    assert oracle.act(40.0, "tanh") == 1.0 and oracle.act(-40.0, "tanh") == -1.0


def test_spmv_act_structure():
    """act = none with a bias is the plain SpMV plus the bias; ReLU is the positive part of that; with
    x = 0 the layer output is act(bias) for every activation; bound grows by |bias|."""
    M, K, B, k = 24, 512, 32, 3
    W = synth.to_numpy(synth.matrix(M, K, "f32", seed=61))
    vals, idx = oracle.prune(W, oracle.F32, B, k)
    x = synth.to_numpy(synth.vector(K, "f32", seed=62))
    bias = synth.to_numpy(synth.vector(M, "f32", seed=63))
    y0, b0 = oracle.spmv(vals, idx, oracle.F32, M, K, B, k, x)
    y1, b1 = oracle.spmv_act(vals, idx, oracle.F32, M, K, B, k, x, bias, "none")
    np.testing.assert_array_equal(y1, y0 + bias.astype(np.float64))
    np.testing.assert_array_equal(b1, b0 + np.abs(bias.astype(np.float64)))
    yr, _ = oracle.spmv_act(vals, idx, oracle.F32, M, K, B, k, x, bias, "relu")
    np.testing.assert_array_equal(yr, np.maximum(y1, 0.0))
    assert (yr == 0).any() and (yr > 0).any()
    yn, _ = oracle.spmv_act(vals, idx, oracle.F32, M, K, B, k, x, None, "none")
    np.testing.assert_array_equal(yn, y0)
    z = np.zeros(K, dtype=np.float32)
    for name in ("relu", "sigmoid", "tanh"):
        yz, _ = oracle.spmv_act(vals, idx, oracle.F32, M, K, B, k, z, bias, name)
        np.testing.assert_array_equal(yz, [oracle.act(float(b), name) for b in bias.astype(np.float64)])


# ------------------------------------------------------------------ block ranks (the mask schedule, NEXT-4)

@pytest.mark.parametrize("B,family", [(4, "ties"), (8, "gaussian"), (16, "ties"), (32, "gaussian")])
def test_block_rank_brute_force(B, family):
    """rank_j = #{i : |w_i| > |w_j|} + #{i < j : |w_i| = |w_j|} per block, counted directly in numpy (not
    by sorting); every block's ranks are a permutation of 0..B-1; rank < k is exactly orc_prune's mask."""
    M, K = 6, 4 * B
    W = synth.to_numpy(synth.matrix(M, K, "f32", family=family, seed=90 + B, B=B))
    R = oracle.block_rank(W, oracle.F32, B)
    A = np.abs(W.astype(np.float64)).reshape(M, K // B, B)
    gt = (A[..., None, :] > A[..., :, None]).sum(-1)
    eq_before = np.tril(A[..., None, :] == A[..., :, None], -1).sum(-1)
    np.testing.assert_array_equal(R.reshape(M, K // B, B), gt + eq_before)
    assert (np.sort(R.reshape(-1, B), axis=1) == np.arange(B)).all()
    for k in (0, 1, B // 2, B):
        vals, idx = oracle.prune(W, oracle.F32, B, k)
        mask = np.zeros((M, K // B, B), dtype=bool)
        for r in range(M):
            for b in range(K // B):
                mask[r, b, idx[r, b]] = True
        np.testing.assert_array_equal(R.reshape(M, K // B, B) < k, mask)


# ------------------------------------------------------------------ Alg. 1's outer loop and the comparison patterns (NEXT-4)

def test_schedule_S195_and_boundaries():
    g = _gold("spec_examples.json")["schedule_S195"]
    assert oracle.schedule(g["target"], g["n"], g["i"]) == pytest.approx(g["value"], abs=1e-15)
    for target in (0.5, 0.9, 0.97):
        for n in (1, 3, 10, 37):
            assert oracle.schedule(target, n, 0) == 0.0
            assert oracle.schedule(target, n, n) == pytest.approx(target, abs=1e-15)
    for bad in ((0.9, 0, 0), (0.9, 10, 11), (0.9, 10, -1), (1.0, 10, 3), (-0.1, 10, 3)):
        assert oracle.schedule(*bad) == -1.0


def test_schedule_rate_decreases():
    """increased from 0 to the target "while the increase rate decreases with pruning iteration"."""
    for target, n in ((0.9, 10), (0.5, 7), (0.97, 25)):
        s = [oracle.schedule(target, n, i) for i in range(n + 1)]
        d = np.diff(s)
        assert np.all(d > 0)
        assert np.all(np.diff(d) < 0)


def _rank_count(Wn: np.ndarray, B: int) -> np.ndarray:
    """Independent rank count per block (not the oracle's sort): #{greater} + #{equal at a lower offset}."""
    M, K = Wn.shape
    mag = np.where(np.isnan(Wn), np.inf, np.abs(Wn)).reshape(M, K // B, B).astype(np.float64)
    nan = np.isnan(Wn).reshape(M, K // B, B)
    key = np.where(nan, 2.0, 1.0)  # NaN class above every number
    gt = (key[..., :, None] > key[..., None, :]) | ((key[..., :, None] == key[..., None, :]) & (mag[..., :, None] > mag[..., None, :]))
    eq = (key[..., :, None] == key[..., None, :]) & ((mag[..., :, None] == mag[..., None, :]) | nan[..., :, None])
    lower = np.arange(B)[:, None] < np.arange(B)[None, :]
    rank = gt.sum(axis=-2) + (eq & lower).sum(axis=-2)  # rank of j: count over i
    return rank.reshape(M, K)


@pytest.mark.parametrize("dname,family,B", [("f32", "gaussian", 16), ("f16", "ties", 8), ("bf16", "ties", 32)])
def test_prune_dense_against_rank_count(dname, family, B):
    """M_p: kept entries are bit copies, the rest +0; kept iff the independent rank count is < k."""
    dt = {"f32": oracle.F32, "f16": oracle.F16, "bf16": oracle.BF16}[dname]
    W = synth.to_numpy(synth.matrix(12, 4 * B, dname, family=family, seed=91))
    Wf = oracle.to_double(W, dt)
    rank = _rank_count(Wf, B)
    for k in (0, 1, B // 3, B - 1, B):
        P = oracle.prune_dense(W, dt, B, k)
        keep = rank < k
        raw = W.view(np.uint32 if W.itemsize == 4 else np.uint16)
        praw = P.view(raw.dtype)
        np.testing.assert_array_equal(praw[keep], raw[keep])
        assert np.all(praw[~keep] == 0)
        assert keep.reshape(12, 4, B).sum(-1).min() == k == keep.reshape(12, 4, B).sum(-1).max()


def test_gradual_schedule_without_retraining_nests():
    """Alg. 1 without retraining: each iteration prunes the previous M_p at k_i = lround((1 - s_i)·B);
    survivors shrink monotonically and the end point equals one step at the target."""
    B, target, n = 32, 0.9, 10
    W = synth.to_numpy(synth.matrix(20, 4 * B, "f16", seed=92))
    cur = W.copy()
    prev_keep = np.ones(W.shape, dtype=bool)
    for i in range(1, n + 1):
        k = oracle.k_from_sparsity(B, oracle.schedule(target, n, i))
        cur = oracle.prune_dense(cur, oracle.F16, B, k)
        keep = cur.view(np.uint16) != 0
        assert np.all(keep <= prev_keep)
        prev_keep = keep
    np.testing.assert_array_equal(cur.view(np.uint16), oracle.prune_dense(W, oracle.F16, B, 3).view(np.uint16))


def test_random_mask_S163():
    g = _gold("spec_examples.json")["random_S163"]
    W = np.array(g["W"], dtype=np.float32)
    for s, want in g["cases"]:
        np.testing.assert_array_equal(oracle.random_mask(W, oracle.F32, s), np.array(want, dtype=np.uint8))


@pytest.mark.parametrize("family,s", [("gaussian", 0.9), ("ties", 0.5), ("ties", 0.75), ("gaussian", 0.0)])
def test_random_mask_optimal_and_ties(family, s):
    """Exactly keep_count kept; no dropped magnitude exceeds a kept one; at the threshold magnitude the
    kept entries precede the dropped ones in row-major order."""
    W = synth.to_numpy(synth.matrix(17, 40, "f32", family=family, seed=93))
    m = oracle.random_mask(W, oracle.F32, s).reshape(-1).astype(bool)
    a = np.abs(W.reshape(-1).astype(np.float64))
    assert m.sum() == oracle.keep_count(W.size, s)
    if m.all():
        return
    T = a[m].min()
    assert a[~m].max() <= T
    eq = np.flatnonzero(a == T)
    kept_eq, drop_eq = eq[m[eq]], eq[~m[eq]]
    if kept_eq.size and drop_eq.size:
        assert kept_eq.max() < drop_eq.min()


def test_random_mask_one_row_is_balanced_with_block_K():
    """random pruning of a single row equals balanced pruning with one block of width K."""
    for family in ("gaussian", "ties"):
        W = synth.to_numpy(synth.matrix(1, 64, "f16", family=family, seed=94))
        for s in (0.5, 0.75, 0.9):
            k = oracle.k_from_sparsity(64, s)
            _, idx = oracle.prune(W, oracle.F16, 64, k)
            want = np.zeros((1, 64), dtype=np.uint8)
            want[0, idx.reshape(-1)] = 1
            np.testing.assert_array_equal(oracle.random_mask(W, oracle.F16, s), want)


def test_random_mask_sign_and_nan():
    W = synth.to_numpy(synth.matrix(9, 32, "f32", seed=95))
    np.testing.assert_array_equal(oracle.random_mask(W, oracle.F32, 0.8), oracle.random_mask(-W, oracle.F32, 0.8))
    W2 = W.copy()
    W2[3, 7] = np.nan
    W2[5, 1] = np.inf
    m = oracle.random_mask(W2, oracle.F32, 0.99)  # keep lround(0.01·288) = 3: NaN, Inf, then the largest
    assert m[3, 7] == 1 and m[5, 1] == 1 and m.sum() == 3


def test_block_mask_S172_S173():
    g = _gold("spec_examples.json")["block_S172"]
    W = np.array(g["W"], dtype=np.float32)
    np.testing.assert_array_equal(oracle.block_mask(W, oracle.F32, 2, 2, 0.5, "max"), np.array(g["max_keep"], dtype=np.uint8))
    W2 = np.array(g["meanmax_W"], dtype=np.float32)
    np.testing.assert_array_equal(oracle.block_mask(W2, oracle.F32, 2, 2, 0.5, "max"), np.array(g["meanmax_max"], dtype=np.uint8))
    np.testing.assert_array_equal(oracle.block_mask(W2, oracle.F32, 2, 2, 0.5, "mean"), np.array(g["meanmax_mean"], dtype=np.uint8))


def test_block_mask_tile_scores_brute_force():
    """Integer weights (exact tile sums): kept tiles are the keep_count best by (score desc, tile index
    asc), scored independently here with numpy; every element of a kept tile is kept."""
    M, K, bh, bw = 16, 48, 4, 8
    W = synth.to_numpy(synth.matrix(M, K, "f32", family="ties", seed=96))
    A = np.abs(W.astype(np.float64)).reshape(M // bh, bh, K // bw, bw)
    for crit, score in (("max", A.max(axis=(1, 3))), ("mean", A.sum(axis=(1, 3)))):
        for s in (0.25, 0.5, 0.9):
            m = oracle.block_mask(W, oracle.F32, bh, bw, s, crit)
            flat = score.reshape(-1)
            order = sorted(range(flat.size), key=lambda t: (-flat[t], t))
            keep = np.zeros(flat.size, dtype=np.uint8)
            keep[order[:oracle.keep_count(flat.size, s)]] = 1
            want = np.repeat(np.repeat(keep.reshape(M // bh, K // bw), bh, axis=0), bw, axis=1)
            np.testing.assert_array_equal(m, want, err_msg=f"{crit} s={s}")


def test_block_mask_unit_tiles_equal_random():
    """1×1 tiles with the max criterion score each element by |w|: the random-sparsity mask."""
    W = synth.to_numpy(synth.matrix(10, 24, "bf16", family="ties", seed=97))
    for s in (0.3, 0.8):
        np.testing.assert_array_equal(oracle.block_mask(W, oracle.BF16, 1, 1, s, "max"), oracle.random_mask(W, oracle.BF16, s))


def test_vector_mask_S181_and_transpose():
    g = _gold("spec_examples.json")["vector_S181"]
    W = np.array(g["W"], dtype=np.float32)
    m = oracle.block_mask(W, oracle.F32, 1, W.shape[1], g["sparsity"], "mean")
    np.testing.assert_array_equal(m[:, 0], np.array(g["row_keep"], dtype=np.uint8))
    assert np.all(m == m[:, :1])
    mt = oracle.block_mask(np.ascontiguousarray(W.T), oracle.F32, W.T.shape[0], 1, g["sparsity"], "mean")
    np.testing.assert_array_equal(mt, m.T)


def test_pattern_masks_reject_bad_shapes():
    W = np.zeros((6, 10), dtype=np.float32)
    with pytest.raises(ValueError):
        oracle.block_mask(W, oracle.F32, 4, 5, 0.5)
    with pytest.raises(ValueError):
        oracle.random_mask(W, oracle.F32, 1.0)
    assert oracle.keep_count(10, 0.9) == 1 and oracle.keep_count(100, 0.9) == 10 and oracle.keep_count(7, 0.5) == 4


# ------------------------------------------------------------------ LSTM step with balanced-sparse gates (NEXT-2)

def test_lstm_cell_matches_torch_lstmcell():
    """The LSTM step equals torch's LSTMCell (the library routine, in fp64) on the dense W_bs, after
    undoing the gate-row interleave (row 4j+g <-> PyTorch's block row g·H + j)."""
    In, H, B, k = 64, 48, 16, 5
    K = In + H
    W = synth.to_numpy(synth.matrix(4 * H, K, "f32", seed=101))
    vals, idx = oracle.prune(W, oracle.F32, B, k)
    Wd = oracle.decode(vals, idx, oracle.F32, 4 * H, K, B, k)
    x = synth.to_numpy(synth.vector(K, "f32", seed=102))
    bias = synth.to_numpy(synth.vector(4 * H, "f32", seed=103)) * np.float32(0.5)
    c_prev = synth.to_numpy(synth.vector(H, "f32", seed=104)).astype(np.float64)
    h, c, zb = oracle.lstm_cell(vals, idx, oracle.F32, 4 * H, K, B, k, x, None, bias, c_prev)
    perm = np.array([4 * j + g for g in range(4) for j in range(H)])  # PyTorch row g·H + j = our row 4j + g
    cell = torch.nn.LSTMCell(In, H).double()
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(Wd[perm, :In]))
        cell.weight_hh.copy_(torch.from_numpy(Wd[perm, In:]))
        cell.bias_ih.copy_(torch.from_numpy(bias.astype(np.float64)[perm]))
        cell.bias_hh.zero_()
        ht, ct = cell(torch.from_numpy(x[:In].astype(np.float64))[None], (torch.from_numpy(x[In:].astype(np.float64))[None],
                                                                        torch.from_numpy(c_prev)[None]))
    np.testing.assert_allclose(h, ht[0].numpy(), rtol=0, atol=1e-13)
    np.testing.assert_allclose(c, ct[0].numpy(), rtol=0, atol=1e-13)
    # pre (W_ih·x_t precomputed) + bias is the same as bias alone with pre folded in
    h2, c2, _ = oracle.lstm_cell(vals, idx, oracle.F32, 4 * H, K, B, k, x, bias, None, c_prev)
    np.testing.assert_array_equal(h2, h)
    assert np.all(zb >= 0)


def test_lstm_cell_closed_form():
    """k = 0: z = bias. z_i = 0, z_f = ln 3, z_g = ln 2, z_o = 0, c_prev = 1:
    c = 3/4 + 1/2·3/5 = 1.05 and h = tanh(1.05)/2."""
    H, K, B = 3, 32, 16
    vals = np.zeros((4 * H, K // B, 0), dtype=np.float32)
    idx = np.zeros((4 * H, K // B, 0), dtype=np.uint16)
    bias = np.tile(np.array([0.0, math.log(3.0), math.log(2.0), 0.0], dtype=np.float32), H)
    x = np.zeros(K, dtype=np.float32)
    h, c, _ = oracle.lstm_cell(vals, idx, oracle.F32, 4 * H, K, B, 0, x, None, bias, np.ones(H))
    f = 1.0 / (1.0 + math.exp(-float(np.float32(math.log(3.0)))))
    g = math.tanh(float(np.float32(math.log(2.0))))
    np.testing.assert_allclose(c, f + 0.5 * g, rtol=0, atol=1e-15)
    assert abs(c[0] - 1.05) < 1e-7 and abs(h[0] - math.tanh(1.05) / 2) < 1e-7
    np.testing.assert_allclose(h, 0.5 * np.tanh(c), rtol=0, atol=1e-15)


# ------------------------------------------------------------------ convolution via im2col (NEXT-3)

def _nhwc_weight_to_torch(Wd, Cout, C, kh, kw):
    """Our Cout × (kh·kw·C) matrix with (dy, dx, c) columns -> torch's [Cout][C][kh][kw]."""
    return Wd.reshape(Cout, kh, kw, C).transpose(0, 3, 1, 2)


@pytest.mark.parametrize("kh,kw,pad,stride", [(3, 3, 1, 1), (3, 3, 1, 2), (1, 1, 0, 1), (3, 3, 0, 1), (5, 3, 2, 2)])
def test_conv2d_matches_torch_conv2d(kh, kw, pad, stride):
    """orc_conv2d equals torch.nn.functional.conv2d (the library routine, fp64) on the dense W_bs, and
    the im2col route (orc_im2col, then the oracle's own SpMM) gives the same numbers."""
    Nimg, H, W, C, Cout, B, k = 2, 7, 6, 16, 12, 16, 5
    Kc = kh * kw * C
    Wm = synth.to_numpy(synth.matrix(Cout, Kc, "f32", seed=111))
    vals, idx = oracle.prune(Wm, oracle.F32, B, k)
    Wd = oracle.decode(vals, idx, oracle.F32, Cout, Kc, B, k)
    inp = synth.to_numpy(synth.vector(Nimg * H * W * C, "f32", seed=112)).reshape(Nimg, H, W, C)
    Y, bound = oracle.conv2d(vals, idx, oracle.F32, Cout, B, k, inp, kh, kw, pad, stride)
    ref = torch.nn.functional.conv2d(torch.from_numpy(inp.astype(np.float64)).permute(0, 3, 1, 2),
                                     torch.from_numpy(np.ascontiguousarray(_nhwc_weight_to_torch(Wd, Cout, C, kh, kw))),
                                     stride=stride, padding=pad)
    np.testing.assert_allclose(Y, ref.permute(0, 2, 3, 1).reshape(-1, Cout).numpy(), rtol=0, atol=1e-12)
    X = oracle.im2col(inp, oracle.F32, kh, kw, pad, stride)
    Y2, _ = oracle.spmm(vals, idx, oracle.F32, Cout, Kc, B, k, X)
    np.testing.assert_allclose(Y2, Y, rtol=0, atol=1e-12)
    assert np.all(bound >= np.abs(Y) - 1e-12)


def test_im2col_closed_forms():
    """1×1 / stride 1 / pad 0 im2col is the NHWC tensor itself (rows = pixels); a 3×3 pad-1 patch of an
    image holding its own coordinates reads the neighbours, and zeros past the border."""
    inp = np.arange(2 * 4 * 5 * 3, dtype=np.float32).reshape(2, 4, 5, 3)
    np.testing.assert_array_equal(oracle.im2col(inp, oracle.F32, 1, 1, 0, 1), inp.reshape(-1, 3))
    img = np.zeros((1, 3, 3, 2), dtype=np.float32)
    for y in range(3):
        for x in range(3):
            img[0, y, x] = [10 * y + x + 1, -(10 * y + x + 1)]
    X = oracle.im2col(img, oracle.F32, 3, 3, 1, 1)
    centre = X[4].reshape(3, 3, 2)  # output pixel (1, 1): the whole image
    np.testing.assert_array_equal(centre, img[0])
    corner = X[0].reshape(3, 3, 2)  # output pixel (0, 0): taps (dy, dx) read (dy - 1, dx - 1)
    assert np.all(corner[0] == 0) and np.all(corner[:, 0] == 0)
    np.testing.assert_array_equal(corner[1:, 1:], img[0, :2, :2])


def test_conv2d_identity_kernel():
    """A kernel with one 1 at the centre tap for co = c (B = kh·kw·C, k = 1 per row) reproduces the input
    (stride 1, pad 1)."""
    C, kh, kw = 4, 3, 3
    Kc = kh * kw * C
    Wm = np.zeros((C, Kc), dtype=np.float32)
    for c in range(C):
        Wm[c, (1 * kw + 1) * C + c] = 1.0
    vals, idx = oracle.prune(Wm, oracle.F32, Kc, 1)
    inp = synth.to_numpy(synth.vector(1 * 5 * 6 * C, "f32", seed=113)).reshape(1, 5, 6, C)
    Y, _ = oracle.conv2d(vals, idx, oracle.F32, C, Kc, 1, inp, kh, kw, 1, 1)
    np.testing.assert_array_equal(Y, inp.reshape(-1, C).astype(np.float64))
