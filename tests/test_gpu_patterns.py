"""GPU parity of Alg. 1's dense pruned matrix and schedule, and of the comparison sparsity patterns
(SURVEY §8(f) NEXT-4), against the fp64 oracle. Every result is an integer decision, so the bar is bit
for bit: the dense M_p (bs_decode after bs_prune_k), the random-sparsity mask (bs_random_mask) and the
block / vector masks (bs_block_mask).

Cites: Alg. 1 P:116-140 (GraduallyIncrease P:131), random sparsity P:39/P:274, block sparsity
P:40/P:275 and Table brange (4×4, 8×8, 16×16 tiles; balance ranges 25/50/100), vector sparsity P:40.
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


def _raw(a: np.ndarray) -> np.ndarray:
    return a.view(np.uint32 if a.itemsize == 4 else np.uint16)


@pytest.mark.parametrize("M,K,B,k,dname,family", [
    (64, 64, 16, 8, "f32", "gaussian"),
    (37, 3000, 25, 8, "f16", "gaussian"),     # Table brange balance range 25, 3000-wide PTB rows
    (20, 3000, 50, 6, "bf16", "ties"),
    (9, 3000, 100, 10, "f16", "ties"),
    (33, 8192 + 32, 32, 3, "bf16", "gaussian"),  # segments of 4096 with a ragged last one
    (5, 8192, 8192, 819, "f16", "gaussian"),     # one block per row (row-wise reduction, A8)
    (17, 96, 4, 2, "f32", "ties"),
    (11, 640, 32, 0, "f16", "gaussian"),         # k = 0: all zeros
    (8, 256, 16, 16, "bf16", "gaussian"),        # k = B: W itself
])
def test_prune_dense_matches_oracle(bs, M, K, B, k, dname, family):
    W = synth.matrix(M, K, dname, family=family, seed=synth.seed_for(30, M + K + B))
    ref = oracle.prune_dense(synth.to_numpy(W), DT[dname], B, k)
    P = bs.prune_dense(W.cuda(), B, k=k)
    np.testing.assert_array_equal(_raw(synth.to_numpy(P)), _raw(ref))
    # into a padded destination, and in place
    buf = torch.full((M, K + 24), 7.0, dtype=W.dtype, device="cuda")
    bs.prune_dense(W.cuda(), B, k=k, out=buf[:, :K])
    np.testing.assert_array_equal(_raw(synth.to_numpy(buf[:, :K].contiguous())), _raw(ref))
    assert torch.all(buf[:, K:] == 7.0)
    Wc = W.cuda()
    bs.prune_dense(Wc, B, k=k, out=Wc)
    np.testing.assert_array_equal(_raw(synth.to_numpy(Wc)), _raw(ref))


def test_prune_dense_special_values(bs):
    for dname in ("f32", "f16", "bf16"):
        W = synth.special_block_matrix(dname)
        for k in (1, 5, 9, 16):
            ref = oracle.prune_dense(synth.to_numpy(W), DT[dname], 16, k)
            np.testing.assert_array_equal(_raw(synth.to_numpy(bs.prune_dense(W.cuda(), 16, k=k))), _raw(ref))


def test_gradual_prune_schedule(bs):
    """Alg. 1 without retraining on the GPU: iteration i prunes M_p at k_i = lround((1 - s_i)·B) along
    the cubic schedule; the k sequence and every intermediate M_p equal the oracle's, and the end point
    equals one step at the target (nesting). With a retraining callback that rescales the
    survivors, the result still has exactly k_n nonzeros per block."""
    M, K, B, target, n = 48, 4096, 32, 0.9, 10
    W = synth.matrix(M, K, "f16", seed=synth.seed_for(31, 0))
    P, ks = bs.gradual_prune(W.cuda(), B, target, n)
    cur = synth.to_numpy(W)
    for i in range(1, n + 1):
        k = oracle.k_from_sparsity(B, oracle.schedule(target, n, i))
        assert ks[i - 1] == k
        cur = oracle.prune_dense(cur, oracle.F16, B, k)
    np.testing.assert_array_equal(_raw(synth.to_numpy(P)), _raw(cur))
    np.testing.assert_array_equal(_raw(cur), _raw(oracle.prune_dense(synth.to_numpy(W), oracle.F16, B, 3)))
    calls = []

    def retrain(Wp):
        calls.append(1)
        Wp.mul_(1.5)

    P2, _ = bs.gradual_prune(W.cuda(), B, target, n, retrain=retrain)
    assert len(calls) == n
    nz = (P2 != 0).view(M, K // B, B).sum(-1)
    assert torch.all(nz <= 3) and torch.all(nz == (P != 0).view(M, K // B, B).sum(-1))


@pytest.mark.parametrize("M,K,dname,family", [(300, 1000, "f16", "gaussian"), (128, 777, "f32", "gaussian"),
                                              (200, 512, "bf16", "ties"), (64, 4096, "f16", "ties")])
@pytest.mark.parametrize("s", [0.0, 0.5, 0.9, 0.97])
def test_random_mask_matches_oracle(bs, M, K, dname, family, s):
    W = synth.matrix(M, K, dname, family=family, seed=synth.seed_for(32, M + K))
    ref = oracle.random_mask(synth.to_numpy(W), DT[dname], s)
    got = bs.random_mask(W.cuda(), s).cpu().numpy()
    assert got.sum() == oracle.keep_count(M * K, s)
    np.testing.assert_array_equal(got, ref)


def test_random_mask_strided_and_special(bs):
    W = synth.matrix(40, 300, "f32", seed=synth.seed_for(32, 1), ld=320)
    W[3, 7] = float("nan")
    W[5, 1] = float("inf")
    W[6, 2] = float("-inf")
    Wd = W.cuda()[:, :300]
    for s in (0.2, 0.999):
        ref = oracle.random_mask(synth.to_numpy(W[:, :300].contiguous()), oracle.F32, s)
        np.testing.assert_array_equal(bs.random_mask(Wd, s).cpu().numpy(), ref)


def test_random_mask_large(bs):
    """2048 × 4096 f16 (8 M elements, several CTAs of equal-key ranges): bit-exact at 90%."""
    W = synth.matrix(2048, 4096, "f16", family="ties", seed=synth.seed_for(32, 2))
    ref = oracle.random_mask(synth.to_numpy(W), oracle.F16, 0.9)
    np.testing.assert_array_equal(bs.random_mask(W.cuda(), 0.9).cpu().numpy(), ref)


@pytest.mark.parametrize("bh,bw", [(4, 4), (8, 8), (16, 16), (2, 32)])
@pytest.mark.parametrize("criterion", ["max", "mean"])
@pytest.mark.parametrize("dname,family", [("f16", "gaussian"), ("bf16", "ties"), ("f32", "gaussian")])
def test_block_mask_matches_oracle(bs, bh, bw, criterion, dname, family):
    M, K = 256, 512
    W = synth.matrix(M, K, dname, family=family, seed=synth.seed_for(33, bh * bw))
    for s in (0.6, 0.8, 0.9):  # Table brange sparsities 60/70/80% and the paper's 90%
        ref = oracle.block_mask(synth.to_numpy(W), DT[dname], bh, bw, s, criterion)
        np.testing.assert_array_equal(bs.block_mask(W.cuda(), bh, bw, s, criterion).cpu().numpy(), ref)


@pytest.mark.parametrize("axis", ["row", "col"])
def test_vector_mask_matches_oracle(bs, axis):
    M, K = 96, 640
    W = synth.matrix(M, K, "f16", seed=synth.seed_for(34, 0))
    for s in (0.25, 0.5, 0.9):
        bh, bw = (1, K) if axis == "row" else (M, 1)
        ref = oracle.block_mask(synth.to_numpy(W), oracle.F16, bh, bw, s, "mean")
        got = bs.vector_mask(W.cuda(), s, axis).cpu().numpy()
        np.testing.assert_array_equal(got, ref)


def test_pattern_errors(bs):
    W = synth.matrix(30, 64, "f16", seed=1).cuda()
    with pytest.raises(bs.BSError):
        bs.block_mask(W, 4, 8, 0.5)  # 30 % 4 != 0
    with pytest.raises(bs.BSError):
        bs.random_mask(W, 1.0)
    with pytest.raises(KeyError):
        bs.block_mask(W, 2, 8, 0.5, "median")
