"""GPU parity of convolution as balanced-sparse SpMM (P:286 im2col, P:107 one weight
matrix per conv layer): bs_im2col is a pure copy (bit-exact vs orc_im2col), and conv2d = im2col + bs_spmm
matches the oracle's direct convolution within the north-star tolerance, bit for bit on integer-exact data.
The shapes are VGG-16 layers of Table cnn-perf at reduced spatial size, and the paper's
balanced sparsities for them."""
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


def _img(Nimg, H, W, C, dname, seed, family="gaussian"):
    return synth.vector(Nimg * H * W * C, dname, family=family, seed=seed).reshape(Nimg, H, W, C)


@pytest.mark.parametrize("Nimg,H,W,C,kh,kw,pad,stride,dname", [
    (2, 9, 7, 64, 3, 3, 1, 1, "f16"),     # vector path
    (1, 14, 14, 32, 3, 3, 1, 2, "bf16"),
    (3, 5, 6, 3, 3, 3, 1, 1, "f16"),      # C = 3 (conv1_1): scalar path
    (1, 6, 6, 4, 1, 1, 0, 1, "f32"),
    (1, 4, 4, 8, 5, 5, 2, 1, "f32"),      # kernel wider than the image core
])
def test_im2col_bit_exact(bs, Nimg, H, W, C, kh, kw, pad, stride, dname):
    inp = _img(Nimg, H, W, C, dname, synth.seed_for(50, C))
    X = bs.im2col(inp.cuda(), kh, kw, pad, stride)
    ref = oracle.im2col(synth.to_numpy(inp), DT[dname], kh, kw, pad, stride)
    got = synth.to_numpy(X)
    np.testing.assert_array_equal(got.view(np.uint8), ref.view(np.uint8))


@pytest.mark.parametrize("layer,Cout,C,HW,s,layout,dname", [
    ("conv4_2", 512, 512, 7, 0.91, "spmm", "f16"),   # Table cnn-perf: conv4_2 at 91% (28x28 in VGG; 7x7 here)
    ("conv5_2", 512, 512, 6, 0.90, "spmv", "bf16"),  # the CUDA-core batched path
    ("conv3_3", 256, 256, 8, 0.88, "spmm", "bf16"),
    ("conv2_2", 128, 128, 9, 0.5, "sp24", "f16"),    # 2:4 sparse tensor cores (B = 4, 50%)
])
def test_conv2d_matches_oracle(bs, layer, Cout, C, HW, s, layout, dname):
    kh = kw = 3
    Kc = kh * kw * C
    B = 4 if layout == "sp24" else 32
    k = bs.k_from_sparsity(B, s)
    Wm = synth.matrix(Cout, Kc, dname, seed=synth.seed_for(51, Cout + C))
    vals, idx, _ = bs.prune(Wm.cuda(), B, k=k)
    A = bs.pack(vals, idx, Kc, B, layout=layout)
    inp = _img(1, HW, HW, C, dname, synth.seed_for(51, 7))
    Y = bs.conv2d(A, inp.cuda(), kh, kw, pad=1, stride=1)
    assert Y.shape == (1, HW, HW, Cout)
    ov, oi = oracle.prune(synth.to_numpy(Wm), DT[dname], B, k)
    Yr, bound = oracle.conv2d(ov, oi, DT[dname], Cout, B, k, synth.to_numpy(inp), kh, kw, 1, 1)
    ok, worst = oracle.check_tolerance(oracle.to_double(synth.to_numpy(Y.reshape(-1, Cout)), DT[dname]), Yr, bound,
                                       oracle.TAU[DT[dname]])
    assert ok, f"{layer}: worst |err|/bound {worst}"


@pytest.mark.parametrize("layout", ["spmm", "spmv"])
def test_conv2d_integer_exact(bs, layout):
    """W, input in {-1, 0, 1}: the conv output equals the oracle's direct convolution bit for bit (stride 2,
    padding, 2 images)."""
    Cout, C, kh, kw, B, k = 128, 64, 3, 3, 32, 4
    Kc = kh * kw * C
    Wm = synth.matrix(Cout, Kc, "f16", family="intexact", seed=synth.seed_for(52, 0))
    vals, idx, _ = bs.prune(Wm.cuda(), B, k=k)
    A = bs.pack(vals, idx, Kc, B, layout=layout)
    inp = _img(2, 9, 8, C, "f16", synth.seed_for(52, 1), family="intexact")
    Y = bs.conv2d(A, inp.cuda(), kh, kw, pad=1, stride=2)
    ov, oi = oracle.prune(synth.to_numpy(Wm), oracle.F16, B, k)
    Yr, _ = oracle.conv2d(ov, oi, oracle.F16, Cout, B, k, synth.to_numpy(inp), kh, kw, 1, 2)
    np.testing.assert_array_equal(oracle.to_double(synth.to_numpy(Y.reshape(-1, Cout)), oracle.F16), Yr)


def test_conv_weight_matrix_matches_torch(bs):
    """conv_weight_matrix + im2col + a dense product reproduce torch's conv2d (layout bookkeeping only)."""
    w = torch.randn(6, 5, 3, 3, dtype=torch.float64)
    x = torch.randn(1, 5, 7, 7, dtype=torch.float64)
    ref = torch.nn.functional.conv2d(x, w, padding=1).permute(0, 2, 3, 1).reshape(-1, 6)
    Wm = bs.conv_weight_matrix(w)
    X = torch.from_numpy(oracle.im2col(x.permute(0, 2, 3, 1).contiguous().float().numpy(), oracle.F32, 3, 3, 1, 1)).double()
    assert torch.allclose(X @ Wm.T, ref, atol=1e-5)


@pytest.mark.parametrize("Nimg,H,W,C,Cout,kh,kw,pad,dname,B,s", [
    (1, 8, 8, 256, 256, 3, 3, 1, "f16", 32, 0.88),    # conv3_3-like
    (2, 7, 5, 64, 128, 3, 3, 1, "bf16", 32, 0.9),     # two images: pixel columns run across the image border
    (1, 14, 14, 512, 512, 3, 3, 1, "f16", 16, 0.75),  # B = 16, conv4_x width
    (1, 9, 6, 128, 64, 3, 1, 1, "f16", 32, 0.9),      # kh != kw: corner and filter-offset order
    (1, 5, 5, 64, 32, 1, 1, 0, "bf16", 32, 0.5),      # 1x1
    (3, 4, 4, 64, 200, 5, 5, 2, "f16", 32, 0.9),      # 5x5, pad 2, ragged Cout
])
def test_conv2d_implicit_im2col_matches_explicit(bs, Nimg, H, W, C, Cout, kh, kw, pad, dname, B, s):
    """bs_conv2d (X tiles loaded by TMA in im2col mode straight from the NHWC input) against bs_im2col +
    bs_spmm on the same matrix: the same X values reach the same MMAs in the same order, so the outputs
    are bit-identical; and against the oracle's direct convolution on integer-exact data, bit for bit."""
    Kc = kh * kw * C
    k = bs.k_from_sparsity(B, s)
    Wm = synth.matrix(Cout, Kc, dname, seed=synth.seed_for(53, Cout + C + kh))
    vals, idx, _ = bs.prune(Wm.cuda(), B, k=k)
    A = bs.pack(vals, idx, Kc, B, layout="spmm")
    inp = _img(Nimg, H, W, C, dname, synth.seed_for(53, 9)).cuda()
    Yi = bs.conv2d(A, inp, kh, kw, pad=pad, implicit=True)
    Ye = bs.conv2d(A, inp, kh, kw, pad=pad, implicit=False)
    assert torch.equal(Yi, Ye)
    Wi = synth.matrix(Cout, Kc, dname, family="intexact", seed=synth.seed_for(53, 1))
    vi, ii, _ = bs.prune(Wi.cuda(), B, k=k)
    Ai = bs.pack(vi, ii, Kc, B, layout="spmm")
    xi = _img(Nimg, H, W, C, dname, synth.seed_for(53, 2), family="intexact")
    Y = bs.conv2d(Ai, xi.cuda(), kh, kw, pad=pad, implicit=True)
    ov, oi = oracle.prune(synth.to_numpy(Wi), DT[dname], B, k)
    ref, _ = oracle.conv2d(ov, oi, DT[dname], Cout, B, k, synth.to_numpy(xi), kh, kw, pad, 1)
    np.testing.assert_array_equal(oracle.to_double(synth.to_numpy(Y), DT[dname]).reshape(ref.shape), ref)


def test_conv2d_implicit_errors(bs):
    Wm = synth.matrix(64, 9 * 32, "f16", seed=5).cuda()
    v, i, _ = bs.prune(Wm, 32, k=3)
    inp = _img(1, 6, 6, 32, "f16", 6).cuda()
    with pytest.raises(bs.BSError):   # C % 64 != 0: not eligible when forced
        bs.conv2d(bs.pack(v, i, 9 * 32, 32, layout="spmm"), inp, 3, 3, pad=1, implicit=True)
    Y = bs.conv2d(bs.pack(v, i, 9 * 32, 32, layout="spmm"), inp, 3, 3, pad=1)  # auto: falls back to im2col
    assert Y.shape == (1, 6, 6, 64)
    W2 = synth.matrix(64, 9 * 64, "f16", seed=7).cuda()
    v2, i2, _ = bs.prune(W2, 32, k=3)
    A2 = bs.pack(v2, i2, 9 * 64, 32, layout="spmm")
    x2 = _img(1, 8, 8, 64, "f16", 8).cuda()
    with pytest.raises(bs.BSError):   # stride 2: only the explicit path
        bs.conv2d(A2, x2, 3, 3, pad=1, stride=2, implicit=True)
    assert bs.conv2d(A2, x2, 3, 3, pad=1, stride=2).shape == (1, 4, 4, 64)
    with pytest.raises(ValueError):   # bias of the wrong length
        bs.conv2d(A2, x2, 3, 3, pad=1, bias=torch.zeros(63, dtype=torch.float16, device="cuda"))
    with pytest.raises(ValueError):   # unknown activation
        bs.conv2d(A2, x2, 3, 3, pad=1, act="gelu")


@pytest.mark.parametrize("act,dname", [("relu", "f16"), ("tanh", "bf16"), ("sigmoid", "f16")])
def test_conv2d_fused_bias_act(bs, act, dname):
    """bs_conv2d's layer epilogue: act(conv + bias) in fp32 before the one rounding (Eq. 1's +B),
    against the oracle's direct convolution + bias + act in fp64: bit-exact for ReLU on integer-exact data,
    within the conv bound (the activations are 1-Lipschitz) plus one rounding otherwise."""
    Nimg, H, W, C, Cout, B = 1, 6, 7, 64, 96, 32
    Kc = 9 * C
    k = 3
    fam = "intexact" if act == "relu" else "gaussian"
    Wm = synth.matrix(Cout, Kc, dname, family=fam, seed=synth.seed_for(54, 1))
    vals, idx, _ = bs.prune(Wm.cuda(), B, k=k)
    A = bs.pack(vals, idx, Kc, B, layout="spmm")
    xi = _img(Nimg, H, W, C, dname, synth.seed_for(54, 2), family=fam)
    bias = synth.vector(Cout, dname, family=fam, seed=synth.seed_for(54, 3))
    Y = bs.conv2d(A, xi.cuda(), 3, 3, pad=1, bias=bias.cuda(), act=act)
    ov, oi = oracle.prune(synth.to_numpy(Wm), DT[dname], B, k)
    ref, bound = oracle.conv2d(ov, oi, DT[dname], Cout, B, k, synth.to_numpy(xi), 3, 3, 1, 1)
    b = oracle.to_double(synth.to_numpy(bias), DT[dname])
    want = np.vectorize(lambda v: oracle.act(v, act))(ref + b[None, :])
    got = oracle.to_double(synth.to_numpy(Y), DT[dname]).reshape(want.shape)
    if act == "relu":
        np.testing.assert_array_equal(got, want)
    else:
        ulp = 2.0 ** (-10 if dname == "f16" else -7)
        assert np.all(np.abs(got - want) <= 1e-2 * (bound + np.abs(b)[None, :]) + ulp * np.abs(want) + 1e-6)
    with pytest.raises(ValueError):
        bs.conv2d(A, xi.cuda(), 3, 3, pad=1, bias=bias.cuda(), act=act, implicit=False)


@pytest.mark.parametrize("Nimg,H,W,C,Cout,kh,kw,pad", [
    (1, 8, 8, 128, 256, 3, 3, 1),    # K5 single-CTA kernel with split-K
    (2, 5, 5, 64, 9728, 2, 2, 0),    # >= 75 row tiles: K5 CTA pairs (each CTA loads its half of the pixel column)
])
def test_conv2d_implicit_im2col_sp24(bs, Nimg, H, W, C, Cout, kh, kw, pad):
    """bs_conv2d on the 2:4 layout (K5 with TMA im2col loads of each 64-channel atom): bit-identical to
    bs_im2col + bs_spmm, and with bias + ReLU exact against the oracle on integer-exact data."""
    Kc = kh * kw * C
    Wm = synth.matrix(Cout, Kc, "f16", family="intexact", seed=synth.seed_for(55, Cout))
    vals, idx, _ = bs.prune(Wm.cuda(), 4, k=2)
    A = bs.pack(vals, idx, Kc, 4, layout="sp24")
    xi = _img(Nimg, H, W, C, "f16", synth.seed_for(55, 2), family="intexact")
    Yi = bs.conv2d(A, xi.cuda(), kh, kw, pad=pad, implicit=True)
    Ye = bs.conv2d(A, xi.cuda(), kh, kw, pad=pad, implicit=False)
    assert torch.equal(Yi, Ye)
    bias = synth.vector(Cout, "f16", family="intexact", seed=synth.seed_for(55, 3))
    Y = bs.conv2d(A, xi.cuda(), kh, kw, pad=pad, bias=bias.cuda(), act="relu")
    ov, oi = oracle.prune(synth.to_numpy(Wm), oracle.F16, 4, 2)
    ref, _ = oracle.conv2d(ov, oi, oracle.F16, Cout, 4, 2, synth.to_numpy(xi), kh, kw, pad, 1)
    b = oracle.to_double(synth.to_numpy(bias), oracle.F16)
    np.testing.assert_array_equal(oracle.to_double(synth.to_numpy(Y), oracle.F16).reshape(ref.shape),
                                  np.maximum(ref + b[None, :], 0.0))
