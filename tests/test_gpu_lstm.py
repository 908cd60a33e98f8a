"""GPU parity of the fused LSTM step (bs_lstm_step: gate SpMV + cell in one kernel)
and of the time-batched layer (lstm_sequence: W_ih·X for all steps as one bs_spmm, NEXT-3) against the fp64
oracle (orc_lstm_cell).

Tolerance, derived from the arithmetic: each gate pre-activation z carries the north-star
error e_z = tau·(sum|w||x| + |pre| + |bias|) plus fp32 rounding of the additions. sigmoid' <= 1/4 and
tanh' <= 1, and every gate lies in [-1, 1], so
    |dc| <= |c_prev|·e_f/4 + e_i/4 + e_g + eps,        |dh| <= e_o/4 + |dc| + ulp_D(h) + eps,
with eps = 1e-5·(1 + |value|) for fp32 evaluation of exp/tanh. Over a sequence, an error dh in h_{t-1}
adds (sum_c |W_hh[r][c]|)·dh to every e_z of the next step; the test carries that bound forward.
Workloads: PTB's [W_ih | W_hh] 6000 x 3000 (BJ.configs[1], padded to 3008 per A5) and a Bi-LSTM
direction of TIMIT's CTC model, hidden 1024.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

DT = {"f32": oracle.F32, "f16": oracle.F16, "bf16": oracle.BF16}
TAU = {"f32": 1e-4, "f16": 1e-2, "bf16": 1e-2}
ULP = {"f32": 2.0 ** -23, "f16": 2.0 ** -10, "bf16": 2.0 ** -7}


@pytest.fixture(scope="module")
def bs():
    import paper_1811_00206_b200 as bs
    return bs


def _cell_tol(zb, zextra, c_prev_abs, c_prev_err, h_ref, c_ref, dname):
    """Per-unit bounds on |dc| and |dh| from per-gate-row error bounds e_z = tau·zb + zextra."""
    ez = TAU[dname] * zb + zextra + 1e-6 * (1 + zb)
    ei, ef, eg, eo = ez[0::4], ez[1::4], ez[2::4], ez[3::4]
    dc = c_prev_abs * ef / 4 + ei / 4 + eg + c_prev_err + 1e-5 * (1 + np.abs(c_ref))
    dh = eo / 4 + dc + ULP[dname] * np.maximum(np.abs(h_ref), 2.0 ** -14) + 1e-5 * (1 + np.abs(h_ref))
    return dc, dh


@pytest.mark.parametrize("H,In,B,k,dname,use_pre", [
    (1500, 1500, 32, 3, "f16", False),   # PTB: [W_ih | W_hh] = 6000 x 3000 -> 3008 (A5), 90%
    (1024, 1024, 32, 4, "bf16", True),   # TIMIT direction: W_hh 4096 x 1024 with pre = W_ih·x_t, 87.5%
    (64, 64, 16, 8, "f32", True),        # cfg0-sized, f32
    (37, 91, 4, 2, "f16", False),        # ragged: K = 128, 148 gate rows over many CTAs
])
def test_lstm_step_matches_oracle(bs, H, In, B, k, dname, use_pre):
    K = (H if use_pre else In + H)
    Kp = (K + B - 1) // B * B
    W = synth.matrix(4 * H, Kp, dname, seed=synth.seed_for(40, H + In))
    W[:, K:] = 0
    x = synth.vector(Kp, dname, seed=synth.seed_for(40, 1))
    x[K:] = 0
    bias = (synth.vector(4 * H, dname, seed=synth.seed_for(40, 2)).float() * 0.5).to(W.dtype)
    pre = (synth.vector(4 * H, dname, seed=synth.seed_for(40, 3)).float() * 0.5).to(W.dtype) if use_pre else None
    c_prev = synth.vector(H, "f32", seed=synth.seed_for(40, 4))
    vals, idx, _ = bs.prune(W.cuda(), B, k=k)
    A = bs.pack(vals, idx, Kp, B)
    h, c = bs.lstm_step(A, x.cuda(), c_prev.cuda(), pre=pre.cuda() if use_pre else None, bias=bias.cuda())
    # the direct kernel (half-warp gate rows, the cell after a CTA barrier) and the ring kernel agree bit for bit
    hR, cR = bs.lstm_step(A, x.cuda(), c_prev.cuda(), pre=pre.cuda() if use_pre else None, bias=bias.cuda(),
                          flags=bs.SPMV_PDL | bs.SPMV_RING)
    assert torch.equal(h, hR) and torch.equal(c, cR)
    ov, oi = oracle.prune(synth.to_numpy(W), DT[dname], B, k)
    hr, cr, zb = oracle.lstm_cell(ov, oi, DT[dname], 4 * H, Kp, B, k, synth.to_numpy(x),
                                  synth.to_numpy(pre) if use_pre else None, synth.to_numpy(bias), c_prev.numpy())
    dc, dh = _cell_tol(zb, 0.0, np.abs(c_prev.numpy().astype(np.float64)), 0.0, hr, cr, dname)
    cg = c.cpu().numpy().astype(np.float64)
    hg = oracle.to_double(synth.to_numpy(h), DT[dname])
    assert np.all(np.abs(cg - cr) <= dc), float(np.max(np.abs(cg - cr) / dc))
    assert np.all(np.abs(hg - hr) <= dh), float(np.max(np.abs(hg - hr) / dh))


def test_lstm_step_launch_modes_and_errors(bs):
    """The step gives the same bits with and without PDL; M mod 4 != 0, aliasing checks and the SPMM
    layout are rejected."""
    H, K, B, k = 256, 512, 32, 4
    W = synth.matrix(4 * H, K, "f16", seed=41).cuda()
    vals, idx, _ = bs.prune(W, B, k=k)
    A = bs.pack(vals, idx, K, B)
    x = synth.vector(K, "f16", seed=42).cuda()
    c0 = synth.vector(H, "f32", seed=43).cuda()
    h1, c1 = bs.lstm_step(A, x, c0, flags=0)
    h2, c2 = bs.lstm_step(A, x, c0, flags=bs.SPMV_PDL | bs.SPMV_W_STATIC)
    assert torch.equal(h1, h2) and torch.equal(c1, c2)
    # the direct warp-per-unit kernel and the streaming-ring kernel (cell in a CTA epilogue) agree bit for bit
    h3, c3 = bs.lstm_step(A, x, c0, flags=bs.SPMV_PDL | bs.SPMV_RING)
    assert torch.equal(h1, h3) and torch.equal(c1, c3)
    W3 = synth.matrix(6, K, "f16", seed=44).cuda()
    v3, i3, _ = bs.prune(W3, B, k=k)
    with pytest.raises(ValueError):
        bs.lstm_step(bs.pack(v3, i3, K, B), x, c0[:1])
    with pytest.raises(bs.BSError):
        bs.lstm_step(bs.pack(vals, idx, K, B, layout="spmm"), x, c0)
    with pytest.raises(ValueError):
        bs.lstm_step(A, x, c0.half())


def test_interleave_gates(bs):
    W = torch.arange(4 * 3 * 2).reshape(12, 2)
    Wi = bs.interleave_gates(W)
    for j in range(3):
        for g in range(4):
            assert torch.equal(Wi[4 * j + g], W[g * 3 + j])
    b = torch.arange(12)
    assert torch.equal(bs.interleave_gates(b), torch.tensor([0, 3, 6, 9, 1, 4, 7, 10, 2, 5, 8, 11]))


def test_lstm_sequence_matches_oracle(bs):
    """T steps: U = W_ih·X as one SpMM (N = T), then T fused steps on W_hh, against the fp64 oracle run
    step by step (its U and h rounded to f16 as the layer's outputs are), with the error bound carried
    through the recurrence."""
    T, In, H, B, k = 6, 256, 128, 32, 4
    Wih = synth.matrix(4 * H, In, "f16", seed=synth.seed_for(41, 0))
    Whh = synth.matrix(4 * H, H, "f16", seed=synth.seed_for(41, 1))
    X = synth.vector(In, "f16", seed=synth.seed_for(41, 2), n=T)
    bias = (synth.vector(4 * H, "f16", seed=synth.seed_for(41, 3)).float() * 0.5).half()
    h0 = (synth.vector(H, "f32", seed=synth.seed_for(41, 4)) * 0.5).half()
    c0 = synth.vector(H, "f32", seed=synth.seed_for(41, 5))
    vi, ii, _ = bs.prune(Wih.cuda(), B, k=k)
    vh, ih, _ = bs.prune(Whh.cuda(), B, k=k)
    A_ih = bs.pack(vi, ii, In, B, layout="spmv")
    A_hh = bs.pack(vh, ih, H, B)
    hs, cT = bs.lstm_sequence(A_ih, A_hh, X.cuda(), h0.cuda(), c0.cuda(), bias=bias.cuda())
    hs = hs.cpu()
    # oracle chain
    ovi, oii = oracle.prune(synth.to_numpy(Wih), oracle.F16, B, k)
    ovh, oih = oracle.prune(synth.to_numpy(Whh), oracle.F16, B, k)
    U, Ub = oracle.spmm(ovi, oii, oracle.F16, 4 * H, In, B, k, synth.to_numpy(X))
    Uh = U.astype(np.float16)  # the layer's U is f16 (bs_spmm's output dtype), rounded to nearest
    Whh_abs_rows = np.abs(oracle.decode(ovh, oih, oracle.F16, 4 * H, H, B, k)).sum(axis=1)
    h_prev, c_prev = synth.to_numpy(h0), c0.numpy().astype(np.float64)
    dh_prev, dc_prev = 0.0, 0.0
    for t in range(T):
        hr, cr, zb = oracle.lstm_cell(ovh, oih, oracle.F16, 4 * H, H, B, k, h_prev, Uh[t], synth.to_numpy(bias), c_prev)
        zextra = TAU["f16"] * Ub[t] + 2.0 ** -10 * np.abs(U[t]) + Whh_abs_rows * dh_prev
        dc, dh = _cell_tol(zb - np.abs(Uh[t].astype(np.float64)) + np.abs(U[t]), zextra, np.abs(c_prev), dc_prev, hr, cr, "f16")
        hg = hs[t].float().numpy().astype(np.float64)
        assert np.all(np.abs(hg - hr) <= dh), (t, float(np.max(np.abs(hg - hr) / dh)))
        h_prev, c_prev = hr.astype(np.float16), cr
        dh_prev, dc_prev = float(np.max(dh)) + 2.0 ** -10 * float(np.max(np.abs(hr))), dc
    assert np.all(np.abs(cT.cpu().numpy() - c_prev) <= dc_prev)


def test_layer_stack_graph(bs):
    """LayerStack (the VGG classifier head fc6 -> fc7 -> fc8 at Table cnn-perf's 93 % / 93 % / 75 %, as one
    CUDA graph) gives exactly the eager chain of bs_spmv_fused calls, replay after replay."""
    dims = [(512, 2048, 2, "relu"), (512, 512, 2, "relu"), (128, 512, 8, None)]
    layers = []
    for j, (M, K, k, act) in enumerate(dims):
        W = synth.matrix(M, K, "f16", seed=synth.seed_for(42, j)).cuda()
        v, i, _ = bs.prune(W, 32, k=k)
        b = synth.vector(M, "f16", seed=synth.seed_for(42, 10 + j)).cuda()
        layers.append((bs.pack(v, i, K, 32), b, act))
    x = synth.vector(2048, "f16", seed=synth.seed_for(42, 99)).cuda()
    ref = x
    for A, b, act in layers:
        ref = bs.spmv(A, ref, bias=b, act=act)
    stack = bs.LayerStack(layers).capture()
    for _ in range(3):
        y = stack(x)
        torch.cuda.synchronize()
        assert torch.equal(y, ref)
    with pytest.raises(ValueError):
        bs.LayerStack([layers[1], layers[0]])
