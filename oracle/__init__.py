"""fp64 CPU ORACLE for balanced sparsity (arXiv 1811.00206): test infrastructure only.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` and
``--impl reference`` legs) may import this package. The product package ``paper_1811_00206_b200``
never imports it, and the two share no code. See ``oracle/oracle.c`` for the definitions and their
citations to PAPER.md.

Arrays are passed as numpy arrays. f32 is ``np.float32``, f16 is ``np.float16``, and bf16 is given
as raw ``np.uint16`` bit patterns with ``dt=BF16``.

Parity is pinned in ``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

F32, F16, BF16 = 0, 1, 2
SPMV, SPMM, SP24 = 1, 2, 3

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_c_i64 = ctypes.c_int64
_vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so with plain gcc -O2. No CUDA headers, no SIMD intrinsics."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.orc_k_from_sparsity.argtypes = [ctypes.c_int, ctypes.c_double]
        L.orc_k_from_sparsity.restype = ctypes.c_int
        L.orc_prune.argtypes = [_vp, ctypes.c_int, _c_i64, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int, _vp, _vp]
        L.orc_prune.restype = ctypes.c_int
        L.orc_decode.argtypes = [_vp, _vp, ctypes.c_int, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int, _vp]
        L.orc_decode.restype = ctypes.c_int
        L.orc_packed_bytes.argtypes = [_c_i64, _c_i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.orc_packed_bytes.restype = ctypes.c_size_t
        L.orc_pack.argtypes = [_vp, _vp, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp]
        L.orc_pack.restype = ctypes.c_int
        L.orc_spmv_rows.argtypes = [_vp, _vp, ctypes.c_int, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int, _vp, _vp,
                                    _c_i64, _vp, _vp]
        L.orc_spmv_rows.restype = ctypes.c_int
        L.orc_spmv_rowslice.argtypes = [_vp, _vp, ctypes.c_int, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int, _vp,
                                        _vp, _vp]
        L.orc_spmv_rowslice.restype = ctypes.c_int
        L.orc_gemv_dense.argtypes = [_vp, _c_i64, _c_i64, _vp, _vp]
        L.orc_gemv_dense.restype = ctypes.c_int
        L.orc_spmm.argtypes = [_vp, _vp, ctypes.c_int, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int, _vp, _c_i64,
                               _c_i64, _vp, _vp]
        L.orc_spmm.restype = ctypes.c_int
        L.orc_spmm_rows.argtypes = [_vp, _vp, ctypes.c_int, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int, _vp, _c_i64,
                                    _c_i64, _vp, _c_i64, _vp, _vp]
        L.orc_spmm_rows.restype = ctypes.c_int
        L.orc_ideal_time.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double]
        L.orc_ideal_time.restype = ctypes.c_double
        L.orc_act.argtypes = [ctypes.c_double, ctypes.c_int]
        L.orc_act.restype = ctypes.c_double
        L.orc_spmv_act.argtypes = [_vp, _vp, ctypes.c_int, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int, _vp, _vp,
                                   ctypes.c_int, _vp, _vp]
        L.orc_spmv_act.restype = ctypes.c_int
        L.orc_block_rank.argtypes = [_vp, ctypes.c_int, _c_i64, _c_i64, _c_i64, ctypes.c_int, _vp]
        L.orc_block_rank.restype = ctypes.c_int
        L.orc_schedule.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.orc_schedule.restype = ctypes.c_double
        L.orc_prune_dense.argtypes = [_vp, ctypes.c_int, _c_i64, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int, _vp]
        L.orc_prune_dense.restype = ctypes.c_int
        L.orc_keep_count.argtypes = [_c_i64, ctypes.c_double]
        L.orc_keep_count.restype = _c_i64
        L.orc_random_mask.argtypes = [_vp, ctypes.c_int, _c_i64, _c_i64, _c_i64, ctypes.c_double, _vp]
        L.orc_random_mask.restype = ctypes.c_int
        L.orc_block_mask.argtypes = [_vp, ctypes.c_int, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, ctypes.c_double,
                                     ctypes.c_int, _vp]
        L.orc_block_mask.restype = ctypes.c_int
        L.orc_lstm_cell.argtypes = [_vp, _vp, ctypes.c_int, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp,
                                    _vp, _vp, _vp, _vp]
        L.orc_lstm_cell.restype = ctypes.c_int
        L.orc_im2col.argtypes = [_vp, ctypes.c_int, _c_i64, _c_i64, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_int, _vp]
        L.orc_im2col.restype = ctypes.c_int
        L.orc_conv2d.argtypes = [_vp, _vp, ctypes.c_int, _c_i64, ctypes.c_int, ctypes.c_int, _vp, _c_i64, _c_i64,
                                 _c_i64, _c_i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp]
        L.orc_conv2d.restype = ctypes.c_int
        L.orc_elem.argtypes = [_vp, ctypes.c_int, _c_i64]
        L.orc_elem.restype = ctypes.c_double
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data


def _vdtype(dt: int):
    return {F32: np.float32, F16: np.float16, BF16: np.uint16}[dt]


def _check(arr: np.ndarray, dt: int) -> np.ndarray:
    want = _vdtype(dt)
    if arr.dtype != want:
        raise TypeError(f"dtype code {dt} expects numpy {np.dtype(want)}, got {arr.dtype}")
    return np.ascontiguousarray(arr)


# ---------------------------------------------------------------- API

def k_from_sparsity(block: int, sparsity: float) -> int:
    """k = lround((1 - s) * B) in IEEE double."""
    return lib().orc_k_from_sparsity(int(block), float(sparsity))


def prune(W: np.ndarray, dt: int, block: int, k: int):
    """One balance-aware pruning step (Alg. 1 inner loop): canonical (vals, idx)."""
    W = _check(W, dt)
    M, K = W.shape
    NB = K // block
    vals = np.zeros((M, NB, k), dtype=_vdtype(dt))
    idx = np.zeros((M, NB, k), dtype=np.uint16)
    rc = lib().orc_prune(_ptr(W), dt, M, K, K, block, k, _ptr(vals), _ptr(idx))
    if rc != 0:
        raise ValueError("orc_prune rejected the arguments")
    return vals, idx


def decode(vals: np.ndarray, idx: np.ndarray, dt: int, M: int, K: int, block: int, k: int) -> np.ndarray:
    """W_bs as dense fp64."""
    vals = _check(vals, dt)
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    out = np.zeros((M, K), dtype=np.float64)
    if lib().orc_decode(_ptr(vals), _ptr(idx), dt, M, K, block, k, _ptr(out)) != 0:
        raise ValueError("orc_decode rejected the arguments")
    return out


def packed_bytes(M: int, K: int, block: int, k: int, dt: int, layout: int) -> int:
    return int(lib().orc_packed_bytes(M, K, block, k, dt, layout))


def pack(vals: np.ndarray, idx: np.ndarray, M: int, K: int, block: int, k: int, dt: int, layout: int) -> np.ndarray:
    """Reference permutation pi_L of docs/layout.md: packed bytes (uint8)."""
    vals = _check(vals, dt)
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    n = packed_bytes(M, K, block, k, dt, layout)  # 0 for k == 0 (nothing stored) or invalid
    out = np.zeros(max(n, 1), dtype=np.uint8)
    if lib().orc_pack(_ptr(vals), _ptr(idx), M, K, block, k, dt, layout, _ptr(out)) != 0:
        raise ValueError("orc_pack rejected the arguments")
    return out[:n]


def spmv(vals, idx, dt, M, K, block, k, x, rows=None):
    """fp64 y = W_bs·x (Eq. 1 with B = 0) and the per-row tolerance scale sum|w||x| (O-7).

    With ``rows`` (int64 array), only those rows are computed."""
    vals = _check(vals, dt)
    x = _check(x, dt)
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    if rows is None:
        n = M
        rp = None
    else:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        n = rows.size
        rp = _ptr(rows)
    y = np.zeros(n, dtype=np.float64)
    bound = np.zeros(n, dtype=np.float64)
    if lib().orc_spmv_rows(_ptr(vals), _ptr(idx), dt, M, K, block, k, _ptr(x), rp, n, _ptr(y), _ptr(bound)) != 0:
        raise ValueError("orc_spmv_rows rejected the arguments")
    return y, bound


def block_rank(W: np.ndarray, dt: int, B: int) -> np.ndarray:
    """Position of every element in its block's stable magnitude order (orc_block_rank): uint8 [M][K]."""
    W = _check(np.ascontiguousarray(W), dt)
    M, K = W.shape
    out = np.zeros((M, K), dtype=np.uint8)
    if lib().orc_block_rank(_ptr(W), dt, M, K, K, B, _ptr(out)) != 0:
        raise ValueError("orc_block_rank rejected the arguments")
    return out


ACT = {"none": 0, "relu": 1, "sigmoid": 2, "tanh": 3}


def act(v: float, name: str) -> float:
    """The epilogue activation in fp64, from its definition (orc_act)."""
    return lib().orc_act(float(v), ACT[name])


def spmv_act(vals, idx, dt, M, K, block, k, x, bias, act_name):
    """fp64 y = act(W_bs·x + bias) (Eq. 1 with its +B, and an activation) and the tolerance scale
    sum|w||x| + |bias|. bias may be None."""
    vals = _check(vals, dt)
    x = _check(x, dt)
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    bp = None
    if bias is not None:
        bias = _check(bias, dt)
        bp = _ptr(bias)
    y = np.zeros(M, dtype=np.float64)
    bound = np.zeros(M, dtype=np.float64)
    if lib().orc_spmv_act(_ptr(vals), _ptr(idx), dt, M, K, block, k, _ptr(x), bp, ACT[act_name], _ptr(y), _ptr(bound)) != 0:
        raise ValueError("orc_spmv_act rejected the arguments")
    return y, bound


def spmv_rowslice(vals, idx, dt, K, block, k, x):
    """SpMV where vals/idx hold only some rows ([nrows][NB][k]); returns y, bound for those rows."""
    vals = _check(vals, dt)
    x = _check(x, dt)
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    nrows = vals.shape[0]
    y = np.zeros(nrows, dtype=np.float64)
    bound = np.zeros(nrows, dtype=np.float64)
    if lib().orc_spmv_rowslice(_ptr(vals), _ptr(idx), dt, nrows, K, block, k, _ptr(x), _ptr(y), _ptr(bound)) != 0:
        raise ValueError("orc_spmv_rowslice rejected the arguments")
    return y, bound


def spmm(vals, idx, dt, M, K, block, k, X, rows=None):
    """fp64 Y = W_bs·X. X is [N][K] (column n of the K×N operand is X[n]). Returns Y [N][M'], bound."""
    vals = _check(vals, dt)
    X = _check(X, dt)
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    N = X.shape[0]
    if rows is None:
        Y = np.zeros((N, M), dtype=np.float64)
        bound = np.zeros((N, M), dtype=np.float64)
        rc = lib().orc_spmm(_ptr(vals), _ptr(idx), dt, M, K, block, k, _ptr(X), N, X.shape[1], _ptr(Y), _ptr(bound))
    else:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        Y = np.zeros((N, rows.size), dtype=np.float64)
        bound = np.zeros((N, rows.size), dtype=np.float64)
        rc = lib().orc_spmm_rows(_ptr(vals), _ptr(idx), dt, M, K, block, k, _ptr(X), N, X.shape[1], _ptr(rows),
                                 rows.size, _ptr(Y), _ptr(bound))
    if rc != 0:
        raise ValueError("orc_spmm rejected the arguments")
    return Y, bound


def gemv_dense(Wd: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Plain fp64 dense GEMV (used on orc decode output: the dense-masked product, O-7)."""
    Wd = np.ascontiguousarray(Wd, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(Wd.shape[0], dtype=np.float64)
    lib().orc_gemv_dense(_ptr(Wd), Wd.shape[0], Wd.shape[1], _ptr(x), _ptr(y))
    return y


def to_double(a: np.ndarray, dt: int) -> np.ndarray:
    """Exact fp64 values of a D array (uses the oracle's own binary16/bfloat16 decoders)."""
    a = _check(a, dt)
    flat = a.reshape(-1)
    L = lib()
    p = _ptr(flat)
    return np.array([L.orc_elem(p, dt, i) for i in range(flat.size)], dtype=np.float64).reshape(a.shape)


def lstm_cell(vals, idx, dt, M, K, block, k, x, pre, bias, c_prev):
    """One LSTM step with balanced-sparse gate rows interleaved (row 4j+g = gate g of unit j; i, f, g, o):
    z = W_bs·x + pre + bias (Eq. 1 with its +B), c = f·c_prev + i·g, h = o·tanh(c), fp64 (orc_lstm_cell).
    pre / bias: M elements of dt or None. c_prev: M/4 floats. Returns (h, c, zbound) as float64 arrays."""
    vals = _check(vals, dt)
    x = _check(x, dt)
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    H = M // 4
    cp = np.ascontiguousarray(c_prev, dtype=np.float64)
    h = np.zeros(H, dtype=np.float64)
    c = np.zeros(H, dtype=np.float64)
    zb = np.zeros(M, dtype=np.float64)
    pp = _ptr(_check(pre, dt)) if pre is not None else None
    bp = _ptr(_check(bias, dt)) if bias is not None else None
    keep = (pre, bias)  # noqa: F841 (the arrays stay alive through the call)
    if lib().orc_lstm_cell(_ptr(vals), _ptr(idx), dt, M, K, block, k, _ptr(x), pp, bp, _ptr(cp), _ptr(h), _ptr(c),
                           _ptr(zb)) != 0:
        raise ValueError("orc_lstm_cell rejected the arguments")
    return h, c, zb


def conv_out_hw(H: int, W: int, kh: int, kw: int, pad: int, stride: int):
    return (H + 2 * pad - kh) // stride + 1, (W + 2 * pad - kw) // stride + 1


def im2col(inp: np.ndarray, dt: int, kh: int, kw: int, pad: int, stride: int) -> np.ndarray:
    """NHWC input [Nimg][H][W][C] -> X [Nimg·OH·OW][kh·kw·C] with columns (dy, dx, c) (reading A23)."""
    inp = _check(np.ascontiguousarray(inp), dt)
    Nimg, H, W, C = inp.shape
    OH, OW = conv_out_hw(H, W, kh, kw, pad, stride)
    X = np.zeros((Nimg * OH * OW, kh * kw * C), dtype=_vdtype(dt))
    if lib().orc_im2col(_ptr(inp), dt, Nimg, H, W, C, kh, kw, pad, stride, _ptr(X)) != 0:
        raise ValueError("orc_im2col rejected the arguments")
    return X


def conv2d(vals, idx, dt, Cout, block, k, inp, kh, kw, pad, stride):
    """Direct fp64 convolution with the balanced-sparse Cout × (kh·kw·C) weight matrix; NHWC in, Y
    [Nimg·OH·OW][Cout] and the tolerance scale out (orc_conv2d)."""
    vals = _check(vals, dt)
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    inp = _check(np.ascontiguousarray(inp), dt)
    Nimg, H, W, C = inp.shape
    OH, OW = conv_out_hw(H, W, kh, kw, pad, stride)
    Y = np.zeros((Nimg * OH * OW, Cout), dtype=np.float64)
    bound = np.zeros_like(Y)
    if lib().orc_conv2d(_ptr(vals), _ptr(idx), dt, Cout, block, k, _ptr(inp), Nimg, H, W, C, kh, kw, pad, stride,
                        _ptr(Y), _ptr(bound)) != 0:
        raise ValueError("orc_conv2d rejected the arguments")
    return Y, bound


def schedule(target: float, n: int, i: int) -> float:
    """GraduallyIncrease (Alg. 1), cubic per S:205: target·(1 − (1 − i/n)^3)."""
    return lib().orc_schedule(float(target), int(n), int(i))


def prune_dense(W: np.ndarray, dt: int, block: int, k: int) -> np.ndarray:
    """Alg. 1's pruned matrix M_p after one step at k per block: kept entries bit-copied, +0 elsewhere."""
    W = _check(np.ascontiguousarray(W), dt)
    M, K = W.shape
    out = np.zeros((M, K), dtype=_vdtype(dt))
    if lib().orc_prune_dense(_ptr(W), dt, M, K, K, block, k, _ptr(out)) != 0:
        raise ValueError("orc_prune_dense rejected the arguments")
    return out


def keep_count(n: int, sparsity: float) -> int:
    """Units kept at sparsity s: lround((1 − s)·n)."""
    return int(lib().orc_keep_count(int(n), float(sparsity)))


def random_mask(W: np.ndarray, dt: int, sparsity: float) -> np.ndarray:
    """Random sparsity (global magnitude pruning): uint8 keep mask [M][K]."""
    W = _check(np.ascontiguousarray(W), dt)
    M, K = W.shape
    out = np.zeros((M, K), dtype=np.uint8)
    if lib().orc_random_mask(_ptr(W), dt, M, K, K, float(sparsity), _ptr(out)) != 0:
        raise ValueError("orc_random_mask rejected the arguments")
    return out


def block_mask(W: np.ndarray, dt: int, bh: int, bw: int, sparsity: float, criterion: str = "max") -> np.ndarray:
    """Block sparsity with bh×bw tiles scored by max or mean |w|; vector sparsity is
    bh = 1, bw = K (rows) or bh = M, bw = 1 (columns) with "mean". uint8 keep mask [M][K]."""
    W = _check(np.ascontiguousarray(W), dt)
    M, K = W.shape
    out = np.zeros((M, K), dtype=np.uint8)
    crit = {"max": 0, "mean": 1}[criterion]
    if lib().orc_block_mask(_ptr(W), dt, M, K, K, int(bh), int(bw), float(sparsity), crit, _ptr(out)) != 0:
        raise ValueError("orc_block_mask rejected the arguments")
    return out


def ideal_time(d_time: float, o_time: float, sparsity: float) -> float:
    """i_time = (d_time - o_time) * (1 - sparsity) + o_time."""
    return lib().orc_ideal_time(d_time, o_time, sparsity)


def check_tolerance(y_gpu: np.ndarray, y_ref: np.ndarray, bound: np.ndarray, tau: float):
    """O-7 comparison rule. Requires |y_gpu - y_ref| <= tau * bound per element (and y_gpu == 0 where
    bound == 0). Returns (ok, worst |err|/bound)."""
    y_gpu = np.asarray(y_gpu, dtype=np.float64)
    err = np.abs(y_gpu - y_ref)
    zero = bound == 0
    ok_zero = bool(np.all(y_gpu[zero] == 0))
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(zero, 0.0, err / np.where(zero, 1.0, bound))
    worst = float(rel.max()) if rel.size else 0.0
    return ok_zero and bool(np.all(rel <= tau)), worst


TAU = {F32: 1e-4, F16: 1e-2, BF16: 1e-2}
"""Per-element tolerance factors stated by BASELINE.json's north_star."""
