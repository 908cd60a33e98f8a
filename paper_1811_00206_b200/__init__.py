"""B200-native balanced sparsity (arXiv 1811.00206): thin Python binding over libbs.so.

Every step of the path runs in the CUDA kernels behind the C ABI (include/bs.h). This module only
marshals arguments: it turns torch CUDA tensors into device pointers and passes the current CUDA
stream. There is no CPU fallback: libbs.so is loaded on first use (every entry point below), and if it is
missing that call raises ImportError. Only the host-side helpers of `dist` (slice ranges, the shard
policy) work without it.

    import paper_1811_00206_b200 as bs
    vals, idx, k = bs.prune(W, block=32, sparsity=0.9)    # Alg. 1 step
    A = bs.pack(vals, idx, K=W.shape[1], block=32)          # compact balanced format
    y = bs.spmv(A, x)                                       # y = W_bs·x (Eq. 1)
    Y = bs.spmm(bs.pack(vals, idx, K, 32, layout="spmm"), X)  # X: [N, K] -> Y: [N, M]
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbs.so")

BS_OK, BS_ERR_ARG, BS_ERR_SHAPE, BS_ERR_DTYPE, BS_ERR_UNSUPPORTED, BS_ERR_CUDA = range(6)
DTYPES = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2}
LAYOUTS = {"spmv": 1, "spmm": 2, "sp24": 3}

EXPORTS = ("bs_k_from_sparsity", "bs_packed_bytes", "bs_status_str", "bs_version", "bs_prune", "bs_prune_k",
           "bs_pack", "bs_unpack", "bs_spmv", "bs_spmv_ex", "bs_spmv_fused", "bs_spmv_host", "bs_spmm", "bs_choose_layout", "bs_block_rank",
           "bs_schedule_sparsity", "bs_keep_count", "bs_decode", "bs_pattern_workspace_bytes", "bs_random_mask",
           "bs_block_mask", "bs_lstm_step", "bs_im2col", "bs_spmv_allgather", "bs_allgather_wait", "bs_peer_export",
           "bs_peer_import", "bs_peer_close", "bs_x_slot_offset", "bs_conv2d", "bs_spmm_fused")
ACTS = {None: 0, "none": 0, "relu": 1, "sigmoid": 2, "tanh": 3}  # bs_act (include/bs.h)
SPMV_PDL, SPMV_W_STATIC, SPMV_RING = 1, 2, 4  # bs_spmv_ex flags (include/bs.h)


class BSError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {lib().bs_status_str(status).decode()} ({status})")
        self.status = status


class _Matrix(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int64), ("K", ctypes.c_int64), ("block", ctypes.c_int32), ("k", ctypes.c_int32),
                ("dt", ctypes.c_int32), ("layout", ctypes.c_int32), ("packed", ctypes.c_void_p)]


class _AllGather(ctypes.Structure):
    """bs_allgather (include/bs.h)."""
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("row0", ctypes.c_int64),
                ("y", ctypes.c_void_p * 8), ("flags", ctypes.c_void_p * 8), ("counter", ctypes.c_void_p),
                ("epoch", ctypes.c_uint32)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_1811_00206_b200/build.py` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    L.bs_k_from_sparsity.argtypes = [ci, ctypes.c_double]
    L.bs_k_from_sparsity.restype = ci
    L.bs_packed_bytes.argtypes = [i64, i64, ci, ci, ci, ci]
    L.bs_packed_bytes.restype = ctypes.c_size_t
    L.bs_block_rank.argtypes = [vp, ci, i64, i64, i64, ci, vp, vp]
    L.bs_block_rank.restype = ci
    L.bs_choose_layout.argtypes = [i64, i64, ci, ci, ci, i64]
    L.bs_choose_layout.restype = ci
    L.bs_status_str.argtypes = [ci]
    L.bs_status_str.restype = ctypes.c_char_p
    L.bs_version.argtypes = []
    L.bs_version.restype = ctypes.c_char_p
    L.bs_prune.argtypes = [vp, ci, i64, i64, i64, ci, ctypes.c_double, ctypes.POINTER(ci), vp, vp, vp]
    L.bs_prune_k.argtypes = [vp, ci, i64, i64, i64, ci, ci, vp, vp, vp]
    L.bs_pack.argtypes = [vp, vp, i64, i64, ci, ci, ci, ci, vp, vp]
    L.bs_unpack.argtypes = [vp, i64, i64, ci, ci, ci, ci, vp, vp, vp]
    L.bs_spmv.argtypes = [ctypes.POINTER(_Matrix), vp, vp, vp]
    L.bs_spmv_ex.argtypes = [ctypes.POINTER(_Matrix), vp, vp, ctypes.c_uint, vp]
    L.bs_spmv_fused.argtypes = [ctypes.POINTER(_Matrix), vp, vp, ci, vp, ctypes.c_uint, vp]
    L.bs_spmv_host.argtypes = [ctypes.POINTER(_Matrix), vp, vp, vp, vp, vp]
    L.bs_spmm.argtypes = [ctypes.POINTER(_Matrix), vp, i64, i64, vp, i64, vp]
    L.bs_schedule_sparsity.argtypes = [ctypes.c_double, ci, ci]
    L.bs_schedule_sparsity.restype = ctypes.c_double
    L.bs_keep_count.argtypes = [i64, ctypes.c_double]
    L.bs_keep_count.restype = i64
    L.bs_decode.argtypes = [vp, vp, i64, i64, ci, ci, ci, vp, i64, vp]
    L.bs_pattern_workspace_bytes.argtypes = [i64, i64, i64, i64]
    L.bs_pattern_workspace_bytes.restype = ctypes.c_size_t
    L.bs_random_mask.argtypes = [vp, ci, i64, i64, i64, ctypes.c_double, vp, vp, ctypes.c_size_t, vp]
    L.bs_block_mask.argtypes = [vp, ci, i64, i64, i64, i64, i64, ctypes.c_double, ci, vp, vp, ctypes.c_size_t, vp]
    L.bs_lstm_step.argtypes = [ctypes.POINTER(_Matrix), vp, vp, vp, vp, vp, vp, ctypes.c_uint, vp]
    L.bs_im2col.argtypes = [vp, ci, i64, i64, i64, i64, ci, ci, ci, ci, vp, i64, vp]
    L.bs_conv2d.argtypes = [ctypes.POINTER(_Matrix), vp, i64, i64, i64, i64, ci, ci, ci, ci, vp, ci, vp, vp]
    L.bs_spmm_fused.argtypes = [ctypes.POINTER(_Matrix), vp, i64, i64, vp, ci, vp, i64, vp]
    L.bs_x_slot_offset.argtypes = [i64, ci, ci, ci, i64, ci, ci]
    L.bs_x_slot_offset.restype = i64
    L.bs_spmv_allgather.argtypes = [ctypes.POINTER(_Matrix), vp, vp, ci, ctypes.POINTER(_AllGather), ctypes.c_uint, vp]
    L.bs_allgather_wait.argtypes = [ctypes.POINTER(_AllGather), vp]
    L.bs_peer_export.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_int64)]
    L.bs_peer_import.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]
    L.bs_peer_close.argtypes = [vp, ctypes.c_int64]
    for f in ("bs_decode", "bs_random_mask", "bs_block_mask", "bs_lstm_step", "bs_im2col", "bs_conv2d", "bs_spmm_fused", "bs_spmv_allgather",
              "bs_allgather_wait", "bs_peer_export", "bs_peer_import", "bs_peer_close"):
        getattr(L, f).restype = ci
    for f in ("bs_prune", "bs_prune_k", "bs_pack", "bs_unpack", "bs_spmv", "bs_spmv_ex", "bs_spmv_fused", "bs_spmv_host", "bs_spmm"):
        getattr(L, f).restype = ci
    return L


_LIB = None


def lib() -> ctypes.CDLL:
    """libbs.so, loaded on first use (raises ImportError if it was not built)."""
    global _LIB
    if _LIB is None:
        _LIB = _load()
    return _LIB


def version() -> str:
    return lib().bs_version().decode()


def _stream(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _check(st: int, where: str):
    if st != BS_OK:
        raise BSError(st, where)


def _dt(t: torch.Tensor) -> int:
    try:
        return DTYPES[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype}; use float32, float16 or bfloat16") from None


def _need_cuda(*ts):
    for t in ts:
        if not t.is_cuda:
            raise ValueError("tensors must live on a CUDA device (there is no CPU path)")


def _same_device(A: "BSMatrix", *ts):
    for t in ts:
        if t is not None and A.packed.numel() and t.device != A.packed.device:
            raise ValueError(f"tensor on {t.device} but the matrix lives on {A.packed.device}")


def _check_out(out: torch.Tensor, A: "BSMatrix", shape: tuple):
    """A caller-supplied output buffer: the kernel writes through its raw pointer, so its dtype, device,
    size and strides must match exactly (a short buffer would be an out-of-bounds device write)."""
    _need_cuda(out)
    if out.dtype != A.dtype:
        raise ValueError(f"out has dtype {out.dtype}, expected {A.dtype}")
    if tuple(out.shape) != shape:
        raise ValueError(f"out has shape {tuple(out.shape)}, expected {shape}")
    if out.stride(-1) != 1 or (len(shape) == 1 and not out.is_contiguous()):
        raise ValueError("out must have unit stride along M")
    if len(shape) == 2 and shape[0] > 1 and out.stride(0) < shape[1]:
        raise ValueError("out rows overlap (stride(0) < M)")
    _same_device(A, out)


def k_from_sparsity(block: int, sparsity: float) -> int:
    """k = lround((1 - s)·B)."""
    return lib().bs_k_from_sparsity(int(block), float(sparsity))


def packed_bytes(M: int, K: int, block: int, k: int, dtype: torch.dtype, layout: str = "spmv") -> int:
    return int(lib().bs_packed_bytes(M, K, block, k, DTYPES[dtype], LAYOUTS[layout]))


@dataclass
class BSMatrix:
    """A packed balanced-sparse matrix resident in device memory (docs/layout.md)."""

    M: int
    K: int
    block: int
    k: int
    dtype: torch.dtype
    layout: str
    packed: torch.Tensor  # uint8, bs_packed_bytes bytes

    def cstruct(self) -> _Matrix:
        return _Matrix(self.M, self.K, self.block, self.k, DTYPES[self.dtype], LAYOUTS[self.layout],
                       self.packed.data_ptr() if self.packed.numel() else None)

    @property
    def nnz(self) -> int:
        return self.M * (self.K // self.block) * self.k

    @property
    def nbytes(self) -> int:
        return self.packed.numel()

    @property
    def sparsity(self) -> float:
        """Achieved sparsity 1 - k/B."""
        return 1.0 - self.k / self.block


def prune(W: torch.Tensor, block: int, sparsity: float | None = None, k: int | None = None):
    """One balance-aware pruning step on the GPU (Alg. 1): returns (vals, idx, k).

    vals [M, K/B, k] of W.dtype are bit copies of the kept weights, and idx [M, K/B, k] (int16 holding
    uint16 offsets) are the kept block-local offsets, ascending."""
    _need_cuda(W)
    if W.dim() != 2 or W.stride(1) != 1:
        raise ValueError("W must be a 2-D row-major tensor")
    M, K = W.shape
    if k is None:
        if sparsity is None:
            raise ValueError("give sparsity or k")
        k = k_from_sparsity(block, sparsity)
        if k < 0:
            raise BSError(BS_ERR_ARG, "bs_prune")
    NB = K // block if block > 0 else 0
    vals = torch.empty((M, NB, max(k, 0)), dtype=W.dtype, device=W.device)
    idx = torch.empty((M, NB, max(k, 0)), dtype=torch.int16, device=W.device)
    with torch.cuda.device(W.device):
        st = lib().bs_prune_k(W.data_ptr(), _dt(W), M, K, W.stride(0), block, k, vals.data_ptr() if vals.numel() else None,
                             idx.data_ptr() if idx.numel() else None, _stream(W.device))
    _check(st, "bs_prune_k")
    return vals, idx, k


def block_rank(W: torch.Tensor, block: int) -> torch.Tensor:
    """Every element's position in its block's magnitude order (bs_block_rank): uint8 [M, K]. The mask
    of a pruning step at any k is rank < k (Alg. 1's schedule without retraining)."""
    _need_cuda(W)
    if W.dim() != 2:
        raise ValueError("W must be a 2-D tensor")
    dt = _dt(W)
    M, K = W.shape
    if W.stride(1) != 1:
        W = W.contiguous()
    rank = torch.empty((M, K), dtype=torch.uint8, device=W.device)
    with torch.cuda.device(W.device):
        st = lib().bs_block_rank(W.data_ptr(), dt, M, K, W.stride(0), block, rank.data_ptr(),
                                _stream(W.device))
    _check(st, "bs_block_rank")
    return rank


def choose_layout(M: int, K: int, block: int, k: int, dtype: torch.dtype, batch: int) -> str:
    """bs_choose_layout: the layout bs_spmm runs fastest on for `batch` columns (include/bs.h)."""
    code = lib().bs_choose_layout(M, K, block, k, DTYPES[dtype], batch)
    if code < 0:
        raise ValueError("bs_choose_layout rejected the arguments")
    return {v: n for n, v in LAYOUTS.items()}[code]


def pack(vals: torch.Tensor, idx: torch.Tensor, K: int, block: int, layout: str = "spmv",
         batch: int | None = None) -> BSMatrix:
    """Permute canonical (vals, idx) into a device layout (docs/layout.md). layout="auto" takes
    bs_choose_layout's pick for `batch` columns (default 1)."""
    _need_cuda(vals, idx)
    M, NB, k = vals.shape
    if layout == "auto":
        layout = choose_layout(M, K, block, k, vals.dtype, batch or 1)
    vals = vals.contiguous()
    idx = idx.contiguous()
    n = packed_bytes(M, K, block, k, vals.dtype, layout)
    if n == 0 and k != 0:
        raise BSError(BS_ERR_UNSUPPORTED, "bs_packed_bytes")
    out = torch.empty(n, dtype=torch.uint8, device=vals.device)
    with torch.cuda.device(vals.device):
        st = lib().bs_pack(vals.data_ptr() if vals.numel() else None, idx.data_ptr() if idx.numel() else None, M, K,
                          block, k, _dt(vals), LAYOUTS[layout], out.data_ptr() if n else None, _stream(vals.device))
    _check(st, "bs_pack")
    return BSMatrix(M, K, block, k, vals.dtype, layout, out)


def unpack(A: BSMatrix):
    """Inverse of pack: canonical (vals, idx)."""
    NB = A.K // A.block
    vals = torch.empty((A.M, NB, A.k), dtype=A.dtype, device=A.packed.device)
    idx = torch.empty((A.M, NB, A.k), dtype=torch.int16, device=A.packed.device)
    with torch.cuda.device(A.packed.device):
        st = lib().bs_unpack(A.packed.data_ptr() if A.packed.numel() else None, A.M, A.K, A.block, A.k, DTYPES[A.dtype], LAYOUTS[A.layout],
                            vals.data_ptr() if vals.numel() else None, idx.data_ptr() if idx.numel() else None,
                            _stream(A.packed.device))
    _check(st, "bs_unpack")
    return vals, idx


def spmv(A: BSMatrix, x: torch.Tensor, out: torch.Tensor | None = None, flags: int | None = None,
         bias: torch.Tensor | None = None, act: str | None = None) -> torch.Tensor:
    """y = W_bs·x (Eq. 1 with B = 0). x: [K] of A.dtype; returns y: [M].
    flags: None -> bs_spmv (PDL launch); otherwise bs_spmv_ex with SPMV_PDL / SPMV_W_STATIC bits.
    bias ([M] of A.dtype) and act ("relu" | "sigmoid" | "tanh") select the fused layer epilogue
    y = act(W_bs·x + bias) (bs_spmv_fused, Eq. 1 with its +B)."""
    _need_cuda(x)
    if x.dtype != A.dtype or x.numel() != A.K:
        raise ValueError("x must have A.K elements of A.dtype")
    _same_device(A, x)
    x = x.contiguous()
    if out is not None:
        _check_out(out, A, (A.M,))
        if out.device != x.device:
            raise ValueError("out and x must live on the same device")
    y = out if out is not None else torch.empty(A.M, dtype=A.dtype, device=x.device)
    m = A.cstruct()
    with torch.cuda.device(x.device):
        if bias is not None or act is not None:
            if act not in ACTS:
                raise ValueError(f"act must be one of {sorted(k for k in ACTS if k)}")
            if bias is not None:
                _need_cuda(bias)
                _same_device(A, bias)
                if bias.dtype != A.dtype or bias.numel() != A.M:
                    raise ValueError("bias must have A.M elements of A.dtype")
                bias = bias.contiguous()
            st = lib().bs_spmv_fused(ctypes.byref(m), x.data_ptr(), bias.data_ptr() if bias is not None else None,
                                    ACTS[act], y.data_ptr(), bs_flags_default() if flags is None else flags,
                                    _stream(x.device))
        elif flags is None:
            st = lib().bs_spmv(ctypes.byref(m), x.data_ptr(), y.data_ptr(), _stream(x.device))
        else:
            st = lib().bs_spmv_ex(ctypes.byref(m), x.data_ptr(), y.data_ptr(), flags, _stream(x.device))
    _check(st, "bs_spmv")
    return y


def bs_flags_default() -> int:
    """The launch flags bs_spmv uses (PDL)."""
    return SPMV_PDL


def spmv_host(A: BSMatrix, x_host: torch.Tensor, y_host: torch.Tensor, x_dev: torch.Tensor, y_dev: torch.Tensor):
    """End-to-end product through the C ABI with host buffers: H2D(x) -> SpMV -> D2H(y), enqueued on the
    current stream (bs_spmv_host). y_host is valid after the stream synchronises."""
    if x_host.dtype != A.dtype or y_host.dtype != A.dtype or x_host.numel() < A.K or y_host.numel() < A.M:
        raise ValueError("x_host / y_host must hold A.K / A.M elements of A.dtype")
    if x_host.is_cuda or y_host.is_cuda or not (x_host.is_contiguous() and y_host.is_contiguous()):
        raise ValueError("x_host and y_host must be contiguous host tensors")
    _need_cuda(x_dev)
    _check_out(y_dev, A, (A.M,))
    if x_dev.dtype != A.dtype or x_dev.numel() != A.K or not x_dev.is_contiguous():
        raise ValueError("x_dev must be a contiguous device buffer of A.K elements of A.dtype")
    _same_device(A, x_dev)
    m = A.cstruct()
    with torch.cuda.device(x_dev.device):
        st = lib().bs_spmv_host(ctypes.byref(m), x_host.data_ptr(), y_host.data_ptr(), x_dev.data_ptr(),
                               y_dev.data_ptr(), _stream(x_dev.device))
    _check(st, "bs_spmv_host")


def spmm(A: BSMatrix, X: torch.Tensor, out: torch.Tensor | None = None, bias: torch.Tensor | None = None,
         act: str | None = None) -> torch.Tensor:
    """Y = W_bs·X for a batch. X: [N, K] (row n = column n of the K×N operand); returns Y: [N, M].
    bias ([M] of A.dtype) / act ("relu" | "sigmoid" | "tanh"): the fused layer epilogue Y = act(W_bs·X + bias)
    (bs_spmm_fused; SPMM layout on the tensor cores)."""
    _need_cuda(X)
    if X.dim() != 2 or X.shape[1] != A.K or X.dtype != A.dtype or X.stride(1) != 1:
        raise ValueError("X must be [N, K] of A.dtype with unit column stride")
    if act not in ACTS:
        raise ValueError(f"act must be one of {sorted(k for k in ACTS if k)}")
    if bias is not None and (bias.dtype != A.dtype or bias.numel() != A.M or not bias.is_contiguous()):
        raise ValueError("bias must be a contiguous vector of A.M elements of A.dtype")
    _same_device(A, X, bias)
    if bias is not None or ACTS[act] != 0:
        N = X.shape[0]
        if out is not None:
            _check_out(out, A, (N, A.M))
        Y = out if out is not None else torch.empty((N, A.M), dtype=A.dtype, device=X.device)
        m = A.cstruct()
        with torch.cuda.device(X.device):
            st = lib().bs_spmm_fused(ctypes.byref(m), X.data_ptr(), N, X.stride(0),
                                     bias.data_ptr() if bias is not None else None, ACTS[act], Y.data_ptr(),
                                     Y.stride(0), _stream(X.device))
        _check(st, "bs_spmm_fused")
        return Y
    N = X.shape[0]
    if out is not None:
        _check_out(out, A, (N, A.M))
        if out.device != X.device:
            raise ValueError("out and X must live on the same device")
    Y = out if out is not None else torch.empty((N, A.M), dtype=A.dtype, device=X.device)
    m = A.cstruct()
    with torch.cuda.device(X.device):
        st = lib().bs_spmm(ctypes.byref(m), X.data_ptr(), N, X.stride(0), Y.data_ptr(), Y.stride(0), _stream(X.device))
    _check(st, "bs_spmm")
    return Y


# ---------------------------------------------------------------- Alg. 1's schedule and the comparison patterns

def schedule(target: float, n: int, i: int) -> float:
    """GraduallyIncrease (Alg. 1): s_i = target·(1 − (1 − i/n)^3) (bs_schedule_sparsity)."""
    v = lib().bs_schedule_sparsity(float(target), int(n), int(i))
    if v < 0:
        raise ValueError("schedule needs n >= 1, 0 <= i <= n and 0 <= target < 1")
    return v


def keep_count(n: int, sparsity: float) -> int:
    """Units kept at sparsity s: lround((1 − s)·n) (bs_keep_count)."""
    return int(lib().bs_keep_count(int(n), float(sparsity)))


def decode(vals: torch.Tensor, idx: torch.Tensor, K: int, block: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """Dense W_bs (Alg. 1's pruned matrix M_p) from canonical (vals, idx) (bs_decode)."""
    _need_cuda(vals, idx)
    M, NB, k = vals.shape
    vals = vals.contiguous()
    idx = idx.contiguous()
    if out is None:
        out = torch.empty((M, K), dtype=vals.dtype, device=vals.device)
    else:
        _need_cuda(out)
        if out.dtype != vals.dtype or tuple(out.shape) != (M, K) or out.stride(1) != 1 or out.device != vals.device:
            raise ValueError("out must be [M, K] of vals.dtype on vals.device with unit column stride")
    with torch.cuda.device(vals.device):
        st = lib().bs_decode(vals.data_ptr() if vals.numel() else None, idx.data_ptr() if idx.numel() else None, M, K,
                             block, k, _dt(vals), out.data_ptr(), out.stride(0), _stream(vals.device))
    _check(st, "bs_decode")
    return out


def prune_dense(W: torch.Tensor, block: int, sparsity: float | None = None, k: int | None = None,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """One pruning iteration of Alg. 1 on a dense matrix: W with all but the k largest-magnitude entries of
    every block set to +0 (bs_prune_k + bs_decode). out=W prunes in place."""
    vals, idx, k = prune(W, block, sparsity=sparsity, k=k)
    return decode(vals, idx, W.shape[1], block, out=out)


def gradual_prune(W: torch.Tensor, block: int, target: float, n: int, retrain=None):
    """Alg. 1: n pruning iterations at the GraduallyIncrease sparsities s_1..s_n (schedule),
    each followed by ``retrain(W)`` if given (the paper's "pruning followed by a retraining is one
    iteration"; the callback may update W in place, pruned entries must stay zero for the pattern
    to hold). Works on a copy of W; returns (M_p, [k_1..k_n]). Without retraining the survivors nest and
    M_p equals a single step at the target."""
    cur = W.clone()
    ks = []
    for i in range(1, n + 1):
        k = k_from_sparsity(block, schedule(target, n, i))
        prune_dense(cur, block, k=k, out=cur)
        ks.append(k)
        if retrain is not None:
            retrain(cur)
    return cur, ks


def _workspace(M: int, K: int, bh: int, bw: int, device) -> torch.Tensor:
    n = int(lib().bs_pattern_workspace_bytes(M, K, bh, bw))
    if n == 0:
        raise BSError(BS_ERR_SHAPE, "bs_pattern_workspace_bytes")
    return torch.empty(n, dtype=torch.uint8, device=device)


def random_mask(W: torch.Tensor, sparsity: float) -> torch.Tensor:
    """Random sparsity (global magnitude pruning): uint8 keep mask [M, K] (bs_random_mask)."""
    _need_cuda(W)
    if W.dim() != 2 or W.stride(1) != 1:
        raise ValueError("W must be a 2-D tensor with unit column stride")
    M, K = W.shape
    mask = torch.empty((M, K), dtype=torch.uint8, device=W.device)
    ws = _workspace(M, K, 0, 0, W.device)
    with torch.cuda.device(W.device):
        st = lib().bs_random_mask(W.data_ptr(), _dt(W), M, K, W.stride(0), float(sparsity), mask.data_ptr(),
                                  ws.data_ptr(), ws.numel(), _stream(W.device))
    _check(st, "bs_random_mask")
    return mask


def block_mask(W: torch.Tensor, bh: int, bw: int, sparsity: float, criterion: str = "max") -> torch.Tensor:
    """Block sparsity: bh×bw tiles scored by max or mean |w|, the best lround((1−s)·#tiles)
    kept whole. uint8 keep mask [M, K] (bs_block_mask)."""
    _need_cuda(W)
    if W.dim() != 2 or W.stride(1) != 1:
        raise ValueError("W must be a 2-D tensor with unit column stride")
    M, K = W.shape
    crit = {"max": 0, "mean": 1}[criterion]
    mask = torch.empty((M, K), dtype=torch.uint8, device=W.device)
    ws = _workspace(M, K, bh, bw, W.device)
    with torch.cuda.device(W.device):
        st = lib().bs_block_mask(W.data_ptr(), _dt(W), M, K, W.stride(0), int(bh), int(bw), float(sparsity), crit,
                                 mask.data_ptr(), ws.data_ptr(), ws.numel(), _stream(W.device))
    _check(st, "bs_block_mask")
    return mask


def vector_mask(W: torch.Tensor, sparsity: float, axis: str = "row") -> torch.Tensor:
    """Vector sparsity: whole rows (axis="row") or columns scored by mean |w| (bs_block_mask with a
    1×K or M×1 tile)."""
    M, K = W.shape
    return block_mask(W, 1, K, sparsity, "mean") if axis == "row" else block_mask(W, M, 1, sparsity, "mean")


# ---------------------------------------------------------------- LSTM layers (PTB P:347, TIMIT P:369)

def interleave_gates(W: torch.Tensor) -> torch.Tensor:
    """PyTorch's gate-block row order (blocks i, f, g, o of H rows each) -> bs_lstm_step's interleaved
    order (row 4j + g = gate g of unit j). Works for weights [4H, K] and biases [4H]."""
    H = W.shape[0] // 4
    return W.reshape(4, H, *W.shape[1:]).transpose(0, 1).reshape(W.shape).contiguous()


def lstm_step(A: BSMatrix, x: torch.Tensor, c_prev: torch.Tensor, pre: torch.Tensor | None = None,
              bias: torch.Tensor | None = None, h_out: torch.Tensor | None = None, c_out: torch.Tensor | None = None,
              flags: int | None = None):
    """One LSTM step in one kernel (bs_lstm_step): z = W_bs·x + pre + bias with interleaved gate rows, then
    c = σ(z_f)·c_prev + σ(z_i)·tanh(z_g), h = σ(z_o)·tanh(c). Returns (h [M/4] of A.dtype, c [M/4] fp32)."""
    _need_cuda(x, c_prev)
    if A.M % 4:
        raise ValueError("an LSTM gate matrix has 4·H rows")
    H = A.M // 4
    if x.dtype != A.dtype or x.numel() != A.K or not x.is_contiguous():
        raise ValueError("x must be a contiguous vector of A.K elements of A.dtype")
    if c_prev.dtype != torch.float32 or c_prev.numel() != H or not c_prev.is_contiguous():
        raise ValueError("c_prev must be a contiguous fp32 vector of M/4 elements")
    for v, name in ((pre, "pre"), (bias, "bias")):
        if v is not None and (v.dtype != A.dtype or v.numel() != A.M or not v.is_contiguous() or not v.is_cuda):
            raise ValueError(f"{name} must be a contiguous CUDA vector of A.M elements of A.dtype")
    _same_device(A, x, c_prev, pre, bias)
    if h_out is None:
        h_out = torch.empty(H, dtype=A.dtype, device=x.device)
    elif h_out.dtype != A.dtype or h_out.numel() != H or not h_out.is_contiguous() or h_out.device != x.device:
        raise ValueError("h_out must be a contiguous vector of M/4 elements of A.dtype")
    if c_out is None:
        c_out = torch.empty(H, dtype=torch.float32, device=x.device)
    elif c_out.dtype != torch.float32 or c_out.numel() != H or not c_out.is_contiguous() or c_out.device != x.device:
        raise ValueError("c_out must be a contiguous fp32 vector of M/4 elements")
    m = A.cstruct()
    with torch.cuda.device(x.device):
        st = lib().bs_lstm_step(ctypes.byref(m), x.data_ptr(), pre.data_ptr() if pre is not None else None,
                                bias.data_ptr() if bias is not None else None, c_prev.data_ptr(), h_out.data_ptr(),
                                c_out.data_ptr(), bs_flags_default() if flags is None else flags, _stream(x.device))
    _check(st, "bs_lstm_step")
    return h_out, c_out


def lstm_sequence(A_ih: BSMatrix, A_hh: BSMatrix, X: torch.Tensor, h0: torch.Tensor, c0: torch.Tensor,
                  bias: torch.Tensor | None = None):
    """A whole LSTM layer over T steps with balanced-sparse W_ih and W_hh (gate rows interleaved):
    the input projections of all steps are ONE batched product U = W_ih·X (bs_spmm, N = T; the
    large-N SpMM of SURVEY NEXT-3), then each step is one bs_lstm_step on W_hh with pre = U[t].
    X: [T, In]; h0: [H] of the dtype; c0: [H] fp32. Returns (hs [T, H], c_T)."""
    T = X.shape[0]
    H = A_hh.M // 4
    U = spmm(A_ih, X)  # [T, 4H]
    hs = torch.empty((T, H), dtype=A_hh.dtype, device=X.device)
    c_bufs = (torch.empty(H, dtype=torch.float32, device=X.device), torch.empty(H, dtype=torch.float32, device=X.device))
    h, c = h0, c0
    for t in range(T):
        c_next = c_bufs[t % 2]
        lstm_step(A_hh, h, c, pre=U[t], bias=bias, h_out=hs[t], c_out=c_next)
        h, c = hs[t], c_next
    return hs, c


# ---------------------------------------------------------------- convolution via im2col

def conv_weight_matrix(w: torch.Tensor) -> torch.Tensor:
    """torch conv weight [Cout, C, kh, kw] -> the Cout × (kh·kw·C) matrix with (dy, dx, c) columns that
    bs_im2col's X multiplies (reading A23). Prune / pack this matrix."""
    return w.permute(0, 2, 3, 1).reshape(w.shape[0], -1).contiguous()


def im2col(inp: torch.Tensor, kh: int, kw: int, pad: int = 0, stride: int = 1, out: torch.Tensor | None = None):
    """NHWC [Nimg, H, W, C] -> X [Nimg·OH·OW, kh·kw·C] (bs_im2col)."""
    _need_cuda(inp)
    if inp.dim() != 4 or not inp.is_contiguous():
        raise ValueError("inp must be a contiguous NHWC tensor [Nimg, H, W, C]")
    Nimg, H, W, C = inp.shape
    OH, OW = (H + 2 * pad - kh) // stride + 1, (W + 2 * pad - kw) // stride + 1
    if OH < 1 or OW < 1:
        raise ValueError("kernel larger than the padded image")
    Kc = kh * kw * C
    if out is None:
        out = torch.empty((Nimg * OH * OW, Kc), dtype=inp.dtype, device=inp.device)
    elif out.dtype != inp.dtype or out.shape[0] != Nimg * OH * OW or out.shape[1] != Kc or out.stride(1) != 1:
        raise ValueError("out must be [Nimg·OH·OW, kh·kw·C] of inp.dtype with unit column stride")
    with torch.cuda.device(inp.device):
        st = lib().bs_im2col(inp.data_ptr(), _dt(inp), Nimg, H, W, C, kh, kw, pad, stride, out.data_ptr(),
                             out.stride(0), _stream(inp.device))
    _check(st, "bs_im2col")
    return out


def conv2d(A: BSMatrix, inp: torch.Tensor, kh: int, kw: int, pad: int = 0, stride: int = 1,
           workspace: torch.Tensor | None = None, implicit: bool | None = None,
           bias: torch.Tensor | None = None, act: str | None = None) -> torch.Tensor:
    """A conv layer with the balanced-sparse Cout × (kh·kw·C) weight matrix A. NHWC in [Nimg, H, W, C], NHWC out
    [Nimg, OH, OW, Cout]. implicit=None: bs_conv2d (TMA im2col feeding the tensor cores, no intermediate) when
    eligible (SPMM layout, 16-bit, C % 64 == 0, stride 1), else bs_im2col then bs_spmm; True/False forces one.
    bias ([Cout] of A.dtype) and act ("relu" | "sigmoid" | "tanh") fuse the layer epilogue into bs_conv2d
    (they need the implicit path)."""
    _need_cuda(inp)
    Nimg, H, W, C = inp.shape
    if A.K != kh * kw * C:
        raise ValueError("A.K must equal kh·kw·C")
    if inp.dtype != A.dtype:
        raise ValueError("inp must have A.dtype")
    if act not in ACTS:
        raise ValueError(f"act must be one of {sorted(k for k in ACTS if k)}")
    if bias is not None and (bias.dtype != A.dtype or bias.numel() != A.M or not bias.is_contiguous()):
        raise ValueError("bias must be a contiguous vector of A.M elements of A.dtype")
    _same_device(A, inp, bias)
    fused = bias is not None or ACTS[act] != 0
    if fused and implicit is False:
        raise ValueError("bias/act are fused into bs_conv2d only (implicit=True or None)")
    OH, OW = (H + 2 * pad - kh) // stride + 1, (W + 2 * pad - kw) // stride + 1
    if implicit is not False:
        ok = (A.layout == "spmm" or (A.layout == "sp24" and A.K % 128 == 0)) and A.dtype != torch.float32 and \
            C % 64 == 0 and stride == 1 and A.k > 0
        if ok or implicit:
            x = inp.contiguous()
            Y = torch.empty((Nimg, OH, OW, A.M), dtype=A.dtype, device=inp.device)
            m = A.cstruct()
            with torch.cuda.device(inp.device):
                st = lib().bs_conv2d(ctypes.byref(m), x.data_ptr(), Nimg, H, W, C, kh, kw, pad, stride,
                                     bias.data_ptr() if bias is not None else None, ACTS[act], Y.data_ptr(),
                                     _stream(inp.device))
            if st == 0:
                return Y
            if implicit or fused or st != BS_ERR_UNSUPPORTED:
                _check(st, "bs_conv2d")
        elif fused:
            raise BSError(BS_ERR_UNSUPPORTED, "bs_conv2d (bias/act need the implicit path)")
    X = im2col(inp, kh, kw, pad, stride, out=workspace)
    return spmm(A, X).view(Nimg, OH, OW, A.M)


# ---------------------------------------------------------------- multi-GPU: the all-gather fused into the SpMV

def spmv_allgather(A: BSMatrix, x: torch.Tensor, ag: _AllGather, bias: torch.Tensor | None = None,
                   act: str | None = None, flags: int | None = None):
    """bs_spmv_allgather: this rank's row shard of y = act(W_bs·x + bias), stored by the kernel into every
    rank's y (ag.y[p] + ag.row0). Use through dist.FusedRowShardedBS."""
    _need_cuda(x)
    if x.dtype != A.dtype or x.numel() != A.K or not x.is_contiguous():
        raise ValueError("x must be a contiguous vector of A.K elements of A.dtype")
    if bias is not None and (bias.dtype != A.dtype or bias.numel() != A.M or not bias.is_cuda):
        raise ValueError("bias must be a CUDA vector of A.M elements of A.dtype")
    if act not in ACTS:
        raise ValueError(f"act must be one of {sorted(k for k in ACTS if k)}")
    _same_device(A, x, bias)
    m = A.cstruct()
    with torch.cuda.device(x.device):
        st = lib().bs_spmv_allgather(ctypes.byref(m), x.data_ptr(), bias.data_ptr() if bias is not None else None,
                                     ACTS[act], ctypes.byref(ag), bs_flags_default() if flags is None else flags,
                                     _stream(x.device))
    _check(st, "bs_spmv_allgather")


def allgather_wait(ag: _AllGather, device):
    """bs_allgather_wait on the current stream of `device`."""
    with torch.cuda.device(device):
        st = lib().bs_allgather_wait(ctypes.byref(ag), _stream(device))
    _check(st, "bs_allgather_wait")


# ---------------------------------------------------------------- a stack of layers as one CUDA graph (o_time)

class LayerStack:
    """A stack of balanced-sparse FC layers y_{i+1} = act_i(W_i·y_i + b_i) (Eq. 1 with its +B) run as
    one CUDA graph: the per-layer launch cost the paper calls o_time becomes a graph node, and
    every layer launches with PDL + static weights, so its weight stream starts while the previous layer
    finishes. ``layers`` is a list of (BSMatrix, bias or None, act or None); each K must equal the previous M.
    Call with x (device, K of the first layer); returns the last y (a view of a buffer the next call
    overwrites)."""

    def __init__(self, layers):
        if not layers:
            raise ValueError("at least one layer")
        for (a0, _, _), (a1, _, _) in zip(layers, layers[1:]):
            if a1.K != a0.M or a1.dtype != a0.dtype:
                raise ValueError("layer K must equal the previous layer's M (same dtype)")
        self.layers = layers
        dev = layers[0][0].packed.device
        dt = layers[0][0].dtype
        self.x = torch.zeros(layers[0][0].K, dtype=dt, device=dev)
        self.ys = [torch.empty(A.M, dtype=dt, device=dev) for A, _, _ in layers]
        self.graph = None

    def _run(self):
        cur = self.x
        fl = SPMV_PDL | SPMV_W_STATIC
        for (A, b, act), y in zip(self.layers, self.ys):
            spmv(A, cur, out=y, flags=fl, bias=b, act=act)
            cur = y
        return cur

    def capture(self):
        """Record the stack once (after a warm-up on a side stream, as torch requires)."""
        s = torch.cuda.Stream(device=self.x.device)
        s.wait_stream(torch.cuda.current_stream(self.x.device))
        with torch.cuda.stream(s):
            for _ in range(2):
                self._run()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=s):
                self._run()
        torch.cuda.current_stream(self.x.device).wait_stream(s)
        return self

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        self.x.copy_(x)
        if self.graph is None:
            return self._run()
        self.graph.replay()
        return self.ys[-1]
