"""B200-native balanced sparsity (arXiv 1811.00206): thin Python binding over libbs.so.

Every step of the path runs in the CUDA kernels behind the C ABI (include/bs.h). This module only
marshals arguments: it turns torch CUDA tensors into device pointers and passes the current CUDA
stream. There is no CPU fallback. If libbs.so is missing, importing this package raises.

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
           "bs_pack", "bs_unpack", "bs_spmv", "bs_spmv_ex", "bs_spmv_fused", "bs_spmv_host", "bs_spmm", "bs_choose_layout", "bs_block_rank")
ACTS = {None: 0, "none": 0, "relu": 1, "sigmoid": 2, "tanh": 3}  # bs_act (include/bs.h)
SPMV_PDL, SPMV_W_STATIC = 1, 2  # bs_spmv_ex flags (include/bs.h)


class BSError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {_lib.bs_status_str(status).decode()} ({status})")
        self.status = status


class _Matrix(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int64), ("K", ctypes.c_int64), ("block", ctypes.c_int32), ("k", ctypes.c_int32),
                ("dt", ctypes.c_int32), ("layout", ctypes.c_int32), ("packed", ctypes.c_void_p)]


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
    for f in ("bs_prune", "bs_prune_k", "bs_pack", "bs_unpack", "bs_spmv", "bs_spmv_ex", "bs_spmv_fused", "bs_spmv_host", "bs_spmm"):
        getattr(L, f).restype = ci
    return L


_lib = _load()


def lib() -> ctypes.CDLL:
    return _lib


def version() -> str:
    return _lib.bs_version().decode()


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


def k_from_sparsity(block: int, sparsity: float) -> int:
    """k = lround((1 - s)·B)."""
    return _lib.bs_k_from_sparsity(int(block), float(sparsity))


def packed_bytes(M: int, K: int, block: int, k: int, dtype: torch.dtype, layout: str = "spmv") -> int:
    return int(_lib.bs_packed_bytes(M, K, block, k, DTYPES[dtype], LAYOUTS[layout]))


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
        st = _lib.bs_prune_k(W.data_ptr(), _dt(W), M, K, W.stride(0), block, k, vals.data_ptr() if vals.numel() else None,
                             idx.data_ptr() if idx.numel() else None, _stream(W.device))
    _check(st, "bs_prune_k")
    return vals, idx, k


def block_rank(W: torch.Tensor, block: int) -> torch.Tensor:
    """Every element's position in its block's magnitude order (bs_block_rank): uint8 [M, K]. The mask
    of a pruning step at any k is rank < k (Alg. 1's schedule without retraining)."""
    _need_cuda(W)
    M, K = W.shape
    if W.stride(1) != 1:
        W = W.contiguous()
    rank = torch.empty((M, K), dtype=torch.uint8, device=W.device)
    with torch.cuda.device(W.device):
        st = _lib.bs_block_rank(W.data_ptr(), DTYPES[W.dtype], M, K, W.stride(0), block, rank.data_ptr(),
                                _stream(W.device))
    _check(st, "bs_block_rank")
    return rank


def choose_layout(M: int, K: int, block: int, k: int, dtype: torch.dtype, batch: int) -> str:
    """bs_choose_layout: the layout bs_spmm runs fastest on for `batch` columns (include/bs.h)."""
    code = _lib.bs_choose_layout(M, K, block, k, DTYPES[dtype], batch)
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
        st = _lib.bs_pack(vals.data_ptr() if vals.numel() else None, idx.data_ptr() if idx.numel() else None, M, K,
                          block, k, _dt(vals), LAYOUTS[layout], out.data_ptr() if n else None, _stream(vals.device))
    _check(st, "bs_pack")
    return BSMatrix(M, K, block, k, vals.dtype, layout, out)


def unpack(A: BSMatrix):
    """Inverse of pack: canonical (vals, idx)."""
    NB = A.K // A.block
    vals = torch.empty((A.M, NB, A.k), dtype=A.dtype, device=A.packed.device)
    idx = torch.empty((A.M, NB, A.k), dtype=torch.int16, device=A.packed.device)
    with torch.cuda.device(A.packed.device):
        st = _lib.bs_unpack(A.packed.data_ptr() if A.packed.numel() else None, A.M, A.K, A.block, A.k, DTYPES[A.dtype], LAYOUTS[A.layout],
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
    x = x.contiguous()
    y = out if out is not None else torch.empty(A.M, dtype=A.dtype, device=x.device)
    m = A.cstruct()
    with torch.cuda.device(x.device):
        if bias is not None or act is not None:
            if act not in ACTS:
                raise ValueError(f"act must be one of {sorted(k for k in ACTS if k)}")
            if bias is not None:
                _need_cuda(bias)
                if bias.dtype != A.dtype or bias.numel() != A.M:
                    raise ValueError("bias must have A.M elements of A.dtype")
                bias = bias.contiguous()
            st = _lib.bs_spmv_fused(ctypes.byref(m), x.data_ptr(), bias.data_ptr() if bias is not None else None,
                                    ACTS[act], y.data_ptr(), bs_flags_default() if flags is None else flags,
                                    _stream(x.device))
        elif flags is None:
            st = _lib.bs_spmv(ctypes.byref(m), x.data_ptr(), y.data_ptr(), _stream(x.device))
        else:
            st = _lib.bs_spmv_ex(ctypes.byref(m), x.data_ptr(), y.data_ptr(), flags, _stream(x.device))
    _check(st, "bs_spmv")
    return y


def bs_flags_default() -> int:
    """The launch flags bs_spmv uses (PDL)."""
    return SPMV_PDL


def spmv_host(A: BSMatrix, x_host: torch.Tensor, y_host: torch.Tensor, x_dev: torch.Tensor, y_dev: torch.Tensor):
    """End-to-end product through the C ABI with host buffers: H2D(x) -> SpMV -> D2H(y), enqueued on the
    current stream (bs_spmv_host). y_host is valid after the stream synchronises."""
    m = A.cstruct()
    with torch.cuda.device(x_dev.device):
        st = _lib.bs_spmv_host(ctypes.byref(m), x_host.data_ptr(), y_host.data_ptr(), x_dev.data_ptr(),
                               y_dev.data_ptr(), _stream(x_dev.device))
    _check(st, "bs_spmv_host")


def spmm(A: BSMatrix, X: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Y = W_bs·X for a batch. X: [N, K] (row n = column n of the K×N operand); returns Y: [N, M]."""
    _need_cuda(X)
    if X.dim() != 2 or X.shape[1] != A.K or X.dtype != A.dtype or X.stride(1) != 1:
        raise ValueError("X must be [N, K] of A.dtype with unit column stride")
    N = X.shape[0]
    Y = out if out is not None else torch.empty((N, A.M), dtype=A.dtype, device=X.device)
    m = A.cstruct()
    with torch.cuda.device(X.device):
        st = _lib.bs_spmm(ctypes.byref(m), X.data_ptr(), N, X.stride(0), Y.data_ptr(), Y.stride(0), _stream(X.device))
    _check(st, "bs_spmm")
    return Y
