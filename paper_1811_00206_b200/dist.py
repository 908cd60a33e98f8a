"""Multi-GPU layer: output-row sharding with an all-gather of y, and batch sharding of SpMM.

The method shards cleanly by rows. Every row has its own blocks and the same nnz, so a row
slice of W_bs is itself a balanced-sparse matrix, and each rank prunes and packs its slice on its
own. The only exchange is the all-gather of the y slices. One process per GPU; the
collective is NCCL over NVLink, bootstrapped by torch.distributed. Host-side logic (slice ranges,
padding, gather order) is covered by world_size-2 gloo tests on CPU.

Row sharding is bit-identical to the unsharded product. The SpMV kernel's arithmetic for a row does
not depend on which rows share its launch (see spmv.cu).
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def row_range(M: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [r0, r1) owned by `rank`: consecutive slices of ceil(M/world) rows (the last may be shorter)."""
    per = -(-M // world)
    r0 = min(rank * per, M)
    return r0, min(r0 + per, M)


def rows_per_rank(M: int, world: int) -> int:
    return -(-M // world)


class RowShardedBS:
    """y = W_bs·x with W_bs's rows split across the ranks of `group`.

    ``local`` is this rank's packed slice (a BSMatrix, or anything ``local_fn`` accepts). ``forward``
    runs the local SpMV on the current stream, then all-gathers the padded y slices into the full y.
    """

    def __init__(self, local, M: int, group=None, local_fn: Callable | None = None):
        self.local = local
        self.M = M
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.per = rows_per_rank(M, self.world)
        r0, r1 = row_range(M, self.world, self.rank)
        self.r0, self.r1 = r0, r1
        if local_fn is None:
            from . import spmv as local_fn  # the CUDA path
        self.local_fn = local_fn

    def forward(self, x: torch.Tensor, y_local_buf: torch.Tensor | None = None,
                y_full_buf: torch.Tensor | None = None) -> torch.Tensor:
        n_local = self.r1 - self.r0
        if y_local_buf is None:
            y_local_buf = torch.zeros(self.per, dtype=x.dtype, device=x.device)
        if n_local > 0:
            self.local_fn(self.local, x, out=y_local_buf[:n_local])
        if y_full_buf is None:
            y_full_buf = torch.empty(self.per * self.world, dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(y_full_buf, y_local_buf, group=self.group)
        return y_full_buf[: self.M]

    __call__ = forward


def batch_range(N: int, world: int, rank: int) -> tuple[int, int]:
    """Batch columns [n0, n1) of X owned by `rank` for batch-sharded SpMM (W_bs replicated)."""
    return row_range(N, world, rank)


class BatchShardedBS:
    """Y = W_bs·X with W_bs replicated and the N batch columns split across ranks.

    No exchange is needed unless every rank needs the whole Y (``gather=True``)."""

    def __init__(self, A, group=None, local_fn: Callable | None = None):
        self.A = A
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if local_fn is None:
            from . import spmm as local_fn
        self.local_fn = local_fn

    def forward(self, X: torch.Tensor, gather: bool = False) -> torch.Tensor:
        N = X.shape[0]
        n0, n1 = batch_range(N, self.world, self.rank)
        Y_local = self.local_fn(self.A, X[n0:n1]) if n1 > n0 else X.new_empty((0, self.A.M))
        if not gather:
            return Y_local
        per = -(-N // self.world)
        buf = X.new_zeros((per, self.A.M))
        buf[: n1 - n0] = Y_local
        full = X.new_empty((per * self.world, self.A.M))
        dist.all_gather_into_tensor(full, buf, group=self.group)
        return full[:N]

    __call__ = forward
