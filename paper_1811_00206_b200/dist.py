"""Multi-GPU layer: output-row sharding with an all-gather of y, and batch sharding of SpMM.

The method shards cleanly by rows. Every row has its own blocks and the same nnz, so a row
slice of W_bs is itself a balanced-sparse matrix, and each rank prunes and packs its slice on its
own. The only exchange is the all-gather of the y slices. One process per GPU,
bootstrapped by torch.distributed. Three ways to run the exchange:

  RowShardedBS            local bs_spmv, then one NCCL all_gather_into_tensor (the baseline).
  PipelinedRowShardedBS   rows dealt block-cyclically in chunks of R rows; chunk j's all-gather runs on
                          a side stream while chunk j+1's SpMV computes (SURVEY §8(e) mitigation 1).
  FusedRowShardedBS       bs_spmv_allgather: the SpMV kernel stores its rows straight into every rank's
                          y over NVLink (peer-mapped buffers) and raises a flag; bs_allgather_wait
                          gates the consumer. No separate collective launch (NEXT-1, mitigation 2).

Row sharding is bit-identical to the unsharded product: the SpMV's arithmetic for a row does not
depend on which rows share its launch (spmv.cu). `should_shard` is the policy of SURVEY §8(e): shard
only when the time saved beats the all-gather, t1 - t1/P > t_allgather (BJ.north_star: "Nothing is
partitioned where a layer fits and runs faster on one GPU"), with t_allgather measured live by
`measure_allgather_us`.

Host-side logic (slice ranges, cyclic chunks, padding, gather order, epochs and buffer parity) is
covered by world-size-2 gloo tests on CPU; the fused kernel protocol by a single-GPU simulation of P
ranks (tests/test_gpu_dist.py).
"""
from __future__ import annotations

import ctypes
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


def cyclic_chunks(M: int, world: int, rank: int, R: int) -> list[tuple[int, int]]:
    """Block-cyclic row ownership with chunks of R rows: rank r owns chunk j = rows
    [(j·P + r)·R, (j·P + r + 1)·R) ∩ [0, M) for j = 0, 1, ... (empty ranges kept so every rank has the
    same chunk count). All ranks' chunk j together are the contiguous rows [j·P·R, (j+1)·P·R)."""
    nj = -(-M // (world * R))
    out = []
    for j in range(nj):
        a = (j * world + rank) * R
        out.append((min(a, M), min(a + R, M)))
    return out


def should_shard(t1_us: float, world: int, t_allgather_us: float) -> bool:
    """shard a layer over `world` GPUs only if the compute saved exceeds the exchange,
    t1 − t1/P > t_allgather."""
    return world > 1 and t1_us - t1_us / world > t_allgather_us


def measure_allgather_us(nbytes: int, group=None, device=None, iters: int = 50) -> float:
    """Device time of one all_gather_into_tensor of `nbytes` per rank on `group` (max over ranks),
    for should_shard."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    world = dist.get_world_size(group)
    src = torch.zeros(max(1, nbytes), dtype=torch.uint8, device=device)
    dst = torch.empty(src.numel() * world, dtype=torch.uint8, device=device)
    for _ in range(5):
        dist.all_gather_into_tensor(dst, src, group=group)
    torch.cuda.synchronize(device)
    dist.barrier(group)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        dist.all_gather_into_tensor(dst, src, group=group)
    e1.record()
    torch.cuda.synchronize(device)
    t = torch.tensor([e0.elapsed_time(e1) * 1e3 / iters], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class RowShardedBS:
    """y = W_bs·x with W_bs's rows split across the ranks of `group`.

    ``local`` is this rank's packed slice (a BSMatrix, or anything ``local_fn`` accepts). ``forward``
    runs the local SpMV on the current stream, then all-gathers the padded y slices into the full y.
    The slice and gather buffers are allocated once per (dtype, device) and reused; pass your own to
    control their lifetime.
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
        self._bufs = {}

    def buffers(self, dtype, device):
        key = (dtype, str(device))
        if key not in self._bufs:
            self._bufs[key] = (torch.zeros(self.per, dtype=dtype, device=device),
                               torch.empty(self.per * self.world, dtype=dtype, device=device))
        return self._bufs[key]

    def forward(self, x: torch.Tensor, y_local_buf: torch.Tensor | None = None,
                y_full_buf: torch.Tensor | None = None) -> torch.Tensor:
        n_local = self.r1 - self.r0
        if y_local_buf is None or y_full_buf is None:
            lb, fb = self.buffers(x.dtype, x.device)
            y_local_buf = lb if y_local_buf is None else y_local_buf
            y_full_buf = fb if y_full_buf is None else y_full_buf
        if n_local > 0:
            self.local_fn(self.local, x, out=y_local_buf[:n_local])
        dist.all_gather_into_tensor(y_full_buf, y_local_buf, group=self.group)
        return y_full_buf[: self.M]

    __call__ = forward


class PipelinedRowShardedBS:
    """Row sharding with the all-gather pipelined against the SpMV: rows are dealt block-cyclically in
    chunks of R rows (cyclic_chunks), ``locals`` holds this rank's packed chunk matrices in chunk order
    (None for an empty chunk). Chunk j's SpMV runs on the current stream; its all-gather, which fills
    the contiguous rows [j·P·R, (j+1)·P·R) of y, runs on a side stream after an event, so it overlaps
    chunk j+1's SpMV. The result is bit-identical to RowShardedBS (the same rows, the same kernel)."""

    def __init__(self, locals_, M: int, R: int, group=None, local_fn: Callable | None = None):
        self.locals = list(locals_)
        self.M, self.R = M, R
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.chunks = cyclic_chunks(M, self.world, self.rank, R)
        assert len(self.locals) == len(self.chunks), "one packed matrix (or None) per chunk"
        if local_fn is None:
            from . import spmv as local_fn
        self.local_fn = local_fn
        self._bufs = {}
        self._side = None

    def buffers(self, dtype, device):
        key = (dtype, str(device))
        if key not in self._bufs:
            nj = len(self.chunks)
            self._bufs[key] = (torch.zeros((nj, self.R), dtype=dtype, device=device),
                               torch.empty(nj * self.world * self.R, dtype=dtype, device=device))
        return self._bufs[key]

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        loc, full = self.buffers(x.dtype, x.device)
        cur = torch.cuda.current_stream(x.device) if x.is_cuda else None
        if x.is_cuda and self._side is None:
            self._side = torch.cuda.Stream(device=x.device)
        PR = self.world * self.R
        for j, (a, b) in enumerate(self.chunks):
            if b > a:
                self.local_fn(self.locals[j], x, out=loc[j, : b - a])
            if cur is not None:
                ev = torch.cuda.Event()
                ev.record(cur)
                self._side.wait_event(ev)
                with torch.cuda.stream(self._side):
                    dist.all_gather_into_tensor(full[j * PR:(j + 1) * PR], loc[j], group=self.group)
            else:
                dist.all_gather_into_tensor(full[j * PR:(j + 1) * PR], loc[j], group=self.group)
        if cur is not None:
            ev = torch.cuda.Event()
            ev.record(self._side)
            cur.wait_event(ev)
        return full[: self.M]

    __call__ = forward


class FusedRowShardedBS:
    """Row sharding with the all-gather fused into the SpMV (bs_spmv_allgather, NEXT-1).

    Every rank holds two full y buffers (alternated by epoch parity), nranks arrival flags and one CTA
    counter, all mapped into every rank through CUDA IPC (bs_peer_export / bs_peer_import, handles
    exchanged with all_gather_object on `group`). ``forward(x)`` launches the shard's SpMV, whose
    epilogue writes the rows into all ranks' y, then bs_allgather_wait; the returned y (a view of the
    current buffer) is complete on this stream. Consume it before the call after next (two buffers).

    ``peers`` bypasses the IPC exchange: a dict with the y buffers, flag and counter tensors of every
    rank already addressable from this process (the single-GPU simulation of P ranks in the tests)."""

    def __init__(self, local, M: int, dtype: torch.dtype, device, group=None, rank: int | None = None,
                 world: int | None = None, row0: int | None = None, peers: dict | None = None):
        from . import lib
        self.local = local
        self.M = M
        self.group = group
        self.world = world if world is not None else dist.get_world_size(group)
        self.rank = rank if rank is not None else dist.get_rank(group)
        if self.world > 8:
            raise ValueError("bs_spmv_allgather maps at most 8 ranks")
        self.row0 = row0 if row0 is not None else row_range(M, self.world, self.rank)[0]
        self.epoch = 0
        self._imported = []
        if peers is None:
            self.y_bufs = [torch.empty(M, dtype=dtype, device=device) for _ in range(2)]
            self.flags = torch.zeros(self.world, dtype=torch.int32, device=device)
            self.counter = torch.zeros(1, dtype=torch.int32, device=device)
            torch.cuda.synchronize(device)
            mine = [self._export(t) for t in (*self.y_bufs, self.flags)]
            allh = [None] * self.world
            dist.all_gather_object(allh, mine, group=group)
            ptrs = []
            for q in range(self.world):
                if q == self.rank:
                    ptrs.append([t.data_ptr() for t in (*self.y_bufs, self.flags)])
                else:
                    row = []
                    for h, off in allh[q]:
                        p = ctypes.c_void_p()
                        st = lib().bs_peer_import(h, off, ctypes.byref(p))
                        if st != 0:
                            raise RuntimeError(f"bs_peer_import failed ({st}): no P2P mapping between the GPUs")
                        self._imported.append((p.value, off))
                        row.append(p.value)
                    ptrs.append(row)
            self.y_ptrs = [[ptrs[q][b] for q in range(self.world)] for b in range(2)]
            self.flag_ptrs = [ptrs[q][2] for q in range(self.world)]
        else:
            self.y_bufs = peers["y"][self.rank]
            self.flags = peers["flags"][self.rank]
            self.counter = peers["counter"][self.rank]
            self.y_ptrs = [[peers["y"][q][b].data_ptr() for q in range(self.world)] for b in range(2)]
            self.flag_ptrs = [peers["flags"][q].data_ptr() for q in range(self.world)]

    @staticmethod
    def _export(t: torch.Tensor):
        from . import lib
        h = ctypes.create_string_buffer(64)
        off = ctypes.c_int64()
        st = lib().bs_peer_export(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off))
        if st != 0:
            raise RuntimeError(f"bs_peer_export failed ({st})")
        return bytes(h.raw), off.value

    @staticmethod
    def make_peers(world: int, M: int, dtype: torch.dtype, device) -> dict:
        """Buffers of `world` simulated ranks on one device (tests)."""
        return {"y": [[torch.empty(M, dtype=dtype, device=device) for _ in range(2)] for _ in range(world)],
                "flags": [torch.zeros(world, dtype=torch.int32, device=device) for _ in range(world)],
                "counter": [torch.zeros(1, dtype=torch.int32, device=device) for _ in range(world)]}

    def _ag(self):
        from . import _AllGather
        ag = _AllGather()
        ag.nranks, ag.rank, ag.row0 = self.world, self.rank, self.row0
        for q in range(self.world):
            ag.y[q] = self.y_ptrs[self.epoch % 2][q]
            ag.flags[q] = self.flag_ptrs[q]
        ag.counter = self.counter.data_ptr()
        ag.epoch = self.epoch
        return ag

    def launch(self, x: torch.Tensor, bias: torch.Tensor | None = None, act: str | None = None):
        """Step 1-2 of the protocol (the SpMV with its fused stores); returns the epoch's y buffer."""
        from . import spmv_allgather
        self.epoch += 1
        spmv_allgather(self.local, x, self._ag(), bias=bias, act=act)
        return self.y_bufs[self.epoch % 2]

    def wait(self):
        """Step 3 (bs_allgather_wait on the current stream)."""
        from . import allgather_wait
        allgather_wait(self._ag(), self.flags.device)

    def forward(self, x: torch.Tensor, bias: torch.Tensor | None = None, act: str | None = None) -> torch.Tensor:
        y = self.launch(x, bias=bias, act=act)
        self.wait()
        return y

    __call__ = forward

    def close(self):
        from . import lib
        for p, off in self._imported:
            lib().bs_peer_close(ctypes.c_void_p(p), off)
        self._imported = []


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
