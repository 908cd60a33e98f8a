"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic. It makes random or structured dense matrices and
vectors, and converts tensors to numpy for the oracle. Both sides receive the same bytes. The recipe
is in DESIGN.md §6:

- ``gaussian``: W iid N(0, 1/K) drawn in fp32 and rounded to D. The paper's analysis assumes
  Gaussian priors on w and x. x is iid N(0, 1).
- ``ties``: W uniform on the integers {-2,...,2}. Magnitude ties are everywhere.
- ``intexact``: W and x uniform on {-1, 0, 1}. Every fp32 partial sum is an exact integer, so any
  summation order gives the same y (SURVEY §8(c) pin (ii)).
- ``sameoffset``: |W| strictly decreasing inside every block, with random signs. Every block then
  keeps offsets {0..k-1} (the worst case for any layout in which the bank depends on the offset).

Rows are generated in chunks of ``ROW_CHUNK`` with seed ``seed*1000003 + chunk``, so a row slice
[r0, r1) regenerates byte-identical rows on any rank.
"""
from __future__ import annotations

import numpy as np
import torch

ROW_CHUNK = 4096
BASE_SEED = 1811_00206

TORCH_DT = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}
DT_CODE = {"f32": 0, "f16": 1, "bf16": 2}


def seed_for(config_id: int, sweep_index: int = 0) -> int:
    """seed = 1811_00206 + 100·config_id + sweep_index."""
    return BASE_SEED + 100 * config_id + sweep_index


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    return g


def matrix(M: int, K: int, dtype: str = "f16", family: str = "gaussian", seed: int = BASE_SEED,
           device="cpu", row0: int = 0, B: int | None = None, ld: int | None = None) -> torch.Tensor:
    """Rows [row0, row0+M) of the seeded K-column matrix of ``family``, as a [M, ld] tensor of ``dtype``
    (only the first K columns are meaningful when ld > K).

    Chunks of ROW_CHUNK global rows use their own generator, so any row range is reproducible on its own."""
    tdt = TORCH_DT[dtype]
    ld = K if ld is None else ld
    out = torch.zeros((M, ld), dtype=tdt, device=device)
    r = row0
    end = row0 + M
    while r < end:
        chunk = r // ROW_CHUNK
        c0 = chunk * ROW_CHUNK
        c1 = min(c0 + ROW_CHUNK, end)
        g = _gen(seed * 1000003 + chunk, device)
        n_in_chunk = c1 - c0  # generate from the chunk start so that rows are range-independent
        full = _family_rows(n_in_chunk, K, family, g, device, B)
        lo = r - c0
        out[r - row0:c1 - row0, :K] = full[lo:].to(tdt)
        r = c1
    return out


def _family_rows(n: int, K: int, family: str, g: torch.Generator, device, B: int | None) -> torch.Tensor:
    if family == "gaussian":
        return torch.randn((n, K), generator=g, device=device, dtype=torch.float32) * (1.0 / K ** 0.5)
    if family == "ties":
        return torch.randint(-2, 3, (n, K), generator=g, device=device).to(torch.float32)
    if family == "intexact":
        return torch.randint(-1, 2, (n, K), generator=g, device=device).to(torch.float32)
    if family == "sameoffset":
        assert B is not None, "sameoffset needs the block width"
        j = torch.arange(K, device=device) % B
        mag = (B - j).to(torch.float32) / B  # strictly decreasing inside each block
        sign = torch.randint(0, 2, (n, K), generator=g, device=device).to(torch.float32) * 2 - 1
        return sign * mag
    raise ValueError(f"unknown family {family}")


def vector(K: int, dtype: str = "f16", family: str = "gaussian", seed: int = BASE_SEED + 1, device="cpu",
           n: int | None = None) -> torch.Tensor:
    """x (shape [K]) or X (shape [n, K], torch layout of the K×n operand) for ``family``."""
    g = _gen(seed, device)
    shape = (K,) if n is None else (n, K)
    if family in ("intexact",):
        v = torch.randint(-1, 2, shape, generator=g, device=device).to(torch.float32)
    else:
        v = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    return v.to(TORCH_DT[dtype])


def special_block_matrix(dtype: str = "f32") -> torch.Tensor:
    """A 4×32 matrix whose 16-wide blocks hold ±0, ±Inf, NaN and exact ties (prune parity)."""
    nan, inf = float("nan"), float("inf")
    rows = [
        [0.0, -0.0, 1.0, -1.0, 1.0, 2.0, -2.0, 0.5, -0.5, 3.0, nan, 0.25, -inf, inf, 0.0, 1.0],
        [nan, nan, 1.0, nan, -nan, 0.0, 0.0, 5.0, -5.0, 5.0, inf, -inf, inf, 0.1, 0.2, 0.3],
        [1.0] * 16,
        [-0.0] * 8 + [0.0] * 8,
        [2.0, -2.0] * 8,
        [inf, 1.0, -inf, 2.0] * 4,
        [0.0] * 15 + [nan],
        [float(i) for i in range(16)],
    ]
    t = torch.tensor(rows, dtype=torch.float32).reshape(4, 32)
    return t.to(TORCH_DT[dtype])


def to_numpy(t: torch.Tensor) -> np.ndarray:
    """CPU numpy view for the oracle: f32 -> float32, f16 -> float16, bf16 -> raw uint16 bits."""
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    if t.dtype == torch.uint16:
        return t.numpy()
    return t.numpy()


def from_numpy(a: np.ndarray, dtype: str) -> torch.Tensor:
    """Inverse of to_numpy."""
    if dtype == "bf16":
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(a))
