"""CPU checks of the C-ABI library: it builds, loads, exports every symbol include/bs.h declares, and its
pure host helpers agree with the oracle's independent geometry. No device compute is called here."""
import ctypes
import os
import re

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "bs.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|double|size_t|const char\*)\s+(bs_[a-z0-9_]+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def bs():
    import __graft_entry__
    __graft_entry__._build_module().build()
    import paper_1811_00206_b200 as bs
    return bs


def test_header_declares_the_boundary():
    syms = _declared_symbols()
    for s in ("bs_prune", "bs_prune_k", "bs_pack", "bs_unpack", "bs_spmv", "bs_spmv_ex", "bs_spmv_fused", "bs_spmv_host", "bs_spmm", "bs_block_rank",
              "bs_packed_bytes", "bs_k_from_sparsity", "bs_status_str", "bs_version"):
        assert s in syms


def test_library_exports_every_declared_symbol(bs):
    L = ctypes.CDLL(bs.LIB_PATH)
    for s in _declared_symbols():
        assert hasattr(L, s), f"{s} not exported"
    assert set(bs.EXPORTS) == set(_declared_symbols())


def test_version_names_sm100a(bs):
    assert "sm_100a" in bs.version()


def test_k_matches_oracle(bs):
    for B in (1, 4, 16, 25, 32, 100, 1024):
        for s in (0.0, 0.1, 0.5, 0.7, 0.75, 0.875, 0.9, 0.95, 0.97, 0.999):
            assert bs.k_from_sparsity(B, s) == oracle.k_from_sparsity(B, s)
    assert bs.k_from_sparsity(32, 1.0) == -1


def test_packed_bytes_matches_oracle(bs):
    import torch
    tdt = {oracle.F32: torch.float32, oracle.F16: torch.float16, oracle.BF16: torch.bfloat16}
    lay = {oracle.SPMV: "spmv", oracle.SPMM: "spmm", oracle.SP24: "sp24"}
    for M, K, B, k in ((64, 64, 16, 8), (6000, 3008, 32, 3), (4096, 25088, 32, 3), (7, 2048, 512, 9), (5, 96, 1, 1),
                       (65536, 65536, 32, 3), (33, 1000, 25, 8), (9, 64, 4, 2), (4, 30, 4, 2)):
        for dt in tdt:
            for L in lay:
                assert bs.packed_bytes(M, K, B, k, tdt[dt], lay[L]) == oracle.packed_bytes(M, K, B, k, dt, L)


def test_choose_layout(bs):
    """bs_choose_layout (host helper): 2:4 shapes -> sp24; batch <= 8 -> spmv; larger 16-bit batches with
    B | 64 -> spmm; f32 -> spmv; invalid arguments rejected."""
    import torch
    f16, f32 = torch.float16, torch.float32
    assert bs.choose_layout(4096, 2048, 4, 2, f16, 1) == "sp24"
    assert bs.choose_layout(4096, 2048, 4, 2, f16, 64) == "sp24"
    assert bs.choose_layout(4096, 2000, 4, 2, f16, 64) == "spmm"  # K mod 128 != 0: no TMA chunking
    for N in (1, 2, 8):
        assert bs.choose_layout(4096, 25088, 32, 3, f16, N) == "spmv"
    assert bs.choose_layout(4096, 25088, 32, 3, f16, 32) == "spmm"
    assert bs.choose_layout(4096, 25088, 32, 3, f16, 16) == "spmm"
    assert bs.choose_layout(4096, 2048, 32, 4, f16, 16) == "spmv"  # one 16-column pass (CTC)
    assert bs.choose_layout(4096, 2048, 32, 4, f16, 17) == "spmm"
    assert bs.choose_layout(4096, 25088, 32, 3, f32, 32) == "spmv"
    assert bs.choose_layout(64, 1000, 25, 8, f16, 32) == "spmv"  # 25 does not divide 64
    with pytest.raises(ValueError):
        bs.choose_layout(64, 1000, 32, 3, f16, 4)  # K mod B != 0


def test_no_oracle_in_product_path():
    """The product package never imports, links or runs anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_1811_00206_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text and "liboracle" not in text, f


def test_schedule_and_keep_count_match_oracle(bs):
    """Host helpers of Alg. 1's schedule (bs_schedule_sparsity, bs_keep_count) agree with the oracle."""
    for target in (0.0, 0.5, 0.875, 0.9, 0.97):
        for n in (1, 4, 10, 33):
            for i in range(n + 1):
                assert bs.schedule(target, n, i) == oracle.schedule(target, n, i)
    with pytest.raises(ValueError):
        bs.schedule(0.9, 10, 11)
    for n in (1, 7, 64, 4096 * 4096, 65536 * 65536):
        for s in (0.0, 0.3, 0.5, 0.9, 0.97):
            assert bs.keep_count(n, s) == oracle.keep_count(n, s)
    assert bs.lib().bs_pattern_workspace_bytes(64, 64, 8, 8) > bs.lib().bs_pattern_workspace_bytes(64, 64, 0, 0) > 0
    assert bs.lib().bs_pattern_workspace_bytes(64, 64, 7, 8) == 0
