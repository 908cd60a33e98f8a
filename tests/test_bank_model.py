"""T2: a host model of shared-memory bank conflicts over the build's OWN x-slot function
(bs_x_slot_offset, the function the SpMV kernel stages x through), for every gather a warp step issues.

The paper's claim (Fig. 3): with the dense vector "rearranged and stored in shared memory",
the threads of one step read "V[0], V[4], V[9], V[13] simultaneously" with no bank conflict, whatever the
kept indices are. In the kernel a warp step, for owned block v, has lane l read x at (block 32·g + l,
offset o_l) with o_l arbitrary in [0, B). The model: 32 banks of 4-byte words; a request of w-byte accesses
is served in phases of 128 bytes (w <= 4: one phase of 32 lanes; w = 8: two of 16; w = 16: four of 8);
in a phase, lanes reading the same word are a broadcast and distinct words in one bank serialise.
Conflict factor = wavefronts / phases; the layout is conflict-free iff it is 1 for every offset vector.
A naive row-major x is the negative control (the model must see its conflicts).
"""
import itertools

import numpy as np
import pytest

import oracle



@pytest.fixture(scope="module")
def bs():
    import __graft_entry__
    __graft_entry__._build_module().build()
    import paper_1811_00206_b200 as bs
    return bs


def wavefronts(addrs, width):
    """Shared-memory wavefronts of one warp request (lane i reads `width` bytes at addrs[i])."""
    per_phase = 32 if width <= 4 else 128 // width
    total = 0
    for p0 in range(0, len(addrs), per_phase):
        banks = {}
        for a in addrs[p0:p0 + per_phase]:
            for wd in range(a // 4, (a + max(width, 1) - 1) // 4 + 1):
                banks.setdefault(wd % 32, set()).add(wd)
        total += max(len(s) for s in banks.values())
    return total, -(-len(addrs) // per_phase)


def gather_factor(bs, K, B, dt, nv, g, offsets):
    es = 4 if dt == oracle.F32 else 2
    width = es if nv == 1 else 2 * nv
    addrs = [bs.lib().bs_x_slot_offset(K, B, dt, nv, 32 * g + l, int(offsets[l]), 0) for l in range(32)]
    assert min(addrs) >= 0
    if width == 32:  # NV = 16: two 16-byte loads per slot (parts 0 and 1)
        a2 = [bs.lib().bs_x_slot_offset(K, B, dt, nv, 32 * g + l, int(offsets[l]), 1) for l in range(32)]
        assert sorted({abs(x - y) for x, y in zip(addrs, a2)}) == [16]
        w1, p1 = wavefronts(addrs, 16)
        w2, p2 = wavefronts(a2, 16)
        return (w1 + w2) / (p1 + p2)
    w, p = wavefronts(addrs, width)
    return w / p


def offset_vectors(B, rng, n=200):
    yield np.zeros(32, dtype=int)                     # every block keeps the same offset (same-offset family)
    yield np.full(32, B - 1)
    yield np.arange(32) % B                            # consecutive offsets
    yield (np.arange(32) * 7) % B
    yield (np.arange(32) // 2) % B                     # pairs of lanes on one offset
    for _ in range(n):
        yield rng.integers(0, B, 32)


CONFIGS = [  # (K, B, dtype, nv): V = 1, 2, 4, 8 (paired 16-bit groups), f32, and every batch width
    (65536, 32, oracle.F16, 1), (25088, 32, oracle.BF16, 1), (3008, 32, oracle.F16, 1), (2048, 32, oracle.F16, 1),
    (1024, 32, oracle.F16, 1), (4096, 32, oracle.F32, 1), (8192, 16, oracle.F16, 1), (640, 20, oracle.F16, 1),
    (2048, 512, oracle.F16, 1), (4000, 25, oracle.F32, 1),
    (16384, 32, oracle.F16, 2), (16384, 32, oracle.F16, 4), (16384, 32, oracle.F16, 8), (2048, 32, oracle.BF16, 16),
]


@pytest.mark.parametrize("K,B,dt,nv", CONFIGS)
def test_gathers_conflict_free(bs, K, B, dt, nv):
    rng = np.random.default_rng(K + B + nv)
    NB = K // B
    groups = sorted({0, 1, 2, 3, (NB - 1) // 32} & set(range((NB + 31) // 32)))
    for g in groups:
        if 32 * g + 31 >= NB:  # a partial last group: only full groups are modelled
            continue
        for offs in offset_vectors(B, rng):
            f = gather_factor(bs, K, B, dt, nv, g, offs)
            assert f == 1.0, (K, B, dt, nv, g, offs.tolist(), f)


def test_fig3_instance(bs):
    """Fig. 3: 16-element x, 4 blocks of 4; one step reads V[0], V[4], V[9], V[13] (offsets 0, 0, 1,
    1 of blocks 0..3) in one wavefront."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))["bank_fig3"]
    K, B = g["K"], g["block"]
    idx = g["group"]
    addrs = [bs.lib().bs_x_slot_offset(K, B, oracle.F32, 1, e // B, e % B, 0) for e in idx]
    assert [e // B for e in idx] == [0, 1, 2, 3]
    w, p = wavefronts(addrs, 4)
    assert (w, p) == (1, 1)
    # natural (unrearranged) order: element e at byte 4e. Here blocks 0..3 hit banks 0, 4, 9, 13 (no
    # conflict either), but one offset per lane across 32 blocks of 32 collides in one bank:
    nat = [4 * (b * 32 + 5) for b in range(32)]
    assert wavefronts(nat, 4) == (32, 1)


def test_model_detects_conflicts():
    """Negative control: a naive x (row-major, 2-byte elements) is 16-way conflicted when all lanes read
    the same offset of their blocks; the model is not vacuous."""
    addrs = [2 * (32 * l + 3) for l in range(32)]
    w, p = wavefronts(addrs, 2)
    assert w == 16 and p == 1
    # lanes reading different halves of one word: a broadcast, not a conflict
    assert wavefronts([0, 2] * 16, 2) == (1, 1)


def test_slot_offsets_are_injective(bs):
    """Distinct (block, offset) pairs of one chunk never share a slot (the rearrangement is a permutation)."""
    for K, B, dt, nv in ((2048, 32, oracle.F16, 1), (4096, 32, oracle.F32, 1), (1024, 32, oracle.F16, 8),
                         (640, 20, oracle.F16, 1)):
        es = 4 if dt == oracle.F32 else 2
        width = es if nv == 1 else 2 * nv
        seen = set()
        for b, o in itertools.product(range(K // B), range(B)):
            a = bs.lib().bs_x_slot_offset(K, B, dt, nv, b, o, 0)
            assert a % width == 0 or nv == 1
            assert a not in seen
            seen.add(a)
