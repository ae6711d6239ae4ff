"""CPU checks of the shared-memory tile layout of the 8x8 kernel (expm_n8.cuh).

The unit slot must be a bijection and bank-conflict-free per access phase
(8 lanes for 16-byte, 16 lanes for 8-byte shared accesses) for every access
pattern the kernel issues. Mirrors unit8() in expm_n8.cuh.
"""
import re

from conftest import ROOT


def slot(i, c):
    return ((i >> 1) << 3) | (((i & 1) ^ (i >> 2)) << 2) | ((((c >> 1) ^ (i >> 1)) & 1) << 1) | (c & 1)


def word(i, j):
    return slot(i, j >> 1) * 2 + (j & 1)


def test_formula_matches_kernel_source():
    src = open(f"{ROOT}/paper_1710_10989_b200/csrc/expm_n8.cuh").read()
    assert "((i >> 1) << 3) | (((i & 1) ^ (i >> 2)) << 2) |" in src
    assert "((((c >> 1) ^ (i >> 1)) & 1) << 1) | (c & 1)" in src


def test_bijection_and_xor_structure():
    assert sorted(slot(i, c) for i in range(8) for c in range(4)) == list(range(32))
    assert all(slot(k, q) == slot(k, 0) ^ q for k in range(8) for q in range(4))


def test_store_conflict_free_per_quarter_warp():
    for p in range(4):
        groups = [slot(l >> 2, l & 3) % 8 for l in range(8 * p, 8 * p + 8)]
        assert len(set(groups)) == 8


def test_transposed_loads_conflict_free_per_half_warp():
    for which in (0, 1):
        for p in range(2):
            pairs = [word(2 * (l & 3) + which, l >> 2) % 16 for l in range(16 * p, 16 * p + 16)]
            assert len(set(pairs)) == 16


def test_exact_path_and_norm_loads():
    for cc in range(4):
        for p in range(4):
            units = {slot(l >> 2, cc) for l in range(8 * p, 8 * p + 8)}
            assert len({u % 8 for u in units}) == len(units)
    for k in range(8):
        for p in range(4):
            units = {slot(k, l & 3) for l in range(8 * p, 8 * p + 8)}
            assert len({u % 8 for u in units}) == len(units)
    for i in range(8):
        assert len({word(i, l) % 16 for l in range(8)}) == 8
