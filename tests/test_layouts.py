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


# ---- fp32 operand buffers (expm_small_f32.cu, n = 32 and 64) ----
# chunk c (16 bytes) of row i is stored at chunk c ^ swz(i); a lane (ti, tj)
# owns rows 4 ti + r and the column chunks tj and tj + GC (GC = n / 8).

def swz32(i):
    t = (i >> 2) & 7
    return ((t & 1) << 2) | (t >> 1)


def quad(n, i, c):
    """bank quad (16-byte bank group, 8 per 128 bytes) of chunk c of row i"""
    return (i * n // 4 + (c ^ swz32(i))) % 8


def lanes(n, warp):
    gc = n // 8
    for l in range(32):
        tid = 32 * warp + l
        yield l, tid // gc, tid % gc


def test_fp32_swizzle_formula_matches_kernel_source():
    src = open(f"{ROOT}/paper_1710_10989_b200/csrc/expm_small_f32.cu").read()
    assert "const int t = (i >> 2) & 7;" in src
    assert "return ((t & 1) << 2) | (t >> 1);" in src


def test_fp32_swizzle_is_a_row_permutation():
    for n in (32, 64):
        for i in range(n):
            assert sorted(c ^ swz32(i) for c in range(n // 4)) == list(range(n // 4))


def test_fp32_fragment_stores_conflict_free():
    """STS.128 of (row 4ti + r, chunk tj + h GC): 8 distinct bank quads per
    quarter warp."""
    for n, warps in ((32, 1), (64, 4)):
        gc = n // 8
        for w in range(warps):
            ls = list(lanes(n, w))
            for r in range(4):
                for h in range(2):
                    for p in range(4):
                        q = {quad(n, 4 * ti + r, tj + h * gc) for l, ti, tj in ls[8 * p:8 * p + 8]}
                        assert len(q) == 8, (n, w, r, h, p)


def test_fp32_operand_loads_conflict_free():
    """X chunk loads (rows 4ti + r, chunk q) and Y row loads (row k, chunks
    tj + h GC): per quarter warp, distinct addresses sit in distinct bank
    quads (lanes sharing an address are a broadcast)."""
    for n, warps in ((32, 1), (64, 4)):
        gc = n // 8
        for w in range(warps):
            ls = list(lanes(n, w))
            for p in range(4):
                ph = ls[8 * p:8 * p + 8]
                for r in range(4):
                    for q in range(n // 4):
                        addrs = {(4 * ti + r, q) for l, ti, tj in ph}
                        assert len({quad(n, i, c) for i, c in addrs}) == len(addrs)
                for k in range(n):
                    for h in range(2):
                        addrs = {(k, tj + h * gc) for l, ti, tj in ph}
                        assert len({quad(n, i, c) for i, c in addrs}) == len(addrs)
