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


# ---- the quad lane mapping of the reference-rounded path (Group8T::set_lanes) ----
# An aligned quad of lanes owns a 2x2 block of units. The shared-memory pipe
# merges identical addresses only inside an aligned lane quad and serves 8
# (quad, address) requests per 128-bit wavefront, at least 2 wavefronts per
# LDS.128 (tools/lds_patterns.cu, profiles/lds_patterns_r2.csv).

def quad_lane(l):
    return ((l >> 3) << 1) | ((l >> 1) & 1), (((l >> 2) & 1) << 1) | (l & 1)


def wavefronts_128(addr_of_lane):
    """LDS.128 / STS.128 cost under the measured merge rule, bank conflicts included."""
    reqs = []  # (quad, unit) requests in lane order, merged inside a quad
    for l in range(32):
        r = (l >> 2, addr_of_lane(l))
        if r not in reqs:
            reqs.append(r)
    total = 0
    for w in range(0, len(reqs), 8):
        units = {u for _, u in reqs[w:w + 8]}
        per_group = {}
        for u in units:
            per_group[u % 8] = per_group.get(u % 8, 0) + 1
        total += max(per_group.values())
    return max(2, total)


def test_quad_mapping_matches_kernel_source():
    src = open(f"{ROOT}/paper_1710_10989_b200/csrc/expm_n8.cuh").read()
    assert "r = quads ? ((lane >> 3) << 1) | ((lane >> 1) & 1) : lane >> 2;" in src
    assert "q = quads ? (((lane >> 2) & 1) << 1) | (lane & 1) : lane & 3;" in src


def test_quad_mapping_is_a_bijection_of_2x2_quads():
    assert sorted(quad_lane(l) for l in range(32)) == [(r, q) for r in range(8) for q in range(4)]
    for g in range(8):
        rs = {quad_lane(l)[0] for l in range(4 * g, 4 * g + 4)}
        qs = {quad_lane(l)[1] for l in range(4 * g, 4 * g + 4)}
        assert len(rs) == 2 and len(qs) == 2


def test_reference_product_wavefronts():
    """28 wavefronts per product with the quad mapping, 44 with lane = 4r + q."""
    def product(rq):
        store = wavefronts_128(lambda l: slot(*rq(l)))
        xrow = sum(wavefronts_128(lambda l, c=c: slot(rq(l)[0], c)) for c in range(4))
        ycol = sum(wavefronts_128(lambda l, k=k: slot(k, rq(l)[1])) for k in range(8))
        return store, xrow, ycol
    assert product(quad_lane) == (4, 8, 16)
    assert product(lambda l: (l >> 2, l & 3)) == (4, 8, 32)


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
