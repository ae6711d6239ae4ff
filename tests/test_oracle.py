"""CPU tests: pin the oracle (plain-C restatement) before trusting it.

* the reference's own known-answer tests (proj/tests/test_expm.cpp,
  test_dense_matrix.cpp, test_taylor_schemes.cpp, cli_smoke.sh), re-expressed;
* bit-for-bit agreement with the committed golden fixtures, which were made
  by the compiled reference (tests/golden/make_golden.py);
* bit-for-bit agreement with the compiled reference itself when oracle/_ref
  is present.
"""
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

U53 = 2.0 ** -53


def l1(x):
    return np.abs(x).sum(axis=0).max()


# ---- selection KATs: test_expm.cpp:21-47, 175-208 -------------------------
def test_select_walks_the_table(oracle):
    assert oracle.select(0.0, 1)[1:] == (1, 0)
    assert oracle.select(1.0, 1)[1:] == (18, 0)
    assert oracle.select(10.0, 1)[1:] == (18, 4)
    assert oracle.select(2.18, 1)[1:] == (18, 1)   # 2.18/2 sits exactly on theta_18
    assert oracle.select(float("nan"), 1)[0] == 2
    assert oracle.select(float("inf"), 1)[0] == 2
    assert oracle.select(-1.0, 1)[0] == 2


def test_scaling_grows_by_one_when_norm_doubles(oracle):
    for norm in (1.2, 3.7, 9.0, 40.0, 333.0):
        _, da, sa = oracle.select(norm, 1)
        _, db, sb = oracle.select(2.0 * norm, 1)
        assert da == db == 18 and sb == sa + 1


def test_no_scaling_inside_the_table(oracle):
    for acc, tmax in ((0, 3.01), (1, 1.09)):
        for i in range(41):
            assert oracle.select(tmax * i / 40.0, acc)[2] == 0


def test_single_target_picks_cheaper_scheme(oracle):
    assert oracle.select(0.4, 0)[1] == 8
    assert oracle.select(0.4, 1)[1] == 18


# ---- dense-matrix KATs: test_dense_matrix.cpp:17-55 -----------------------
def test_one_norm_kats(oracle):
    assert oracle.one_norm(np.zeros((3, 3))) == 0.0
    assert oracle.one_norm(np.eye(5)) == 1.0
    assert oracle.one_norm(np.array([[1.0, -2.0], [3.0, 4.0]])) == 6.0


def test_matmul_kats(oracle):
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[5.0, 6.0], [7.0, 8.0]])
    assert np.array_equal(oracle.matmul(a, b), [[19.0, 22.0], [43.0, 50.0]])
    nil = np.array([[0.0, 1.0], [0.0, 0.0]])
    assert np.array_equal(oracle.matmul(nil, nil), np.zeros((2, 2)))


# ---- expm KATs: test_expm.cpp:71-133, cli_smoke.sh:10-19 ------------------
def test_zero_matrix_gives_identity(oracle):
    r = oracle.expm_batch(np.zeros((1, 4, 4)))
    assert np.array_equal(r.out[0], np.eye(4)) and (r.degree[0], r.s[0]) == (1, 0)


def test_rotation_by_pi(oracle):
    pi = 3.141592653589793
    r = oracle.expm_batch(np.array([[[0.0, pi], [-pi, 0.0]]]))
    assert (r.degree[0], r.s[0], r.cost_thirds[0]) == (18, 2, 21)
    assert r.norm_in[0] == pi
    assert l1(r.out[0] + np.eye(2)) <= 1e-12


def test_rotation_by_one_radian_cli_report(oracle):
    r = oracle.expm_batch(np.array([[[0.0, 1.0], [-1.0, 0.0]]]))
    assert (r.degree[0], r.s[0], r.cost_thirds[0] // 3, r.norm_in[0]) == (18, 0, 5, 1.0)


def test_non_finite_rejected(oracle):
    a = np.zeros((1, 2, 2))
    a[0, 0, 1] = np.inf
    assert oracle.expm_batch(a).status[0] == 1
    a[0, 0, 1] = np.nan
    assert oracle.expm_batch(a).status[0] == 1


def test_inverse_identity(oracle):
    rng = np.random.default_rng(42)
    for _ in range(34):
        n = int(rng.integers(2, 17))
        a = rng.uniform(-1, 1, (n, n))
        a *= (5.0 * rng.uniform() + 1e-6) / l1(a)
        x = oracle.expm_batch(a[None]).out[0]
        y = oracle.expm_batch(-a[None]).out[0]
        assert l1(oracle.matmul(x, y) - np.eye(n)) <= 1e-12


def test_skew_input_orthogonal(oracle):
    rng = np.random.default_rng(43)
    for rep in range(20):
        b = rng.uniform(-1, 1, (10, 10))
        a = b - b.T
        a *= 3.0 * (rep % 5 + 1) / 5.0 / l1(a)
        x = oracle.expm_batch(a[None]).out[0]
        assert l1(oracle.matmul(x.T.copy(), x) - np.eye(10)) <= 1e-12


# ---- scheme KATs: test_taylor_schemes.cpp ---------------------------------
def horner(a, degree):
    """Plain Horner Taylor polynomial (taylor_schemes.cpp:87-94), numpy."""
    n = a.shape[0]
    t = np.eye(n)
    for k in range(degree, 0, -1):
        t = np.eye(n) + (a @ t) / k
    return t


@pytest.mark.parametrize("degree,theta,tol", [(8, 4.99e-2, 50 * U53), (12, 2.99e-1, 1e-13),
                                              (18, 1.09, 1e-13), (4, 3.40e-4, 1e-13),
                                              (2, 2.58e-8, 1e-13)])
def test_schemes_match_horner(oracle, degree, theta, tol):
    rng = np.random.default_rng(21 + degree)
    worst = 0.0
    for rep in range(60):
        n = (2, 4, 8, 16, 32)[rep % 5]
        a = rng.uniform(-1, 1, (n, n))
        a *= theta * (0.1, 0.5, 1.0)[(rep // 5) % 3] / l1(a)
        k, got = oracle.eval_taylor_new(a, degree)
        assert k == {2: 1, 4: 2, 8: 3, 12: 4, 18: 5}[degree]   # product ledger
        want = horner(a, degree)
        worst = max(worst, l1(got - want) / l1(want))
    assert worst <= tol


def test_unsupported_degree(oracle):
    assert oracle.eval_taylor_new(np.eye(2), 7)[0] == -1


# frozen 50-digit closed forms, rounded to double (tests/support/frozen_coefficients.hpp)
FROZEN_T8 = [0.1083646567852278, 0.02709116419630695, 0.6666666666666666, 0.5467614579707241,
             0.16112557339541758, 0.014090917158378208, 0.033792797010870505, 1.0, 1.0,
             0.13549236135285064]


def ulps(a, b):
    a, b = np.float64(a), np.float64(b)
    return abs(int(a.view(np.int64)) - int(b.view(np.int64)))


def test_coefficients_within_one_ulp_of_frozen(oracle):
    t8, t12, _, _ = oracle.coefficients()
    for got, want in zip(t8, FROZEN_T8):
        assert ulps(got, want) <= 1
    assert t12[0, 0] == 9.0198e-16 and t12[0, 3] == -2.0861320e-13


def test_oracle_coefficients_equal_reference(oracle, golden):
    g = golden("coefficients.npz")
    t8, t12, a, b = oracle.coefficients()
    for x, y in ((t8, g["t8"]), (t12, g["t12"]), (a, g["t18a"]), (b, g["t18b"])):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))


def macro_body(src, name):
    """The text of a (backslash-continued) #define, without its name."""
    lines = src[src.index("#define " + name + " "):].splitlines()
    out = []
    for ln in lines:
        out.append(ln.rstrip("\\"))
        if not ln.endswith("\\"):
            break
    return " ".join(out)[len("#define " + name):]


def test_device_coefficients_equal_reference(golden):
    """The coefficient tables the kernels and the drop-in share (scheme_tables.h,
    expm_common.cuh) are the reference's doubles bit for bit."""
    csrc = os.path.join(ROOT, "paper_1710_10989_b200", "csrc")
    src = open(os.path.join(csrc, "expm_common.cuh")).read() + \
        open(os.path.join(csrc, "scheme_tables.h")).read()
    g = golden("coefficients.npz")
    t8 = dict(re.findall(r"double (x\d|y\d) = ([^;]+);", src))
    names = ["x1", "x2", "x3", "x4", "x5", "x6", "x7", "y0", "y1", "y2"]
    for name, want in zip(names, g["t8"]):
        got = float.fromhex(t8[name]) if "0x" in t8[name] else float(t8[name])
        assert got == want, name

    def block(name):
        m = re.search(r"constexpr double " + name + r"\[[^=]*=\s*\{(.*?)\};", src, re.S)
        return np.array([float(v) for v in re.findall(r"[-+]?\d[\d.e+-]*", m.group(1))])

    def macro(name):
        return np.array([float(v) for v in re.findall(r"[-+]?\d[\d.e+-]*", macro_body(src, name))])

    assert "c_t12[4][4] = MEXP_T12_TABLE" in src and "c_t18b[4][5] = MEXP_T18B_TABLE" in src
    assert np.array_equal(macro("MEXP_T12_TABLE"), g["t12"].ravel())
    assert np.array_equal(macro("MEXP_T18A_TABLE"), g["t18a"])
    assert np.array_equal(macro("MEXP_T18B_TABLE"), g["t18b"].ravel())
    th = block("c_theta")
    assert np.array_equal(th, [1.19e-7, 5.98e-4, 5.12e-2, 5.80e-1, 1.46, 3.01,
                               2.22e-16, 2.58e-8, 3.40e-4, 4.99e-2, 2.99e-1, 1.09])


# ---- golden fixtures made by the compiled reference -----------------------
def test_select_matches_golden(oracle, golden):
    g = golden("select.npz")
    for acc in (0, 1):
        for v, d, s, st in zip(g["norms"], g[f"degree_acc{acc}"], g[f"s_acc{acc}"],
                               g[f"status_acc{acc}"]):
            got = oracle.select(float(v), acc)
            assert got[0] == st
            if st == 0:
                assert got[1:] == (d, s), (v, acc)


def golden_cases(golden):
    g = golden("expm_cases.npz")
    for entry in g["names"]:
        key, name = str(entry).split(":", 1)
        acc = int(key.split("_acc")[1])
        yield (name, acc, g[key + "_a"], g[key + "_out"], g[key + "_meta"],
               g[key + "_norm"][0])


def test_expm_matches_golden_bitwise(oracle, golden):
    count = 0
    for name, acc, a, out, meta, norm in golden_cases(golden):
        r = oracle.expm_batch(a[None], accuracy=acc)
        assert r.status[0] == meta[3], name
        assert (r.degree[0], r.s[0], r.cost_thirds[0]) == tuple(meta[:3]), name
        assert r.norm_in[0] == norm, name
        assert np.array_equal(r.out[0].view(np.uint64), out.view(np.uint64)), name
        count += 1
    assert count > 300
    degrees = {int(m[0]) for _, _, _, _, m, _ in golden_cases(golden)}
    assert degrees == {1, 2, 4, 8, 12, 18}


def test_cfg_slices_match_golden(oracle, golden):
    g = golden("cfg_slices.npz")
    r = oracle.expm_batch(g["cfg2_a"], accuracy=1)
    assert np.array_equal(r.out.view(np.uint64), g["cfg2_out"].view(np.uint64))
    assert np.array_equal(r.degree, g["cfg2_degree"]) and np.array_equal(r.s, g["cfg2_s"])
    r = oracle.expm_batch(g["cfg3_a"], accuracy=0)
    assert np.array_equal(r.out.view(np.uint64), g["cfg3_out"].view(np.uint64))
    assert np.array_equal(r.degree, g["cfg3_degree"]) and np.array_equal(r.s, g["cfg3_s"])


def test_generators_reproduce_golden_inputs(golden):
    from paper_1710_10989_b200 import workloads
    g = golden("cfg_slices.npz")
    assert np.array_equal(workloads.generate("cfg2", 0, 512), g["cfg2_a"])
    assert np.array_equal(workloads.generate("cfg3", 32768 - 32, 64), g["cfg3_a"])


# ---- restatement vs the compiled reference (build container / GPU box) ----
def test_oracle_bitwise_equals_reference(oracle, reference):
    from paper_1710_10989_b200 import workloads
    a = workloads.generate("cfg2", 1000, 4096)
    r1 = reference.expm_batch(a, accuracy=1)
    r2 = oracle.expm_batch(a, accuracy=1)
    assert np.array_equal(r1.out.view(np.uint64), r2.out.view(np.uint64))
    for f in ("degree", "s", "cost_thirds", "norm_in", "status"):
        assert np.array_equal(getattr(r1, f), getattr(r2, f)), f
    b = workloads.generate("cfg3", 0, 16)
    r1 = reference.expm_batch(b, accuracy=0)
    r2 = oracle.expm_batch(b, accuracy=0)
    assert np.array_equal(r1.out, r2.out) and np.array_equal(r1.s, r2.s)


def test_forced_selection_equals_expm(oracle):
    from paper_1710_10989_b200 import workloads
    a = workloads.generate("cfg2", 77, 64)
    r = oracle.expm_batch(a)
    for k in range(64):
        got = oracle.expm_forced(a[k], int(r.degree[k]), int(r.s[k]))
        assert np.array_equal(got.view(np.uint64), r.out[k].view(np.uint64))


def test_leading_block_of_triangular_matrix(oracle):
    """The size-independent check used for cfg5: for upper-triangular A the
    leading k x k block of e^A is T_m(2^-s A_k)^(2^s) with the FULL matrix's
    (m, s); in the reference's arithmetic the extra terms are exact zeros, so
    the two agree bit for bit."""
    rng = np.random.default_rng(8)
    n, k = 48, 12
    a = np.triu(rng.standard_normal((n, n)) / np.sqrt(n), 1) + np.diag(-5 * rng.uniform(size=n))
    a *= 30.0 / l1(a)
    r = oracle.expm_batch(a[None])
    blk = oracle.expm_forced(a[:k, :k].copy(), int(r.degree[0]), int(r.s[0]))
    assert np.array_equal(blk.view(np.uint64), r.out[0][:k, :k].copy().view(np.uint64))
    assert np.all(np.tril(r.out[0], -1) == 0.0)


# ---- Family::TaylorPS (Paterson-Stockmeyer; §8(f) next row) ---------------
def test_ps_select_matches_golden(oracle, golden):
    g = golden("taylor_ps.npz")
    for acc in (0, 1):
        for v, d, s, st in zip(g["norms"], g[f"degree_acc{acc}"], g[f"s_acc{acc}"],
                               g[f"status_acc{acc}"]):
            got = oracle.select(float(v), acc, 1)
            assert got[0] == st
            if st == 0:
                assert got[1:] == (d, s), (v, acc)


def test_ps_expm_matches_golden_bitwise(oracle, golden):
    g = golden("taylor_ps.npz")
    degrees = set()
    for n in (1, 2, 3, 8, 13, 16, 32, 64):
        a = g[f"n{n}_a"]
        for acc in (0, 1):
            r = oracle.expm_batch(a, accuracy=acc, family=1)
            meta = g[f"n{n}_acc{acc}_meta"]
            assert np.array_equal(r.degree, meta[:, 0]) and np.array_equal(r.s, meta[:, 1])
            assert np.array_equal(r.cost_thirds, meta[:, 2])
            assert np.array_equal(r.norm_in, g[f"n{n}_acc{acc}_norm"])
            assert np.array_equal(r.out.view(np.uint64), g[f"n{n}_acc{acc}_out"].view(np.uint64)), (n, acc)
            degrees |= set(int(d) for d in r.degree)
    assert degrees == {1, 2, 4, 6, 9, 16}


def test_ps_eval_matches_horner(oracle):
    """eval_taylor_ps(m) is the degree-m Taylor polynomial (within rounding)."""
    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, (6, 6))
    a *= 0.3 / l1(a)
    for m in (1, 2, 4, 6, 9, 16):
        k, got = oracle.eval_taylor_ps(a, m)
        want = np.eye(6)
        term = np.eye(6)
        for j in range(1, m + 1):
            term = term @ a / j
            want = want + term
        assert k == {1: 0, 2: 1, 4: 2, 6: 3, 9: 4, 16: 6}[m]
        assert np.abs(got - want).max() < 1e-15, m
    assert oracle.eval_taylor_ps(a, 8)[0] == -1


def test_ps_oracle_bitwise_equals_reference(oracle, reference):
    rng = np.random.default_rng(11)
    for n in (4, 8, 20):
        norms = 10.0 ** rng.uniform(-17, 2.5, 64)
        a = rng.standard_normal((64, n, n))
        a *= (norms / np.abs(a).sum(axis=1).max(axis=1))[:, None, None]
        for acc in (0, 1):
            r1 = reference.expm_batch(a, accuracy=acc, family=1)
            r2 = oracle.expm_batch(a, accuracy=acc, family=1)
            assert np.array_equal(r1.out.view(np.uint64), r2.out.view(np.uint64)), (n, acc)
            for f in ("degree", "s", "cost_thirds", "norm_in", "status"):
                assert np.array_equal(getattr(r1, f), getattr(r2, f)), f


# ---- Family::PadeDiagonal (§8(f) next row) ---------------------------------
def test_pade_select_matches_golden(oracle, golden):
    g = golden("pade.npz")
    for acc in (0, 1):
        for v, d, s, st in zip(g["norms"], g[f"degree_acc{acc}"], g[f"s_acc{acc}"],
                               g[f"status_acc{acc}"]):
            got = oracle.select(float(v), acc, 2)
            assert got[0] == st
            if st == 0:
                assert got[1:] == (d, s), (v, acc)


def test_pade_coefficients(oracle, golden):
    """pade_coeffs(1..13): the oracle's int128 / long double restatement and
    the device table (expm_common.cuh c_pade) equal the reference's doubles."""
    g = golden("pade.npz")["coeffs"]
    for m in range(1, 14):
        assert np.array_equal(oracle.pade_coeffs(m).view(np.uint64), g[m - 1, :m + 1].view(np.uint64))
    src = open(os.path.join(ROOT, "paper_1710_10989_b200", "csrc", "scheme_tables.h")).read()
    body = macro_body(src, "MEXP_PADE_TABLE")
    vals = [float.fromhex(t) if "0x" in t else float(t)
            for t in re.findall(r"0x[0-9a-fA-Fp.+-]+|\d+\.\d+", body)]
    dev = np.array(vals).reshape(13, 14)
    assert np.array_equal(dev.view(np.uint64), g.view(np.uint64))


def test_pade_expm_matches_golden_bitwise(oracle, golden):
    g = golden("pade.npz")
    degrees = set()
    for n in (1, 2, 3, 8, 13, 16, 32, 64):
        a = g[f"n{n}_a"]
        for acc in (0, 1):
            r = oracle.expm_batch(a, accuracy=acc, family=2)
            meta = g[f"n{n}_acc{acc}_meta"]
            assert np.array_equal(r.status, meta[:, 3])
            assert np.array_equal(r.degree, meta[:, 0]) and np.array_equal(r.s, meta[:, 1])
            assert np.array_equal(r.cost_thirds, meta[:, 2])
            assert np.array_equal(r.norm_in, g[f"n{n}_acc{acc}_norm"])
            assert np.array_equal(r.out.view(np.uint64), g[f"n{n}_acc{acc}_out"].view(np.uint64)), (n, acc)
            degrees |= set(int(d) for d in r.degree)
    assert degrees == set(range(2, 27, 2))


def test_pade_approximant_kats(oracle):
    """r_m(A) approximates exp(A) (pade.hpp); order 2 is (I - A/2)^-1 (I + A/2);
    invalid orders refuse (pade.cpp:79-80)."""
    rng = np.random.default_rng(4)
    a = rng.uniform(-1, 1, (5, 5))
    a *= 0.2 / l1(a)
    want = np.eye(5)
    term = np.eye(5)
    for j in range(1, 30):
        term = term @ a / j
        want = want + term
    for order in range(2, 27, 2):
        k, got = oracle.eval_pade(a, order)
        assert k >= 0
        if order >= 12:
            assert np.abs(got - want).max() < 1e-15, order
    k, r2 = oracle.eval_pade(a, 2)
    assert k == 0
    assert np.allclose(r2, np.linalg.solve(np.eye(5) - a / 2, np.eye(5) + a / 2), atol=1e-15)
    for bad in (0, 3, 28):
        assert oracle.eval_pade(a, bad)[0] == -1


def test_pade_oracle_bitwise_equals_reference(oracle, reference):
    rng = np.random.default_rng(12)
    for n in (3, 8, 20):
        for order in range(2, 27, 2):
            a = rng.standard_normal((n, n))
            a *= 0.5 / l1(a)
            k1, x1 = oracle.eval_pade(a, order)
            k2, x2 = reference.eval_pade(a, order)
            assert k1 == k2 and np.array_equal(x1.view(np.uint64), x2.view(np.uint64)), (n, order)
        norms = 10.0 ** rng.uniform(-9, 2.5, 64)
        a = rng.standard_normal((64, n, n))
        a *= (norms / np.abs(a).sum(axis=1).max(axis=1))[:, None, None]
        for acc in (0, 1):
            r1 = reference.expm_batch(a, accuracy=acc, family=2)
            r2 = oracle.expm_batch(a, accuracy=acc, family=2)
            assert np.array_equal(r1.out.view(np.uint64), r2.out.view(np.uint64)), (n, acc)
            for f in ("degree", "s", "cost_thirds", "norm_in", "status"):
                assert np.array_equal(getattr(r1, f), getattr(r2, f)), f
