"""GPU parity of Family::TaylorPS (Paterson-Stockmeyer Taylor, the paper's
baseline family) through the C ABI: (m, s) and norm_in bit
for bit, REFERENCE rounding bit-identical to the reference for n <= 64,
every other rounding within relative Frobenius 50*n*u."""
import numpy as np
import pytest

import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads

pytestmark = pytest.mark.gpu

U53 = 2.0 ** -53
U24 = 2.0 ** -24
PS = mx.Family.TaylorPS
MODES = {"reference": mx.ROUND_REFERENCE, "auto": mx.ROUND_AUTO, "fast": mx.ROUND_FAST}


def rel_fro(got, want):
    g = got.reshape(got.shape[0], -1).astype(np.float64)
    w = want.reshape(want.shape[0], -1).astype(np.float64)
    return np.linalg.norm(g - w, axis=1) / np.linalg.norm(w, axis=1)


def exact_s_min(n):
    return 0 if n < 8 else 3 + int(np.floor(np.log2(n)))


@pytest.mark.parametrize("mode", ["reference", "auto", "fast"])
def test_ps_golden(cuda, golden, mode):
    g = golden("taylor_ps.npz")
    for n in (1, 2, 3, 8, 13, 16, 32, 64):
        a = g[f"n{n}_a"]
        for acc in (0, 1):
            out, sel, st = mx.expm_batched_host(a, accuracy=mx.Accuracy(acc),
                                                rounding=MODES[mode], family=PS)
            assert st == mx.OK
            meta = g[f"n{n}_acc{acc}_meta"]
            want = g[f"n{n}_acc{acc}_out"]
            assert np.array_equal(sel["degree"], meta[:, 0]), (n, acc)
            assert np.array_equal(sel["s"], meta[:, 1]), (n, acc)
            assert np.array_equal(sel["norm_in"], g[f"n{n}_acc{acc}_norm"]), (n, acc)
            if mode == "reference":
                assert np.array_equal(out.view(np.uint64), want.view(np.uint64)), (n, acc)
                continue
            err = rel_fro(out, want)
            tol = 50 * n * U53
            if mode == "fast":  # the band is promised where AUTO keeps FMA rounding
                keep = sel["s"] < exact_s_min(n)
                err = err[keep]
            assert err.size == 0 or err.max() <= tol, (n, acc, err.max(), tol)


def test_ps_cfg2_slice(cuda, oracle):
    a = workloads.generate("cfg2", 0, 4096)
    ref = oracle.expm_batch(a, accuracy=1, family=int(PS))
    out, sel, st = mx.expm_batched_host(a, family=PS)
    assert st == mx.OK
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    err = rel_fro(out, ref.out)
    assert err.max() <= 50 * 8 * U53, err.max()
    out_r, _, _ = mx.expm_batched_host(a, family=PS, rounding=mx.ROUND_REFERENCE)
    assert np.array_equal(out_r.view(np.uint64), ref.out.view(np.uint64))


@pytest.mark.parametrize("n", [3, 8, 16, 32, 64])
def test_ps_fp32(cuda, oracle, n):
    rng = np.random.default_rng(300 + n)
    norms = np.array([1e-8, 1e-3, 0.04, 0.2, 0.7, 2.0, 12.0, 40.0])
    a = rng.standard_normal((len(norms), n, n))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    a = a.astype(np.float32)
    ref = oracle.expm_batch(a, accuracy=0, family=int(PS))
    out, sel, st = mx.expm_batched_host(a, accuracy=mx.Accuracy.Single, family=PS)
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    assert rel_fro(out, ref.out).max() <= 50 * n * U24


@pytest.mark.parametrize("n", [96, 128, 200])
def test_ps_large_n_every_degree(cuda, oracle, n):
    rng = np.random.default_rng(2000 + n)
    # norms hitting degrees 1, 2, 4, 6, 9, 16 and s = 0..7
    norms = np.array([1e-17, 1e-9, 1e-4, 5e-3, 0.05, 0.5, 1.2, 7.0, 30.0, 100.0])
    a = rng.uniform(-1, 1, (len(norms), n, n))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    ref = oracle.expm_batch(a, family=int(PS))
    assert set(ref.degree) == {1, 2, 4, 6, 9, 16}
    out, sel, st = mx.expm_batched_host(a, family=PS)
    assert st == mx.OK
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    assert np.array_equal(sel["norm_in"], ref.norm_in)
    err = rel_fro(out, ref.out)
    assert err.max() <= 50 * n * U53, err


def test_ps_drop_in_report(cuda):
    pi = 3.141592653589793
    r = mx.expm(np.array([[0.0, pi], [-pi, 0.0]]), family=PS)
    assert (r.degree, r.s, r.cost_thirds) == (16, 3, 27)
    assert np.abs(r.result + np.eye(2)).max() < 1e-12
