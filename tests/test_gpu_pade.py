"""GPU parity of Family::PadeDiagonal (diagonal Pade r_m, m = 2..26 even, with
the batched pivoted LU solve) through the C ABI, for
n <= 64: (m, s), norm_in and cost bit for bit; REFERENCE rounding
bit-identical to the reference (products, lincombs AND the LU solve in the
reference's operation order); the other modes within 50*n*u."""
import numpy as np
import pytest

import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads

pytestmark = pytest.mark.gpu

U53 = 2.0 ** -53
U24 = 2.0 ** -24
PADE = mx.Family.PadeDiagonal
MODES = {"reference": mx.ROUND_REFERENCE, "auto": mx.ROUND_AUTO, "fast": mx.ROUND_FAST}


def rel_fro(got, want):
    g = got.reshape(got.shape[0], -1).astype(np.float64)
    w = want.reshape(want.shape[0], -1).astype(np.float64)
    return np.linalg.norm(g - w, axis=1) / np.linalg.norm(w, axis=1)


def exact_s_min(n):
    return 0 if n < 8 else 3 + int(np.floor(np.log2(n)))


@pytest.mark.parametrize("mode", ["reference", "auto", "fast"])
def test_pade_golden(cuda, golden, mode):
    g = golden("pade.npz")
    for n in (1, 2, 3, 8, 13, 16, 32, 64):
        a = g[f"n{n}_a"]
        for acc in (0, 1):
            out, sel, st = mx.expm_batched_host(a, accuracy=mx.Accuracy(acc),
                                                rounding=MODES[mode], family=PADE)
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
            if mode == "fast":
                err = err[sel["s"] < exact_s_min(n)]
            assert err.size == 0 or err.max() <= 50 * n * U53, (n, acc, err.max())


def test_pade_cfg2_slice(cuda, oracle):
    a = workloads.generate("cfg2", 0, 2048)
    ref = oracle.expm_batch(a, accuracy=1, family=int(PADE))
    out, sel, st = mx.expm_batched_host(a, family=PADE, rounding=mx.ROUND_REFERENCE)
    assert st == mx.OK
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    assert np.array_equal(out.view(np.uint64), ref.out.view(np.uint64))
    out_a, _, _ = mx.expm_batched_host(a, family=PADE)
    assert rel_fro(out_a, ref.out).max() <= 50 * 8 * U53


@pytest.mark.parametrize("n", [3, 8, 16, 32, 64])
def test_pade_fp32(cuda, oracle, n):
    rng = np.random.default_rng(400 + n)
    norms = np.array([1e-6, 1e-3, 0.05, 0.3, 1.0, 2.0, 4.0, 9.0, 30.0, 100.0])
    a = rng.standard_normal((len(norms), n, n))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    a = a.astype(np.float32)
    ref = oracle.expm_batch(a, accuracy=0, family=int(PADE))
    out, sel, st = mx.expm_batched_host(a, accuracy=mx.Accuracy.Single, family=PADE)
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    assert rel_fro(out, ref.out).max() <= 50 * n * U24


def test_pade_drop_in_and_limits(cuda):
    pi = 3.141592653589793
    r = mx.expm(np.array([[0.0, pi], [-pi, 0.0]]), family=PADE)
    assert (r.degree, r.s, r.cost_thirds) == (22, 0, 22)
    assert np.abs(r.result + np.eye(2)).max() < 1e-12
    a = np.zeros((2, 65, 65))
    out, sel, st = mx.expm_batched_host(a, family=PADE)
    assert st == mx.OK and np.array_equal(out, np.broadcast_to(np.eye(65), out.shape))
    b = np.zeros((3, 8, 8))
    b[1, 2, 2] = np.nan
    out, sel, st = mx.expm_batched_host(b, family=PADE, raise_on_error=False)
    assert st == mx.ERR_NONFINITE and list(sel["status"]) == [0, 1, 0]
    assert np.array_equal(out[0], np.eye(8))


@pytest.mark.parametrize("n", [96, 128, 200])
def test_pade_large_n_every_order(cuda, oracle, n):
    """n > 64: U, V on the DMMA GEMM chain with fused lincombs, M = V - U and
    R = V + U from the last epilogue, the batched blocked LU (lu_batched.cu),
    then the squarings; within 50 n u of the reference."""
    rng = np.random.default_rng(3000 + n)
    theta = [3.65e-8, 5.32e-4, 1.50e-2, 8.54e-2, 2.54e-1, 5.41e-1, 9.50e-1, 1.47, 2.10, 2.81,
             3.60, 4.46, 5.37]
    norms = np.array([0.9 * t for t in theta] + [20.0, 300.0])
    a = rng.uniform(-1, 1, (len(norms), n, n))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    ref = oracle.expm_batch(a, family=int(PADE))
    assert set(ref.degree) == set(range(2, 27, 2))
    out, sel, st = mx.expm_batched_host(a, family=PADE)
    assert st == mx.OK
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    assert np.array_equal(sel["norm_in"], ref.norm_in)
    err = rel_fro(out, ref.out)
    assert err.max() <= 50 * n * U53, err


def test_pade_large_n_pivoting(cuda, oracle):
    """A matrix whose Pade denominator needs row exchanges at every step of
    the blocked LU (a permutation-like dominant part) still matches."""
    n = 150
    rng = np.random.default_rng(77)
    perm = rng.permutation(n)
    a = np.zeros((2, n, n))
    a[0][np.arange(n), perm] = 1.0
    a[0] += 0.01 * rng.standard_normal((n, n))
    a[0] *= 4.0 / workloads.one_norm_batched(a[:1])[0]
    a[1] = rng.standard_normal((n, n)) * 0.02
    ref = oracle.expm_batch(a, family=int(PADE))
    out, sel, st = mx.expm_batched_host(a, family=PADE)
    assert st == mx.OK and np.array_equal(sel["s"], ref.s)
    assert rel_fro(out, ref.out).max() <= 50 * n * U53


_LU_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads
out_path = sys.argv[2]
res = {}
for n in (130, 500, 600):
    rng = np.random.default_rng(n)
    perm = rng.permutation(n)
    a = rng.standard_normal((4, n, n)) * 0.05
    a[0][np.arange(n), perm] += 1.0          # row exchanges at every column
    a[1] = np.triu(a[1])                     # triangular: no exchanges
    a *= (np.array([4.0, 30.0, 0.7, 9.0]) / workloads.one_norm_batched(a))[:, None, None]
    out, sel, st = mx.expm_batched_host(a, family=mx.Family.PadeDiagonal, raise_on_error=False)
    res[f"out{n}"] = out
    res[f"st{n}"] = sel["status"]
np.savez(out_path, **res)
"""


def test_pade_lu_panel_kernel_bitwise(cuda, tmp_path):
    """The cluster panel factorisation (lu_panel_cluster_kernel, panels of <=
    512 rows) and the per-column kernels (MEXP_LU_PANEL=0) give the same bits:
    same pivots, multipliers and updates; n = 600 mixes both paths."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        path = str(tmp_path / f"lu{flag}.npz")
        env = dict(os.environ, MEXP_LU_PANEL=flag)
        r = subprocess.run([sys.executable, "-c", _LU_SCRIPT, root, path], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        outs.append(np.load(path))
    for k in outs[0].files:
        assert np.array_equal(outs[0][k].view(np.uint8), outs[1][k].view(np.uint8)), k
