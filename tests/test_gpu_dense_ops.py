"""The reference's lower-level layer on the device (csrc/dense_ops.cu):
dense_matrix.hpp:40-58 value operations, kernels.hpp:15-24 and the scheme
evaluators of taylor_schemes.hpp / pade.hpp, through the same operation codes
on both sides -- the product's mexp_b200_dense_call (what the C++ drop-in
calls) and the compiled reference's ref_dense_call (oracle/ref_shim.cpp) --
on the same inputs: results bit-identical, CostContext ledgers equal. The
batched device entries of the public C ABI (mexp_matmul_batched, ...) are
checked against the reference the same way.
"""
import ctypes as C

import numpy as np
import pytest

import paper_1710_10989_b200 as mx

pytestmark = pytest.mark.gpu

P = C.c_void_p


def _sig(f):
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_int, P, C.c_int, P, C.c_int, P, P, P, P, P]
    return f


@pytest.fixture(scope="module")
def both(reference):
    from oracle.oracle import REF_SO
    return _sig(mx.library().mexp_b200_dense_call), _sig(C.CDLL(REF_SO).ref_dense_call)


def call(fn, op, arg, mats, n, coeffs=None, iin=None, out_len=None, want_iout=False):
    mats = [np.ascontiguousarray(m, np.float64) for m in mats]
    arr = (C.c_void_p * max(len(mats), 1))(*[m.ctypes.data for m in mats])
    out = np.zeros(out_len if out_len is not None else n * n)
    iout = np.zeros(n, np.int32) if want_iout else None
    cf = None if coeffs is None else np.ascontiguousarray(coeffs, np.float64)
    pr, so = C.c_int64(-1), C.c_int64(-1)
    st = fn(op, arg, arr, len(mats), None if cf is None else cf.ctypes.data, n, out.ctypes.data,
            None if iin is None else iin.ctypes.data, None if iout is None else iout.ctypes.data,
            C.byref(pr), C.byref(so))
    return st, out, iout, pr.value, so.value


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


def rand(n, norm, seed):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, (n, n))
    return a * (norm / np.abs(a).sum(axis=0).max())


@pytest.mark.parametrize("n", [1, 3, 8, 13, 64, 65, 130])
def test_matmul_lincomb_norm_lu_bitwise(cuda, both, n):
    ours, ref = both
    a, b = rand(n, 3.0, n), rand(n, 0.7, n + 1)
    for fn_args in [(0, 0, [a, b]), (2, 0, [a]), (3, 0, [a + n * np.eye(n), b])]:
        op, arg, mats = fn_args
        ol = 1 if op == 2 else None
        r1 = call(ours, op, arg, mats, n, out_len=ol)
        r2 = call(ref, op, arg, mats, n, out_len=ol)
        assert r1[0] == r2[0] == 0, (op, r1[0], r2[0])
        assert same(r1[1], r2[1]), (op, n)
    # lincomb, k = 1..11 (chunks of 8 continue the running sum)
    rng = np.random.default_rng(n)
    mats = [rand(n, 1.0 + k, 50 + k) for k in range(11)]
    for k in (1, 2, 5, 8, 9, 11):
        c = rng.standard_normal(k)
        r1 = call(ours, 1, 0, mats[:k], n, coeffs=c)
        r2 = call(ref, 1, 0, mats[:k], n, coeffs=c)
        assert r1[0] == r2[0] == 0 and same(r1[1], r2[1]), (n, k)


def test_lu_factor_apply_and_singular(cuda, both):
    ours, ref = both
    n = 37
    a = rand(n, 5.0, 3)
    a[[2, 30]] = a[[30, 2]]
    r1 = call(ours, 15, 0, [a], n, want_iout=True)
    r2 = call(ref, 15, 0, [a], n, want_iout=True)
    assert r1[0] == r2[0] == 0 and same(r1[1], r2[1]) and np.array_equal(r1[2], r2[2])
    rhs = rand(n, 1.0, 4)
    lu = r2[1].reshape(n, n)
    s1 = call(ours, 16, 0, [lu, rhs], n, iin=r2[2])
    s2 = call(ref, 16, 0, [lu, rhs], n, iin=r2[2])
    assert s1[0] == s2[0] == 0 and same(s1[1], s2[1])
    sing = a.copy()
    sing[:, 5] = 0.0
    assert call(ours, 3, 0, [sing, rhs], n)[0] == call(ref, 3, 0, [sing, rhs], n)[0] == mx.ERR_SINGULAR
    # ties and NaN in the pivot column follow the reference's strict '>' scan
    t = np.eye(6) * 2.0
    t[3, 0] = t[4, 0] = -2.0
    t[5, 1] = np.nan
    r1 = call(ours, 15, 0, [t], 6, want_iout=True)
    r2 = call(ref, 15, 0, [t], 6, want_iout=True)
    assert r1[0] == r2[0] and np.array_equal(r1[2], r2[2]) and same(r1[1], r2[1])


@pytest.mark.parametrize("op,arg", [(5, 0), (6, 0), (7, 0), (9, 0), (8, 2), (8, 4), (8, 6), (8, 9),
                                    (8, 16), (10, 0), (10, 7), (11, 1), (11, 9), (13, 1), (13, 8),
                                    (13, 18), (14, 16), (4, 3), (12, 2), (12, 6), (12, 10),
                                    (12, 20), (12, 26)])
@pytest.mark.parametrize("n", [5, 32, 70])
def test_schemes_bitwise_and_ledger(cuda, both, op, arg, n):
    ours, ref = both
    a = rand(n, 0.8, 100 * op + arg + n)
    r1 = call(ours, op, arg, [a], n)
    r2 = call(ref, op, arg, [a], n)
    assert r1[0] == r2[0] == 0, (r1[0], r2[0])
    assert same(r1[1], r2[1])
    assert (r1[3], r1[4]) == (r2[3], r2[4])  # products, solves


def test_invalid_arguments_match(cuda, both):
    ours, ref = both
    a = np.eye(4)
    for op, arg in ((8, 5), (13, 7), (14, 8), (12, 7), (12, 28)):
        assert call(ours, op, arg, [a], 4)[0] in (mx.ERR_INVALID_ARGUMENT, mx.ERR_UNSUPPORTED)
        assert call(ref, op, arg, [a], 4)[0] == mx.ERR_INVALID_ARGUMENT


def test_batched_device_entries(cuda, reference):
    import torch
    rng = np.random.default_rng(5)
    for n in (8, 24, 96):
        a = rng.uniform(-1, 1, (5, n, n))
        b = rng.uniform(-1, 1, (5, n, n))
        da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        c = mx.matmul_batched(da, db).cpu().numpy()
        for i in range(5):
            assert same(c[i], reference.matmul(a[i], b[i]))
        cf = mx.matmul_batched(da, db, rounding=mx.ROUND_FAST).cpu().numpy()
        assert np.abs(cf - c).max() <= 1e-13 * n
        norms = mx.one_norm_batched(da).cpu().numpy()
        assert same(norms, [reference.one_norm(a[i]) for i in range(5)])
        lc = mx.lincomb_batched([0.5, -2.0, 3.0], [da, db, da]).cpu().numpy()
        assert same(lc, (0.5 * a + -2.0 * b) + 3.0 * a)
        m = da + n * torch.eye(n, dtype=torch.float64, device="cuda")
        x, st = mx.lu_solve_batched(m, db)
        assert (st.cpu().numpy() == 0).all()
        assert np.abs(torch.bmm(m, x).cpu().numpy() - b).max() <= 1e-12
    # non-finite column sums never win the norm (strict '>')
    z = np.zeros((1, 4, 4))
    z[0, 1, 2] = np.nan
    z[0, 0, 3] = 2.5
    assert mx.one_norm_batched(torch.from_numpy(z).cuda()).item() == reference.one_norm(z[0]) == 2.5
