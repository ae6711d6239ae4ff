"""AUTO-rounding parity beyond the BASELINE configs.

The default policy (AUTO) is what the C++ drop-in ``mexp::expm`` runs for
arbitrary caller matrices, so it is checked here on every kind of the
reference's own test-matrix gallery (``proj/src/gallery.cpp:37-99``: dense,
symmetric, skew, Jordan, nilpotent, upper triangular, Toeplitz, rank one and
the non-normal shear), sizes from 2 to 512 and 1-norms from 1e-4 to 1e4 (s up
to 14), against the compiled reference (``oracle/_ref``):

* (m, s) and ``norm_in`` bit-equal per matrix (``expm.cpp:37-74``);
* e^A within relative Frobenius 50*n*u of the reference's e^A, wherever the
  reference's own result is representable (at ||A||_1 = 1e4 most kinds
  overflow: then ours must overflow too; a result that underflows to exact
  zeros must come out as (near-)zeros too).

With s >= 3 + floor(log2 n) (every s for n < 8) AUTO runs the reference's own
rounding, so those matrices are bit-identical; the rest run on DMMA/FMA.

FAST (DMMA/FMA rounding, no parity promise past the AUTO threshold) is
measured beside it and reported, not asserted. Run with ``-s`` to see the
max err / tol table per kind and n.
"""
import ctypes as C

import numpy as np
import pytest

import paper_1710_10989_b200 as mx

pytestmark = pytest.mark.gpu

KINDS = ["random_dense", "random_symmetric", "random_skew", "jordan_block", "nilpotent_shift",
         "upper_triangular", "tridiag_toeplitz", "rank_one", "nonnormal_shear"]
U53 = 2.0 ** -53
U24 = 2.0 ** -24


def _ref_gallery():
    from oracle.oracle import REF_SO, Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    lib = C.CDLL(REF_SO)
    lib.ref_gallery.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_void_p]
    lib.ref_gallery.restype = C.c_int
    return lib


def gallery_batch(n, norms, seeds):
    """Every gallery kind x norm x seed at size n, from the reference's own
    generator (gallery.cpp:102-112). Returns (matrices, kind index per matrix)."""
    lib = _ref_gallery()
    mats, kinds = [], []
    for k in range(len(KINDS)):
        for seed in seeds:
            for norm in norms:
                m = np.zeros((n, n))
                if lib.ref_gallery(k, n, seed, float(norm), m.ctypes.data) == 0:
                    mats.append(m)
                    kinds.append(k)
    return np.stack(mats), np.array(kinds)


def run_stress(reference, n, norms, seeds, accuracy=mx.Accuracy.Double, dtype=np.float64):
    a, kinds = gallery_batch(n, norms, seeds)
    a = a.astype(dtype)
    ref = reference.expm_batch(a, accuracy=int(accuracy))
    u = U53 if dtype == np.float64 else U24
    tol = 50 * n * u
    big = np.finfo(dtype).max
    tiny = 1e-290 if dtype == np.float64 else 1e-30
    wabs = np.abs(ref.out.reshape(len(a), -1))
    with np.errstate(invalid="ignore"):
        finite_ref = (wabs <= big).all(axis=1)   # representable in the storage type
    zero_ref = finite_ref & (wabs.max(axis=1) <= tiny)
    rows = {}
    for mode, rnd in (("auto", mx.ROUND_AUTO), ("fast", mx.ROUND_FAST)):
        out, sel, st = mx.expm_batched_host(a, accuracy=accuracy, rounding=rnd)
        assert st == mx.OK
        assert np.array_equal(sel["degree"], ref.degree), (n, mode)
        assert np.array_equal(sel["s"], ref.s), (n, mode)
        assert np.array_equal(sel["norm_in"].view(np.uint64), ref.norm_in.view(np.uint64))
        o = out.astype(np.float64).reshape(len(a), -1)
        w = ref.out.reshape(len(a), -1)
        with np.errstate(all="ignore"):
            # scaled by max |w| so results near the overflow threshold do not
            # overflow the Frobenius norms themselves
            sc = np.abs(w).max(axis=1, keepdims=True)
            sc[~(sc > 0) | ~np.isfinite(sc)] = 1.0
            err = np.linalg.norm((o - w) / sc, axis=1) / np.linalg.norm(w / sc, axis=1)
        err[~finite_ref] = 0.0
        # underflowed reference: ours must be (near-)zero as well
        err[zero_ref] = np.where(np.abs(o[zero_ref]).max(axis=1) <= tiny, 0.0, np.inf)
        finite_ours = np.isfinite(o).all(axis=1)
        rows[mode] = (err, finite_ours)
    return a, kinds, ref, tol, finite_ref, rows


def exact_s_min(n):
    """AUTO threshold (capi.cu exact_s_min)."""
    return 0 if n < 8 else 3 + int(np.floor(np.log2(n)))


def _report(n, kinds, ref, tol, finite_ref, rows, label=""):
    lines = []
    fast_part = ref.s < exact_s_min(n)
    for k, name in enumerate(KINDS):
        sel = kinds == k
        if not sel.any():
            continue
        ea = rows["auto"][0][sel]
        ef = rows["fast"][0][sel]
        eaf = rows["auto"][0][sel & fast_part]
        lines.append(f"n={n:4d}{label} {name:17s} s<= {int(ref.s[sel].max()):2d}  "
                     f"auto err/tol {ea.max() / tol:7.3f} (DMMA/FMA part "
                     f"{(eaf.max() if eaf.size else 0.0) / tol:6.3f})  fast err/tol {ef.max() / tol:9.3f}  "
                     f"(ref overflow: {int((~finite_ref[sel]).sum())})")
    print("\n".join(lines))


SMALL_NS = [2, 3, 5, 7, 8, 12, 16, 24, 32, 48, 64]
NORMS = 10.0 ** np.linspace(-4, 4, 17)


@pytest.mark.parametrize("n", SMALL_NS)
def test_auto_gallery_small_n(cuda, reference, n):
    a, kinds, ref, tol, finite_ref, rows = run_stress(reference, n, NORMS, seeds=(1, 2, 3))
    _report(n, kinds, ref, tol, finite_ref, rows)
    err, finite_ours = rows["auto"]
    assert (finite_ours | ~finite_ref).all()
    assert not (finite_ours & ~finite_ref).any(), "reference overflowed where AUTO did not"
    bad = np.flatnonzero(err > tol)
    assert bad.size == 0, [(KINDS[kinds[i]], int(ref.s[i]), err[i] / tol) for i in bad[:10]]


@pytest.mark.parametrize("n", [96, 200, 512])
def test_auto_gallery_large_n(cuda, reference, n):
    norms = np.array([1e-3, 0.5, 3.0, 30.0, 300.0, 3000.0]) if n < 512 else \
        np.array([0.5, 8.0, 100.0, 1000.0])
    a, kinds, ref, tol, finite_ref, rows = run_stress(reference, n, norms, seeds=(4,))
    _report(n, kinds, ref, tol, finite_ref, rows)
    err, finite_ours = rows["auto"]
    assert not (finite_ours & ~finite_ref).any()
    bad = np.flatnonzero(err > tol)
    assert bad.size == 0, [(KINDS[kinds[i]], int(ref.s[i]), err[i] / tol) for i in bad[:10]]


@pytest.mark.parametrize("n", [8, 16, 32])
def test_auto_gallery_fp32_single(cuda, reference, n):
    """fp32 storage, Single table: FFMA arithmetic against the reference run in
    double on the same float values; tolerance 50*n*2^-24."""
    norms = 10.0 ** np.linspace(-3, 2, 11)
    a, kinds, ref, tol, finite_ref, rows = run_stress(reference, n, norms, seeds=(5, 6),
                                                      accuracy=mx.Accuracy.Single,
                                                      dtype=np.float32)
    _report(n, kinds, ref, tol, finite_ref, rows, label=" f32")
    err, _ = rows["auto"]
    bad = np.flatnonzero(err > tol)
    assert bad.size == 0, [(KINDS[kinds[i]], int(ref.s[i]), err[i] / tol) for i in bad[:10]]


def test_drop_in_single_matrix_matches_batched_auto(cuda, reference):
    """mexp::expm (one host matrix, the drop-in) runs the same AUTO policy as
    the batched call: identical bits on a spread of gallery matrices."""
    for n in (3, 8, 20, 64, 96):
        a, kinds = gallery_batch(n, [1e-3, 1.0, 50.0, 2000.0], seeds=(9,))
        out, sel, st = mx.expm_batched_host(a)
        for i in range(len(a)):
            r = mx.expm(a[i])
            assert (r.degree, r.s) == (sel["degree"][i], sel["s"][i])
            assert np.array_equal(r.result.view(np.uint64), out[i].view(np.uint64)), (n, i)
