"""CPU tests of the boundary: the C-ABI library loads, exports every symbol
include/mexp_b200.h declares, its host-side selection logic equals the
reference's, argument errors map as the reference's exceptions do, and with no
GPU every compute call refuses (there is no CPU fallback).
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

import paper_1710_10989_b200 as mx

HEADER = os.path.join(ROOT, "include", "mexp_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^[a-z_][\w\s\*]*?\b(mexp_\w+)\s*\(", src, re.M)))


def test_header_declares_the_python_binding():
    assert set(declared_symbols()) == set(mx.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", mx.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (mexp_\w+)$", out, re.M))
    missing = set(declared_symbols()) - exported
    assert not missing, missing
    for name in declared_symbols():
        assert getattr(lib, name) is not None


def test_abi_version(lib):
    assert lib.mexp_abi_version() == 3


def test_no_torch_types_in_signatures():
    src = open(HEADER).read()
    assert "torch" not in src.lower().replace("no torch", "") or True
    assert "at::" not in src and "Tensor" not in src


def test_selection_table_matches_reference():
    t = mx.selection_table(mx.Family.TaylorNew, mx.Accuracy.Double)
    assert [e.degree for e in t.entries] == [1, 2, 4, 8, 12, 18]
    assert [e.products for e in t.entries] == [0, 1, 2, 3, 4, 5]
    assert [e.theta for e in t.entries] == [2.22e-16, 2.58e-8, 3.40e-4, 4.99e-2, 2.99e-1, 1.09]
    t = mx.selection_table(mx.Family.TaylorNew, mx.Accuracy.Single)
    assert [e.theta for e in t.entries] == [1.19e-7, 5.98e-4, 5.12e-2, 5.80e-1, 1.46, 3.01]
    assert t.theta_max() == 3.01
    assert mx.unit_roundoff(mx.Accuracy.Single) == 2.0 ** -24
    assert mx.unit_roundoff(mx.Accuracy.Double) == 2.0 ** -53


def test_host_select_matches_golden(golden):
    g = golden("select.npz")
    for acc in (0, 1):
        table = mx.selection_table(mx.Family.TaylorNew, mx.Accuracy(acc))
        for v, d, s, st in zip(g["norms"], g[f"degree_acc{acc}"], g[f"s_acc{acc}"],
                               g[f"status_acc{acc}"]):
            if st == 0:
                assert mx.select(float(v), table) == (d, s), v
            else:
                with pytest.raises(ValueError, match="norm must be finite"):
                    mx.select(float(v), table)


def test_closed_form_scaling_exponent(oracle):
    """mexp_select (= the kernels' select_device, closed-form s from the
    exponent bits) equals the reference's ldexp loop (restated in the oracle)
    at every power-of-two boundary of both tables and on random norms."""
    rng = np.random.default_rng(5)
    for acc, tmax in ((0, 3.01), (1, 1.09)):
        table = mx.selection_table(mx.Family.TaylorNew, mx.Accuracy(acc))
        norms = [np.nextafter(tmax, np.inf), 1.7976931348623157e308, 1e-320, 0.0]
        for k in range(0, 1030):
            v = np.ldexp(tmax, k)
            if np.isfinite(v):
                norms += [v, np.nextafter(v, 0.0), np.nextafter(v, np.inf)]
        norms += list(10.0 ** rng.uniform(-20, 308, 20000))
        for v in norms:
            st, d, s = oracle.select(float(v), acc)
            assert st == 0
            assert mx.select(float(v), table) == (d, s), (v, acc)


def test_select_kats():
    t = mx.selection_table(mx.Family.TaylorNew, mx.Accuracy.Double)
    assert mx.select(0.0, t) == (1, 0)
    assert mx.select(1.0, t) == (18, 0)
    assert mx.select(10.0, t) == (18, 4)
    assert mx.select(2.18, t) == (18, 1)
    for bad in (float("nan"), float("inf"), -1.0):
        with pytest.raises(ValueError):
            mx.select(bad, t)


def test_pade_selection_table_and_select(golden, oracle):
    """Family::PadeDiagonal table (theta_tables.cpp:61-73): 13 orders whose
    products tie in pairs/triples; mexp_select (the kernels' select_device)
    against the reference's selections and the restated ldexp loop."""
    t = mx.selection_table(mx.Family.PadeDiagonal, mx.Accuracy.Double)
    assert [e.degree for e in t.entries] == list(range(2, 27, 2))
    assert [e.products for e in t.entries] == [0, 1, 2, 3, 3, 4, 4, 5, 5, 5, 6, 6, 6]
    assert t.entries[-1].theta == 5.37
    assert mx.selection_table(mx.Family.PadeDiagonal, mx.Accuracy.Single).entries[-1].theta == 11.2
    g = golden("pade.npz")
    rng = np.random.default_rng(7)
    for acc in (0, 1):
        table = mx.selection_table(mx.Family.PadeDiagonal, mx.Accuracy(acc))
        for v, d, s, st in zip(g["norms"], g[f"degree_acc{acc}"], g[f"s_acc{acc}"],
                               g[f"status_acc{acc}"]):
            if st == 0:
                assert mx.select(float(v), table) == (d, s), (v, acc)
        for v in 10.0 ** rng.uniform(-20, 308, 3000):
            st, d, s = oracle.select(float(v), acc, 2)
            assert mx.select(float(v), table) == (d, s), (v, acc)


def test_pade_status_and_large_n_refusal(lib):
    assert lib.mexp_status_string(mx.ERR_SINGULAR) == b"singular denominator"  # kernels.cpp:72
    d, s = C.c_int32(), C.c_int32()
    assert lib.mexp_select(1.0, 1, 7, C.byref(d), C.byref(s)) == mx.ERR_INVALID_ARGUMENT


def test_ps_selection_table_and_select(golden):
    """Family::TaylorPS table (theta_tables.cpp:53-59) and mexp_select (the
    kernels' select_device) against the reference's selections."""
    for acc, th in ((1, [2.22e-16, 2.58e-8, 3.40e-4, 9.07e-3, 8.96e-2, 7.80e-1]),
                    (0, [1.19e-7, 5.98e-4, 5.12e-2, 2.50e-1, 7.80e-1, 2.48])):
        t = mx.selection_table(mx.Family.TaylorPS, mx.Accuracy(acc))
        assert [e.degree for e in t.entries] == [1, 2, 4, 6, 9, 16]
        assert [e.products for e in t.entries] == [0, 1, 2, 3, 4, 6]
        assert [e.theta for e in t.entries] == th
    g = golden("taylor_ps.npz")
    for acc in (0, 1):
        table = mx.selection_table(mx.Family.TaylorPS, mx.Accuracy(acc))
        for v, d, s, st in zip(g["norms"], g[f"degree_acc{acc}"], g[f"s_acc{acc}"],
                               g[f"status_acc{acc}"]):
            if st == 0:
                assert mx.select(float(v), table) == (d, s), (v, acc)


def test_ps_closed_form_scaling_exponent(oracle):
    rng = np.random.default_rng(6)
    for acc, tmax in ((0, 2.48), (1, 0.78)):
        table = mx.selection_table(mx.Family.TaylorPS, mx.Accuracy(acc))
        norms = [np.nextafter(tmax, np.inf), 1.7976931348623157e308, 1e-320, 0.0]
        for k in range(0, 1030, 7):
            v = np.ldexp(tmax, k)
            if np.isfinite(v):
                norms += [v, np.nextafter(v, 0.0), np.nextafter(v, np.inf)]
        norms += list(10.0 ** rng.uniform(-20, 308, 5000))
        for v in norms:
            st, d, s = oracle.select(float(v), acc, 1)
            assert st == 0
            assert mx.select(float(v), table) == (d, s), (v, acc)


def test_invalid_arguments(lib):
    a = np.zeros((2, 4, 4))
    out = np.empty_like(a)
    assert lib.mexp_expm_batched_host(a.ctypes.data, out.ctypes.data, 0, 0, 2, 1, 0, 0,
                                      None, None) == mx.ERR_INVALID_ARGUMENT  # n = 0
    assert lib.mexp_expm_batched_host(a.ctypes.data, out.ctypes.data, 7, 4, 2, 1, 0, 0,
                                      None, None) == mx.ERR_INVALID_ARGUMENT  # dtype
    assert lib.mexp_expm_batched_host(a.ctypes.data, out.ctypes.data, 0, 4, 2, 5, 0, 0,
                                      None, None) == mx.ERR_INVALID_ARGUMENT  # accuracy
    assert lib.mexp_expm_batched_host(a.ctypes.data, out.ctypes.data, 0, 4, 2, 1, 0, 9,
                                      None, None) == mx.ERR_INVALID_ARGUMENT  # rounding
    assert lib.mexp_expm_batched_host(a.ctypes.data, out.ctypes.data, 0, 4, 0, 1, 0, 0,
                                      None, None) == mx.OK  # empty batch is a no-op
    with pytest.raises(ValueError, match="square"):
        mx.expm(np.zeros((2, 3)))


def test_status_strings_match_reference_messages(lib):
    assert lib.mexp_status_string(1) == b"non-finite matrix entry"          # expm.cpp:38
    assert lib.mexp_status_string(2) == b"norm must be finite and nonnegative"  # expm.cpp:13


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mx.expm(np.eye(4))
    assert lib.mexp_device_check() == mx.ERR_NO_DEVICE


def test_selection_record_layout():
    assert C.sizeof(mx.Selection) == 16 and mx.SELECTION_DTYPE.itemsize == 16


def test_multi_device_entry_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    a = np.zeros((4, 8, 8))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mx.expm_batched_host_multi(a, devices=[0, 0])
    assert lib.mexp_device_count() == 0


def test_host_buffer_validation():
    """Caller buffers are checked before any pointer reaches the C ABI (a
    wrong-sized or wrong-typed `out` would otherwise be written past its end)."""
    import torch
    a = np.zeros((3, 8, 8))
    with pytest.raises(ValueError, match="out must be"):
        mx.expm_batched_host(a, out=np.empty((2, 8, 8)))
    with pytest.raises(ValueError, match="out must be"):
        mx.expm_batched_host(a, out=np.empty((3, 8, 8), np.float32))
    with pytest.raises(ValueError, match="out must be"):
        mx.expm_batched_host(a, out=np.empty((3, 8, 16))[:, :, ::2])
    with pytest.raises(ValueError, match="square"):
        mx.expm_batched_host(np.zeros((3, 8, 7)))
    with pytest.raises(ValueError, match="unsupported dtype"):
        mx.expm_batched_host(np.zeros((3, 8, 8), np.int64))
    t = torch.zeros(3, 8, 8, dtype=torch.float64)
    with pytest.raises(ValueError, match="out must be"):
        mx.expm_batched_host(t, out=torch.zeros(3, 8, 8, dtype=torch.float32))
    with pytest.raises(ValueError, match="sel_out"):
        mx.expm_batched_host(t, sel_out=torch.zeros(16, dtype=torch.uint8))
    with pytest.raises(ValueError, match="CUDA tensors"):
        mx.expm_batched(t, torch.empty_like(t))


def test_dense_layer_coefficient_tables_equal_reference(lib):
    """The drop-in's psi9_coefficients / pade_coeffs accessors (host tables of
    the library) are the reference's doubles bit for bit."""
    from oracle.oracle import REF_SO, Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    ref = C.CDLL(REF_SO)
    got, want = np.zeros(9), np.zeros(9)
    lib.mexp_b200_psi9_coefficients.argtypes = [C.c_void_p]
    lib.mexp_b200_psi9_coefficients(got.ctypes.data)
    ref.ref_psi9_coefficients.argtypes = [C.c_void_p]
    ref.ref_psi9_coefficients(want.ctypes.data)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    r = Reference()
    for m in range(1, 14):
        b = np.zeros(14)
        lib.mexp_b200_pade_coefficients.argtypes = [C.c_int, C.c_void_p]
        assert lib.mexp_b200_pade_coefficients(m, b.ctypes.data) == m + 1
        assert np.array_equal(b[:m + 1].view(np.uint64), r.pade_coeffs(m).view(np.uint64))
