"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

Two libraries, both built by ``oracle/Makefile``:

* ``_ref/libmexp_ref.so``: the unmodified reference (`mexp`) compiled from
  /root/reference/proj/src plus ``ref_shim.cpp`` (the ``ref_*`` symbols).
* ``_build/libexpm_oracle.so``: the plain-C restatement ``expm_oracle.c``
  (the ``oracle_*`` symbols).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) import this module, and only as
the checker or the CPU baseline. The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmexp_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "libexpm_oracle.so")

_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_D = C.c_double


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _Lib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.prefix = prefix

    def fn(self, name, restype, *argtypes):
        f = getattr(self.lib, self.prefix + name)
        f.restype = restype
        f.argtypes = list(argtypes)
        return f


class ExpmResult:
    """Per-matrix outputs of a batched expm: e^A plus the ExpmReport fields."""

    def __init__(self, out, degree, s, cost_thirds, norm_in, status, ret):
        self.out = out
        self.degree = degree
        self.s = s
        self.cost_thirds = cost_thirds
        self.norm_in = norm_in
        self.status = status
        self.ret = ret


def _alloc(batch: int, n: int):
    return (np.empty((batch, n, n), np.float64), np.zeros(batch, np.int32),
            np.zeros(batch, np.int32), np.zeros(batch, np.int64),
            np.zeros(batch, np.float64), np.zeros(batch, np.int32))


class Reference:
    """The compiled reference library (oracle/_ref)."""

    available = staticmethod(lambda: os.path.exists(REF_SO))

    def __init__(self):
        L = _Lib(REF_SO, "ref_")
        self._batch64 = L.fn("expm_batch_f64", _I, _P, _P, _I, _I64, _I, _I, _P, _P, _P, _P, _P)
        self._batch32 = L.fn("expm_batch_f32_out64", _I, _P, _P, _I, _I64, _I, _I, _P, _P, _P, _P, _P)
        self._select = L.fn("select", _I, _D, _I, _I, _P, _P)
        self._one_norm = L.fn("one_norm", _D, _P, _I)
        self._matmul = L.fn("matmul", None, _P, _P, _P, _I)
        self._theta = L.fn("theta_table", _I, _I, _I, _P, _P, _P, _I)
        self._eval = L.fn("eval_taylor_new", _I, _P, _I, _I, _P)
        self._horner = L.fn("taylor_oracle", None, _P, _I, _I, _P)
        self._coef = L.fn("coefficients", None, _P, _P, _P, _P)
        self._pade_b = L.fn("pade_coeffs", _I, _I, _P)
        self._eval_pade = L.fn("eval_pade", _I, _P, _I, _I, _P)

    def pade_coeffs(self, m: int) -> np.ndarray:
        b = np.zeros(14)
        k = self._pade_b(m, _ptr(b))
        return b[:k]

    def eval_pade(self, a, order):
        a = np.ascontiguousarray(a, np.float64)
        out = np.empty_like(a)
        k = self._eval_pade(_ptr(a), a.shape[0], order, _ptr(out))
        return k, out

    def expm_batch(self, a: np.ndarray, accuracy: int = 1, family: int = 0) -> ExpmResult:
        batch, n, _ = a.shape
        out, deg, s, cost, norm, st = _alloc(batch, n)
        if a.dtype == np.float32:
            a = np.ascontiguousarray(a)
            ret = self._batch32(_ptr(a), _ptr(out), n, batch, accuracy, family, _ptr(deg),
                                _ptr(s), _ptr(cost), _ptr(norm), _ptr(st))
        else:
            a = np.ascontiguousarray(a, np.float64)
            ret = self._batch64(_ptr(a), _ptr(out), n, batch, accuracy, family, _ptr(deg),
                                _ptr(s), _ptr(cost), _ptr(norm), _ptr(st))
        return ExpmResult(out, deg, s, cost, norm, st, ret)

    def select(self, norm: float, accuracy: int = 1, family: int = 0):
        d, s = C.c_int32(), C.c_int32()
        st = self._select(norm, accuracy, family, C.byref(d), C.byref(s))
        return st, d.value, s.value

    def one_norm(self, a: np.ndarray) -> float:
        a = np.ascontiguousarray(a, np.float64)
        return self._one_norm(_ptr(a), a.shape[0])

    def matmul(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        c = np.empty_like(a)
        self._matmul(_ptr(a), _ptr(b), _ptr(c), a.shape[0])
        return c

    def theta_table(self, accuracy: int = 1, family: int = 0):
        d = np.zeros(16, np.int32); p = np.zeros(16, np.int32); t = np.zeros(16, np.float64)
        k = self._theta(accuracy, family, _ptr(d), _ptr(p), _ptr(t), 16)
        return d[:k], p[:k], t[:k]

    def eval_taylor_new(self, a, degree):
        a = np.ascontiguousarray(a, np.float64)
        out = np.empty_like(a)
        k = self._eval(_ptr(a), a.shape[0], degree, _ptr(out))
        return k, out

    def taylor_oracle(self, a, degree):
        a = np.ascontiguousarray(a, np.float64)
        out = np.empty_like(a)
        self._horner(_ptr(a), a.shape[0], degree, _ptr(out))
        return out

    def coefficients(self):
        t8 = np.zeros(10); t12 = np.zeros(16); a = np.zeros(4); b = np.zeros(20)
        self._coef(_ptr(t8), _ptr(t12), _ptr(a), _ptr(b))
        return t8, t12.reshape(4, 4), a, b.reshape(4, 5)


class Oracle:
    """The plain-C restatement (oracle/expm_oracle.c)."""

    def __init__(self):
        L = _Lib(ORACLE_SO, "oracle_")
        self._batch = L.fn("expm_batch_family", _I, _P, _P, _I, _I64, _I, _I, _P, _P, _P, _P, _P)
        self._select = L.fn("select_family", _I, _D, _I, _I, _P, _P)
        self._eval_ps = L.fn("eval_taylor_ps", _I, _P, _I, _I, _P)
        self._pade_b = L.fn("pade_coeffs", _I, _I, _P)
        self._eval_pade = L.fn("eval_pade", _I, _P, _I, _I, _P)
        self._one_norm = L.fn("one_norm", _D, _P, _I)
        self._matmul = L.fn("matmul", None, _P, _P, _P, _I)
        self._eval = L.fn("eval_taylor_new", _I, _P, _I, _I, _P)
        self._coef = L.fn("coefficients", None, _P, _P, _P, _P)
        self._forced = L.fn("expm_forced", _I, _P, _I, _I, _I, _P)

    def pade_coeffs(self, m: int) -> np.ndarray:
        b = np.zeros(14)
        k = self._pade_b(m, _ptr(b))
        return b[:k]

    def eval_pade(self, a, order):
        a = np.ascontiguousarray(a, np.float64)
        out = np.empty_like(a)
        k = self._eval_pade(_ptr(a), a.shape[0], order, _ptr(out))
        return k, out

    def expm_forced(self, a: np.ndarray, degree: int, s: int) -> np.ndarray:
        """T_degree(2^-s A)^(2^s) with the given (m, s) (oracle_expm_forced)."""
        a = np.ascontiguousarray(a, np.float64)
        out = np.empty_like(a)
        k = self._forced(_ptr(a), a.shape[0], degree, s, _ptr(out))
        if k < 0:
            raise ValueError("unsupported degree")
        return out

    def expm_batch(self, a: np.ndarray, accuracy: int = 1, family: int = 0) -> ExpmResult:
        batch, n, _ = a.shape
        a = np.ascontiguousarray(a.astype(np.float64, copy=False))
        out, deg, s, cost, norm, st = _alloc(batch, n)
        ret = self._batch(_ptr(a), _ptr(out), n, batch, accuracy, family, _ptr(deg), _ptr(s),
                          _ptr(cost), _ptr(norm), _ptr(st))
        return ExpmResult(out, deg, s, cost, norm, st, ret)

    def select(self, norm: float, accuracy: int = 1, family: int = 0):
        d, s = C.c_int32(), C.c_int32()
        st = self._select(norm, accuracy, family, C.byref(d), C.byref(s))
        return st, d.value, s.value

    def eval_taylor_ps(self, a, degree):
        a = np.ascontiguousarray(a, np.float64)
        out = np.empty_like(a)
        k = self._eval_ps(_ptr(a), a.shape[0], degree, _ptr(out))
        return k, out

    def one_norm(self, a):
        a = np.ascontiguousarray(a, np.float64)
        return self._one_norm(_ptr(a), a.shape[0])

    def matmul(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        c = np.empty_like(a)
        self._matmul(_ptr(a), _ptr(b), _ptr(c), a.shape[0])
        return c

    def eval_taylor_new(self, a, degree):
        a = np.ascontiguousarray(a, np.float64)
        out = np.empty_like(a)
        k = self._eval(_ptr(a), a.shape[0], degree, _ptr(out))
        return k, out

    def coefficients(self):
        t8 = np.zeros(10); t12 = np.zeros(16); a = np.zeros(4); b = np.zeros(20)
        self._coef(_ptr(t8), _ptr(t12), _ptr(a), _ptr(b))
        return t8, t12.reshape(4, 4), a, b.reshape(4, 5)


def rel_frobenius(got: np.ndarray, want: np.ndarray) -> np.ndarray:
    """Per-matrix ||got - want||_F / ||want||_F over a (batch, n, n) stack."""
    g = got.astype(np.float64).reshape(got.shape[0], -1)
    w = want.astype(np.float64).reshape(want.shape[0], -1)
    return np.linalg.norm(g - w, axis=1) / np.linalg.norm(w, axis=1)
