"""B200-native scaling-and-squaring expm (arXiv 1710.10989, Family::TaylorNew).

Python mirror of the reference's C++ API (namespace ``mexp``:
proj/include/mexp/expm.hpp, theta_tables.hpp) over the C ABI in
``include/mexp_b200.h`` (library ``_lib/libmexp_b200.so``, built by ``make``).

* ``expm(a, accuracy, family) -> ExpmReport``      mexp::expm (expm.hpp:37)
* ``select(norm, table) -> Selection``             mexp::select (expm.hpp:18)
* ``selection_table(family, accuracy)``            theta_tables.hpp:32
* ``expm_batched(a, out, ...)``                    batched, device tensors
* ``expm_batched_host(a, ...)``                    batched, host arrays (e2e)
* ``expm_batched_host_multi(a, devices=...)``      the same, sharded by matrix
                                                   across several GPUs

Errors follow the reference: ``std::invalid_argument`` becomes ``ValueError``
with the reference's message. There is no CPU fallback: without the CUDA
library or a device every compute call raises ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libmexp_b200.so")

# mexp_status (include/mexp_b200.h)
OK, ERR_NONFINITE, ERR_NORM_NONFINITE, ERR_INVALID_ARGUMENT = 0, 1, 2, 3
ERR_UNSUPPORTED, ERR_CUDA, ERR_NO_DEVICE, ERR_SINGULAR = 4, 5, 6, 7
F64, F32 = 0, 1
ROUND_AUTO, ROUND_REFERENCE, ROUND_FAST = 0, 1, 2


class Family(enum.IntEnum):
    """theta_tables.hpp:8."""
    TaylorNew = 0
    TaylorPS = 1
    PadeDiagonal = 2


class Accuracy(enum.IntEnum):
    """theta_tables.hpp:9: u = 2^-24 (Single) or 2^-53 (Double)."""
    Single = 0
    Double = 1


class Selection(C.Structure):
    """mexp_selection: one 16-byte record per matrix."""
    _fields_ = [("norm_in", C.c_double), ("degree", C.c_int16), ("s", C.c_int16),
                ("status", C.c_int32)]


SELECTION_DTYPE = np.dtype([("norm_in", "<f8"), ("degree", "<i2"), ("s", "<i2"),
                            ("status", "<i4")])


class _Report(C.Structure):
    _fields_ = [("family", C.c_int32), ("degree", C.c_int32), ("s", C.c_int32),
                ("reserved", C.c_int32), ("cost_thirds", C.c_int64), ("norm_in", C.c_double)]


@dataclass
class SchemeDescriptor:
    """theta_tables.hpp:15-20."""
    family: Family
    degree: int
    products: int
    theta: float


@dataclass
class SelectionTable:
    """theta_tables.hpp:22-28."""
    family: Family
    accuracy: Accuracy
    entries: list

    def asymptotic(self) -> SchemeDescriptor:
        return self.entries[-1]

    def theta_max(self) -> float:
        return self.entries[-1].theta


@dataclass
class ExpmReport:
    """expm.hpp:23-32."""
    result: np.ndarray
    family: Family
    degree: int
    s: int
    cost_thirds: int
    norm_in: float

    def product_cost(self) -> float:
        return self.cost_thirds / 3.0


_lib = None


def library() -> C.CDLL:
    """Load the in-tree CUDA library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `make` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I, I64, D = C.c_void_p, C.c_int, C.c_int64, C.c_double
    sig = {
        "mexp_abi_version": (I, []),
        "mexp_device_check": (I, []),
        "mexp_status_string": (C.c_char_p, [I]),
        "mexp_last_cuda_error": (C.c_char_p, []),
        "mexp_launch_count": (C.c_uint64, []),
        "mexp_unit_roundoff": (D, [I]),
        "mexp_selection_table": (I, [I, I, P, P, P, I]),
        "mexp_select": (I, [D, I, I, P, P]),
        "mexp_expm": (I, [P, I, I, I, P, P]),
        "mexp_expm_batched": (I, [P, P, I, I, I64, I, I, I, P, P]),
        "mexp_expm_batched_host": (I, [P, P, I, I, I64, I, I, I, P, P]),
        "mexp_squarings_batched": (I, [P, I, I64, I, I, P]),
        "mexp_expm_batched_host_multi": (I, [P, P, I, I, I64, I, I, I, P, P, P, I]),
        "mexp_device_count": (I, []),
        "mexp_matmul_batched": (I, [P, P, P, I, I64, I, P]),
        "mexp_lincomb_batched": (I, [P, P, I, P, I64, P]),
        "mexp_one_norm_batched": (I, [P, I, I64, P, P]),
        "mexp_lu_solve_batched": (I, [P, P, P, I, I64, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


EXPORTED_SYMBOLS = (
    "mexp_abi_version", "mexp_device_check", "mexp_status_string", "mexp_last_cuda_error",
    "mexp_launch_count", "mexp_unit_roundoff", "mexp_selection_table", "mexp_select",
    "mexp_expm", "mexp_expm_batched", "mexp_expm_batched_host", "mexp_squarings_batched",
    "mexp_expm_batched_host_multi", "mexp_device_count",
    "mexp_matmul_batched", "mexp_lincomb_batched", "mexp_one_norm_batched", "mexp_lu_solve_batched",
)


def _raise(status: int):
    lib = library()
    msg = lib.mexp_status_string(status).decode()
    if status in (ERR_NONFINITE, ERR_NORM_NONFINITE, ERR_INVALID_ARGUMENT, ERR_UNSUPPORTED):
        raise ValueError(msg)
    if status == ERR_CUDA:
        raise RuntimeError(f"{msg}: {lib.mexp_last_cuda_error().decode()}")
    raise RuntimeError(msg)


def unit_roundoff(u: Accuracy) -> float:
    return library().mexp_unit_roundoff(int(u))


def selection_table(family: Family, u: Accuracy) -> SelectionTable:
    """mexp::selection_table (theta_tables.cpp:77-85)."""
    d = np.zeros(16, np.int32)
    p = np.zeros(16, np.int32)
    t = np.zeros(16, np.float64)
    k = library().mexp_selection_table(int(u), int(family), d.ctypes.data, p.ctypes.data,
                                       t.ctypes.data, 16)
    if k < 0:
        _raise(-k)
    return SelectionTable(Family(family), Accuracy(u),
                          [SchemeDescriptor(Family(family), int(d[i]), int(p[i]), float(t[i]))
                           for i in range(k)])


def select(norm: float, table: SelectionTable):
    """mexp::select (expm.cpp:11-29) -> (degree, s)."""
    d, s = C.c_int32(), C.c_int32()
    st = library().mexp_select(float(norm), int(table.accuracy), int(table.family),
                               C.byref(d), C.byref(s))
    if st != OK:
        _raise(st)
    return d.value, s.value


def expm(a: np.ndarray, u: Accuracy = Accuracy.Double,
         family: Family = Family.TaylorNew) -> ExpmReport:
    """mexp::expm (expm.cpp:37-74) on one host matrix, computed on the GPU."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] < 1:
        raise ValueError("matrix must be square")
    n = a.shape[0]
    out = np.empty_like(a)
    rep = _Report()
    st = library().mexp_expm(a.ctypes.data, n, int(u), int(family), out.ctypes.data, C.byref(rep))
    if st != OK:
        _raise(st)
    return ExpmReport(out, Family(family), rep.degree, rep.s, rep.cost_thirds, rep.norm_in)


def _dtype_code(dt) -> int:
    s = str(dt)
    if "float64" in s:
        return F64
    if "float32" in s:
        return F32
    raise ValueError(f"unsupported dtype {dt}")


def expm_batched(a, out, sel=None, accuracy: Accuracy = Accuracy.Double,
                 rounding: int = ROUND_AUTO, stream=None, family: Family = Family.TaylorNew):
    """Batched expm on device tensors (torch, CUDA, contiguous (batch, n, n)).

    ``sel``: optional uint8 device tensor of 16*batch bytes (SELECTION_DTYPE
    records). Asynchronous on ``stream`` (default: torch's current stream).
    """
    import torch
    if not (a.is_cuda and out.is_cuda):
        raise ValueError("expm_batched takes CUDA tensors (expm_batched_host takes host buffers)")
    if a.dim() != 3 or a.shape[1] != a.shape[2]:
        raise ValueError("a must be a (batch, n, n) stack of square matrices")
    batch, n, _ = a.shape
    if out.shape != a.shape or out.dtype != a.dtype:
        raise ValueError("dimension mismatch")
    if not (a.is_contiguous() and out.is_contiguous()):
        raise ValueError("a and out must be contiguous")
    if a.device != out.device or a.device.index != torch.cuda.current_device():
        raise ValueError("a and out must live on the current CUDA device")
    if sel is not None and (not sel.is_cuda or sel.device != a.device or not sel.is_contiguous()
                            or sel.numel() * sel.element_size() < SELECTION_DTYPE.itemsize * batch):
        raise ValueError(f"sel must be a contiguous device buffer of >= {SELECTION_DTYPE.itemsize} "
                         "bytes per matrix on a's device")
    if stream is None:
        stream = torch.cuda.current_stream(a.device)
    st = library().mexp_expm_batched(a.data_ptr(), out.data_ptr(), _dtype_code(a.dtype), n,
                                     batch, int(accuracy), int(family), int(rounding),
                                     None if sel is None else sel.data_ptr(),
                                     C.c_void_p(stream.cuda_stream))
    if st != OK:
        _raise(st)


_PINNED_SEL = {}


def _pinned_selection(batch: int):
    """A cached pinned uint8 tensor holding >= batch selection records."""
    import torch
    buf = _PINNED_SEL.get("buf")
    need = batch * SELECTION_DTYPE.itemsize
    if buf is None or buf.numel() < need:
        buf = torch.empty(need, dtype=torch.uint8, pin_memory=True)
        _PINNED_SEL["buf"] = buf
    return buf


def _host_args(a, out):
    """Validate host (numpy or CPU torch) buffers; returns (a, out, ptrs, batch, n, dtype code)."""
    if isinstance(a, np.ndarray):
        if a.ndim != 3 or a.shape[1] != a.shape[2]:
            raise ValueError("a must be a (batch, n, n) stack of square matrices")
        a = np.ascontiguousarray(a)
        dt = _dtype_code(a.dtype)
        if out is None:
            out = np.empty_like(a)
        elif not isinstance(out, np.ndarray) or out.shape != a.shape or out.dtype != a.dtype \
                or not out.flags.c_contiguous or not out.flags.writeable:
            raise ValueError("out must be a writeable C-contiguous array of a's shape and dtype")
        return a, out, a.ctypes.data, out.ctypes.data, a.shape[0], a.shape[1], dt
    import torch
    if not isinstance(a, torch.Tensor) or a.is_cuda:
        raise ValueError("expm_batched_host takes host buffers (numpy arrays or CPU tensors)")
    if a.dim() != 3 or a.shape[1] != a.shape[2]:
        raise ValueError("a must be a (batch, n, n) stack of square matrices")
    a = a.contiguous()
    dt = _dtype_code(a.dtype)
    if out is None:
        out = a.new_empty(a.shape)
    elif not isinstance(out, torch.Tensor) or out.is_cuda or out.shape != a.shape \
            or out.dtype != a.dtype or not out.is_contiguous():
        raise ValueError("out must be a contiguous CPU tensor of a's shape and dtype")
    return a, out, a.data_ptr(), out.data_ptr(), a.shape[0], a.shape[1], dt


def _host_sel(a, batch, sel_out):
    if isinstance(a, np.ndarray):
        sel = np.zeros(batch, SELECTION_DTYPE)
        return sel, sel.ctypes.data
    import torch
    # pinned like the caller's tensors, so the records are DMA'd straight
    # in; the pinned buffer is cached (cudaHostAlloc costs ~ms per call)
    if sel_out is None:
        sel_t = _pinned_selection(batch) if a.is_pinned() else \
            torch.empty(batch * SELECTION_DTYPE.itemsize, dtype=torch.uint8)
    else:
        if not isinstance(sel_out, torch.Tensor) or sel_out.is_cuda or sel_out.dtype != torch.uint8 \
                or not sel_out.is_contiguous() or sel_out.numel() < batch * SELECTION_DTYPE.itemsize:
            raise ValueError(f"sel_out must be a contiguous CPU uint8 tensor of >= "
                             f"{SELECTION_DTYPE.itemsize} bytes per matrix")
        sel_t = sel_out
    return sel_t.numpy().view(SELECTION_DTYPE)[:batch], sel_t.data_ptr()


def expm_batched_host(a, out=None, accuracy: Accuracy = Accuracy.Double,
                      rounding: int = ROUND_AUTO, family: Family = Family.TaylorNew,
                      raise_on_error: bool = True, sel_out=None):
    """Batched expm on host buffers (numpy arrays or pinned CPU torch tensors).

    For torch inputs the selection records land in ``sel_out`` (a uint8
    tensor of >= 16*batch bytes) or in a cached pinned buffer; the returned
    records view is only valid until the next call in that case.

    Returns (out, selection records as a numpy structured array, status).
    """
    a, out, pa, po, batch, n, dt = _host_args(a, out)
    sel, psel = _host_sel(a, batch, sel_out)
    first = C.c_int64(-1)
    st = library().mexp_expm_batched_host(pa, po, dt, n, batch, int(accuracy), int(family),
                                          int(rounding), psel, C.byref(first))
    if st not in (OK, ERR_NONFINITE, ERR_NORM_NONFINITE) or (st != OK and raise_on_error):
        _raise(st)
    return out, sel, st


def expm_batched_host_multi(a, out=None, devices=None, accuracy: Accuracy = Accuracy.Double,
                            rounding: int = ROUND_AUTO, family: Family = Family.TaylorNew,
                            raise_on_error: bool = True, sel_out=None):
    """``expm_batched_host`` sharded by matrix across ``devices`` (default: all
    visible GPUs), one host thread and copy pipeline per GPU
    (``mexp_expm_batched_host_multi``). Same results, records and status as
    the single-device call. Returns (out, records, status, first_error)."""
    a, out, pa, po, batch, n, dt = _host_args(a, out)
    sel, psel = _host_sel(a, batch, sel_out)
    devs = None if devices is None else np.ascontiguousarray(devices, dtype=np.int32)
    first = C.c_int64(-1)
    st = library().mexp_expm_batched_host_multi(
        pa, po, dt, n, batch, int(accuracy), int(family), int(rounding), psel, C.byref(first),
        None if devs is None else devs.ctypes.data, 0 if devs is None else len(devs))
    if st not in (OK, ERR_NONFINITE, ERR_NORM_NONFINITE) or (st != OK and raise_on_error):
        _raise(st)
    return out, sel, st, first.value


def device_count() -> int:
    return int(library().mexp_device_count())


# ---- the reference's dense-matrix layer on device tensors (kernels.hpp) ----
def _stream(t, stream):
    import torch
    return C.c_void_p((stream or torch.cuda.current_stream(t.device)).cuda_stream)


def _dev_f64(*ts):
    for t in ts:
        if not (t.is_cuda and t.dtype.is_floating_point and t.element_size() == 8 and t.is_contiguous()):
            raise ValueError("expected contiguous float64 CUDA tensors")


def matmul_batched(a, b, out=None, rounding: int = ROUND_REFERENCE, stream=None):
    """kernels::matmul (kernels.cpp:16-27) on (batch, n, n) or (n, n) device
    tensors; REFERENCE rounding is bit-identical to the reference."""
    import torch
    out = torch.empty_like(a) if out is None else out
    _dev_f64(a, b, out)
    if a.shape != b.shape or out.shape != a.shape or a.shape[-1] != a.shape[-2]:
        raise ValueError("dimension mismatch")
    n = a.shape[-1]
    st = library().mexp_matmul_batched(a.data_ptr(), b.data_ptr(), out.data_ptr(), n,
                                       a.numel() // (n * n), int(rounding), _stream(a, stream))
    if st != OK:
        _raise(st)
    return out


def lincomb_batched(coeffs, mats, out=None, stream=None):
    """kernels::lincomb (kernels.cpp:29-37): sum_i coeffs[i] * mats[i], left to right."""
    import torch
    if len(coeffs) != len(mats) or not mats:
        raise ValueError("lincomb needs equally long nonempty lists")
    out = torch.empty_like(mats[0]) if out is None else out
    _dev_f64(out, *mats)
    if any(m.shape != out.shape for m in mats):
        raise ValueError("dimension mismatch")
    c = (C.c_double * len(coeffs))(*[float(x) for x in coeffs])
    p = (C.c_void_p * len(mats))(*[m.data_ptr() for m in mats])
    st = library().mexp_lincomb_batched(c, p, len(mats), out.data_ptr(), out.numel(),
                                        _stream(out, stream))
    if st != OK:
        _raise(st)
    return out


def one_norm_batched(a, stream=None):
    """kernels::one_norm (kernels.cpp:44-53) per matrix of a (batch, n, n) tensor."""
    import torch
    _dev_f64(a)
    n = a.shape[-1]
    batch = a.numel() // (n * n)
    out = torch.empty(batch, dtype=a.dtype, device=a.device)
    st = library().mexp_one_norm_batched(a.data_ptr(), n, batch, out.data_ptr(), _stream(a, stream))
    if st != OK:
        _raise(st)
    return out


def lu_solve_batched(m, rhs, stream=None):
    """lu_solve (kernels.cpp:55-112) per matrix: returns (X, status) with
    status[i] = ERR_SINGULAR where the reference throws "singular denominator"."""
    import torch
    _dev_f64(m, rhs)
    if m.shape != rhs.shape:
        raise ValueError("dimension mismatch")
    n = m.shape[-1]
    batch = m.numel() // (n * n)
    x = torch.empty_like(m)
    status = torch.empty(batch, dtype=torch.int32, device=m.device)
    st = library().mexp_lu_solve_batched(m.data_ptr(), rhs.data_ptr(), x.data_ptr(), n, batch,
                                         status.data_ptr(), _stream(m, stream))
    if st != OK:
        _raise(st)
    return x, status


def launch_count() -> int:
    return int(library().mexp_launch_count())


def products_of_degree(m: int) -> int:
    return {1: 0, 2: 1, 4: 2, 8: 3, 12: 4, 18: 5}[int(m)]
