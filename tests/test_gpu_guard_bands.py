"""Out-of-bounds and aliasing checks of our own (compute-sanitizer is closed on
this GPU pool: it has left GPUs needing a reset). Every device entry point
runs on buffers carved out of larger allocations filled with a canary
pattern; after the call the canaries before and after each input, output and
record buffer must be untouched, and the inputs unchanged. Covers the 8x8
kernels (every rounding, work tickets, captured graphs), the n <= 64 group
kernels (padded n, fp32), the 32x32 fp32 pair kernel, the 64x64 cluster kernel, the large-n GEMM chain
(TaylorNew, PS, Pade LU), the dense layer and the multi-device host entry.
"""
import numpy as np
import pytest

import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements of canary on each side
CANARY = -1.2345678e30  # representable in fp32 and fp64; never produced by the kernels here


def guarded(shape, dtype, fill=None):
    import torch
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), CANARY, dtype=dtype, device="cuda")
    view = buf[GUARD:GUARD + n].view(shape)
    if fill is not None:
        view.copy_(fill)
    return buf, view


def intact(buf, n):
    import torch
    c = torch.tensor(CANARY, dtype=buf.dtype, device=buf.device)
    return bool((buf[:GUARD] == c).all()) and bool((buf[GUARD + n:] == c).all())


CASES = [  # (n, batch, dtype, family, rounding)
    (8, 1000, "f64", 0, mx.ROUND_AUTO), (8, 1000, "f64", 0, mx.ROUND_REFERENCE),
    (8, 999, "f64", 1, mx.ROUND_FAST), (8, 513, "f64", 2, mx.ROUND_AUTO),
    (5, 77, "f64", 0, mx.ROUND_AUTO), (13, 50, "f64", 0, mx.ROUND_AUTO),
    (32, 40, "f32", 0, mx.ROUND_AUTO), (24, 9, "f32", 2, mx.ROUND_AUTO),
    (64, 1, "f64", 0, mx.ROUND_AUTO), (64, 200, "f64", 0, mx.ROUND_REFERENCE),
    (100, 3, "f64", 0, mx.ROUND_AUTO), (128, 2, "f64", 1, mx.ROUND_FAST),
    (130, 2, "f64", 2, mx.ROUND_AUTO), (96, 2, "f64", 0, mx.ROUND_REFERENCE),
]


@pytest.mark.parametrize("n,batch,dt,family,rounding", CASES)
def test_expm_batched_stays_in_bounds(cuda, n, batch, dt, family, rounding):
    _in_bounds(n, batch, dt, family, rounding)


@pytest.mark.parametrize("n,batch", [(32, 333), (20, 101), (32, 8193)])
def test_pair_kernel_stays_in_bounds(cuda, n, batch, monkeypatch):
    # the 32x32 fp32 pair kernel and its pre-pass (csrc/expm32_pairs.cu), forced at any batch
    monkeypatch.setenv("MEXP_F32_PAIRS", "1")
    _in_bounds(n, batch, "f32", 0, mx.ROUND_AUTO)


def _in_bounds(n, batch, dt, family, rounding):
    import torch
    tdt = torch.float64 if dt == "f64" else torch.float32
    rng = np.random.default_rng(n * 1000 + batch)
    norms = 10.0 ** rng.uniform(-3, 2.5, batch)
    a = rng.uniform(-1, 1, (batch, n, n))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    a[batch // 2, 0, n - 1] = np.nan
    src = torch.from_numpy(a).to(tdt)
    ab, av = guarded((batch, n, n), tdt, src.cuda())
    ob, ov = guarded((batch, n, n), tdt)
    sb, sv = guarded((batch * 2,), torch.float64)  # 16-byte records under 8-byte canaries
    sel = sv.view(torch.uint8)
    acc = mx.Accuracy.Single if dt == "f32" else mx.Accuracy.Double
    mx.expm_batched(av, ov, sel, accuracy=acc, rounding=rounding, family=mx.Family(family))
    torch.cuda.synchronize()
    assert intact(ab, batch * n * n) and intact(ob, batch * n * n) and intact(sb, batch * 2)
    ibits = torch.int64 if dt == "f64" else torch.int32
    assert torch.equal(av.cpu().view(ibits), src.view(ibits))  # input untouched (NaN included)
    rec = sel.cpu().numpy().view(mx.SELECTION_DTYPE)
    assert rec["status"][batch // 2] == mx.ERR_NONFINITE
    assert (rec["status"] != mx.ERR_NONFINITE).sum() == batch - 1


def test_graph_replays_and_dense_layer_stay_in_bounds(cuda):
    import torch
    a = torch.from_numpy(workloads.generate("cfg2", 0, 3000)).cuda()
    ob, ov = guarded(tuple(a.shape), torch.float64)
    g = torch.cuda.CUDAGraph()
    mx.expm_batched(a, ov)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        mx.expm_batched(a, ov, stream=torch.cuda.current_stream())
    for _ in range(5):
        g.replay()
        mx.expm_batched(a, ov)  # eager launches between replays use other ticket slots
    torch.cuda.synchronize()
    assert intact(ob, a.numel())
    for n in (7, 64, 100):
        x = torch.from_numpy(np.random.default_rng(n).uniform(-1, 1, (3, n, n))).cuda()
        cb, cv = guarded((3, n, n), torch.float64)
        mx.matmul_batched(x, x, out=cv)
        mx.lincomb_batched([1.0, 2.0], [x, x], out=cv)
        nb, nv = guarded((3,), torch.float64)
        nv.copy_(mx.one_norm_batched(x))
        torch.cuda.synchronize()
        assert intact(cb, 3 * n * n) and intact(nb, 3)


def test_multi_device_host_entry_stays_in_bounds(cuda):
    a = workloads.generate("cfg2", 0, 1001)
    out = np.full((1001 + 2 * 8, 8, 8), CANARY)
    o = out[8:-8]
    mx.expm_batched_host_multi(a, out=o, devices=[0, 0, 0])
    assert (out[:8] == CANARY).all() and (out[-8:] == CANARY).all()
