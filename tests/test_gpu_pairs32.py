"""The 32x32 fp32 pair kernel (csrc/expm32_pairs.cu: two same-class matrices
per warp, 8x8 lane tiles, TMEM-parked intermediates) against the one-warp
kernel (csrc/expm_small_f32.cu) it replaces for Family::TaylorNew.

Both evaluate eval_taylor_new and the squarings with the same fp32 operations
in the same order (taylor_schemes.cpp:104-157, 211-227), so e^A must agree
bit for bit, and the selection records of the pre-pass must equal the
one-warp kernel's (kernels.cpp:44-53, expm.cpp:11-29). Inputs cover every
degree of the Single table (norms 1e-9 .. 1e3, so s up to ~9), class
boundaries that force mixed pairs, odd batch sizes, non-finite matrices in the
middle of a class and padded n.
"""
import os

import numpy as np
import pytest

import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads

pytestmark = pytest.mark.gpu
U24 = 2.0 ** -24


def _run(a, pairs, accuracy=mx.Accuracy.Single):
    old = os.environ.get("MEXP_F32_PAIRS")
    os.environ["MEXP_F32_PAIRS"] = "1" if pairs else "0"
    try:
        out, sel, st = mx.expm_batched_host(a, accuracy=accuracy, raise_on_error=False)
    finally:
        if old is None:
            del os.environ["MEXP_F32_PAIRS"]
        else:
            os.environ["MEXP_F32_PAIRS"] = old
    assert st in (mx.OK, mx.ERR_NONFINITE)
    return out, sel


def _spread(n, batch, seed, lo=1e-9, hi=1e3):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((batch, n, n)) / np.sqrt(n)
    a[1::3] = a[1::3] - np.swapaxes(a[1::3], 1, 2)  # some skew-symmetric
    norms = np.abs(a).sum(axis=1).max(axis=1)
    target = np.exp(rng.uniform(np.log(lo), np.log(hi), batch))
    return (a * (target / norms)[:, None, None]).astype(np.float32)


def _same_bits(x, y):
    return np.array_equal(x.view(np.uint32), y.view(np.uint32))


@pytest.mark.parametrize("batch", [1, 2, 3, 65, 4097])
def test_pairs_bitwise_equal_one_warp_kernel(cuda, batch):
    a = _spread(32, batch, seed=batch)
    o1, s1 = _run(a, True)
    o0, s0 = _run(a, False)
    assert np.array_equal(s1.view(np.uint8), s0.view(np.uint8))
    assert _same_bits(o1, o0)
    degrees = set(s1["degree"].tolist())
    if batch >= 4097:
        assert degrees == {1, 2, 4, 8, 12, 18}, degrees


def test_pairs_cfg3_bitwise_and_oracle(cuda, oracle):
    # the full batch: four chunks, the pre-pass of chunks 1..3 pipelined on side streams
    a = workloads.generate("cfg3")
    o1, s1 = _run(a, True)
    o0, s0 = _run(a, False)
    assert np.array_equal(s1.view(np.uint8), s0.view(np.uint8))
    assert _same_bits(o1, o0)
    ref = oracle.expm_batch(a[:2048].astype(np.float64), accuracy=0)
    assert np.array_equal(s1["degree"][:2048], ref.degree) and np.array_equal(s1["s"][:2048], ref.s)
    err = np.linalg.norm((o1[:2048] - ref.out).reshape(2048, -1), axis=1) / np.linalg.norm(
        ref.out.reshape(2048, -1), axis=1)
    assert err.max() <= 50 * 32 * U24


def test_pairs_non_finite_inside_classes(cuda):
    a = _spread(32, 301, seed=7, lo=0.5, hi=2.0)  # few classes, long runs
    a[5, 3, 4] = np.nan
    a[100, 0, 0] = np.inf
    a[101, 31, 31] = -np.inf
    o1, s1 = _run(a, True)
    o0, s0 = _run(a, False)
    assert np.array_equal(s1.view(np.uint8), s0.view(np.uint8))
    assert _same_bits(o1, o0)
    bad = [5, 100, 101]
    assert (s1["status"][bad] == mx.ERR_NONFINITE).all()
    assert np.isnan(o1[bad]).all()
    good = np.setdiff1d(np.arange(301), bad)
    assert np.isfinite(o1[good]).all()


@pytest.mark.parametrize("n", [17, 24, 31])
def test_pairs_padded_sizes(cuda, n):
    a = _spread(n, 513, seed=n)
    o1, s1 = _run(a, True)
    o0, s0 = _run(a, False)
    assert np.array_equal(s1.view(np.uint8), s0.view(np.uint8))
    assert _same_bits(o1, o0)


def test_pairs_large_s(cuda):
    # s > 126 takes the fp64 scaling branch: 2^-s is no longer a normal float
    a = _spread(32, 64, seed=3, lo=1e30, hi=1e38)
    o1, s1 = _run(a, True)
    o0, s0 = _run(a, False)
    assert s1["s"].max() > 100
    assert np.array_equal(s1.view(np.uint8), s0.view(np.uint8))
    assert _same_bits(o1, o0)


def test_pairs_pipelined_under_graph_capture(cuda):
    # the chunked pipeline forks onto side streams; captured into a CUDA graph
    # and replayed it must give the eager call's bits
    import torch
    a_np = _spread(32, 70001, seed=11, lo=1e-3, hi=60.0)
    a = torch.from_numpy(a_np).cuda()
    ref = torch.empty_like(a)
    sel_ref = torch.empty(a.shape[0] * 16, dtype=torch.uint8, device=cuda)
    mx.expm_batched(a, ref, sel_ref, accuracy=mx.Accuracy.Single)
    out = torch.full_like(a, float("nan"))
    sel = torch.zeros_like(sel_ref)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        mx.expm_batched(a, out, sel, accuracy=mx.Accuracy.Single)  # warm (allocations)
        with torch.cuda.graph(g, stream=s):
            mx.expm_batched(a, out, sel, accuracy=mx.Accuracy.Single)
    out.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int32), ref.view(torch.int32))
    assert torch.equal(sel, sel_ref)


def test_pairs_double_table(cuda):
    # fp32 storage with the Double table: larger s for the same norms, every degree
    a = _spread(32, 2049, seed=5, lo=1e-12, hi=1e4)
    o1, s1 = _run(a, True, mx.Accuracy.Double)
    o0, s0 = _run(a, False, mx.Accuracy.Double)
    assert np.array_equal(s1.view(np.uint8), s0.view(np.uint8))
    assert _same_bits(o1, o0)
    assert s1["s"].max() >= 10
