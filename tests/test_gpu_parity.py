"""GPU parity: the CUDA path, called through the C ABI, against the oracle.

Bars (BASELINE.json north_star): the selected (m, s) equal per matrix, bit
for bit, with norm_in; e^A within relative Frobenius 50*N*u of the
reference; in REFERENCE rounding, e^A bit-identical to the reference.
"""
import numpy as np
import pytest

import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads

pytestmark = pytest.mark.gpu

U53 = 2.0 ** -53
MODES = {"reference": mx.ROUND_REFERENCE, "auto": mx.ROUND_AUTO, "fast": mx.ROUND_FAST}


def rel_fro(got, want):
    g = got.reshape(got.shape[0], -1).astype(np.float64)
    w = want.reshape(want.shape[0], -1).astype(np.float64)
    return np.linalg.norm(g - w, axis=1) / np.linalg.norm(w, axis=1)


def bits(x):
    return np.ascontiguousarray(x).view(np.uint64)


def golden_groups(golden):
    """Golden expm cases grouped by (n, accuracy) -> stacked arrays."""
    g = golden("expm_cases.npz")
    groups = {}
    for entry in g["names"]:
        key, name = str(entry).split(":", 1)
        acc = int(key.split("_acc")[1])
        a = g[key + "_a"]
        groups.setdefault((a.shape[0], acc), []).append(
            (name, a, g[key + "_out"], g[key + "_meta"], g[key + "_norm"][0]))
    return groups


@pytest.mark.parametrize("mode", ["reference", "auto", "fast"])
def test_golden_cases(cuda, golden, mode):
    for (n, acc), cases in golden_groups(golden).items():
        a = np.stack([c[1] for c in cases])
        out, sel, st = mx.expm_batched_host(a, accuracy=mx.Accuracy(acc), rounding=MODES[mode])
        assert st == mx.OK
        want = np.stack([c[2] for c in cases])
        meta = np.stack([c[3] for c in cases])
        assert np.array_equal(sel["degree"], meta[:, 0]), (n, acc)
        assert np.array_equal(sel["s"], meta[:, 1]), (n, acc)
        assert np.array_equal(sel["norm_in"], [c[4] for c in cases]), (n, acc)
        if mode == "reference":
            assert np.array_equal(bits(out), bits(want)), (n, acc)
        else:
            tol = 50 * n * U53
            err = rel_fro(out, want)
            if mode == "fast":
                # FMA/DMMA rounding alone: the tolerance band is only promised
                # where AUTO would not switch to reference rounding
                keep = meta[:, 1] < exact_s_min(n)
                err = err[keep] if keep.any() else np.zeros(1)
            assert err.max() <= tol, (n, acc, err.max(), tol)


def exact_s_min(n):
    """AUTO policy threshold (capi.cu exact_s_min)."""
    return 0 if n < 8 else 3 + int(np.floor(np.log2(n)))


def test_drop_in_expm_kats(cuda):
    pi = 3.141592653589793
    r = mx.expm(np.array([[0.0, pi], [-pi, 0.0]]))
    assert (r.degree, r.s, r.cost_thirds, r.norm_in) == (18, 2, 21, pi)
    assert np.abs(r.result + np.eye(2)).sum(axis=0).max() <= 1e-12
    r = mx.expm(np.zeros((4, 4)))
    assert np.array_equal(r.result, np.eye(4)) and (r.degree, r.s) == (1, 0)
    r = mx.expm(np.array([[0.0, 1.0], [-1.0, 0.0]]))
    assert (r.degree, r.s, r.cost_thirds, r.norm_in) == (18, 0, 15, 1.0)
    bad = np.zeros((2, 2))
    bad[0, 1] = np.inf
    with pytest.raises(ValueError, match="non-finite matrix entry"):
        mx.expm(bad)
    huge = np.full((3, 3), 1e308)
    with pytest.raises(ValueError, match="norm must be finite"):
        mx.expm(huge)
    # a single-precision target picks a cheaper scheme (test_expm.cpp:175-186)
    r = mx.expm(np.array([[0.3, 0.1], [0.0, 0.2]]), mx.Accuracy.Single)
    assert r.degree == 8
    assert mx.expm(np.array([[0.3, 0.1], [0.0, 0.2]])).degree == 18


@pytest.fixture(scope="module")
def cfg2(oracle):
    a = workloads.generate("cfg2")
    r = oracle.expm_batch(a, accuracy=1)
    return a, r


@pytest.mark.parametrize("mode", ["reference", "auto", "fast"])
def test_cfg2_full_batch(cuda, cfg2, mode):
    a, ref = cfg2
    out, sel, st = mx.expm_batched_host(a, rounding=MODES[mode])
    assert st == mx.OK
    assert np.array_equal(sel["degree"], ref.degree)
    assert np.array_equal(sel["s"], ref.s)
    assert np.array_equal(bits(sel["norm_in"]), bits(ref.norm_in))
    cost = 3 * (np.vectorize(mx.products_of_degree)(sel["degree"]) + sel["s"])
    assert np.array_equal(cost, ref.cost_thirds)
    err = rel_fro(out, ref.out)
    tol = 50 * 8 * U53
    if mode == "reference":
        assert np.array_equal(bits(out), bits(ref.out))
    elif mode == "auto":
        assert err.max() <= tol, err.max()
    else:
        # FMA/DMMA rounding: outside the band only where >= 6 squarings amplify it
        assert (err[ref.s < 6] <= tol).all(), err[ref.s < 6].max()
    print(f"cfg2 {mode}: max rel err {err.max():.3e} (tol {tol:.3e}), "
          f"over tol: {(err > tol).sum()}")


def test_device_api_and_determinism(cuda, cfg2):
    import torch
    a, ref = cfg2
    da = torch.from_numpy(a[:50000]).to(cuda)
    o1 = torch.empty_like(da)
    o2 = torch.empty_like(da)
    sel = torch.empty(50000 * 16, dtype=torch.uint8, device=cuda)
    mx.expm_batched(da, o1, sel)
    mx.expm_batched(da, o2)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    s = sel.cpu().numpy().view(mx.SELECTION_DTYPE)
    assert np.array_equal(s["degree"], ref.degree[:50000])
    # sharding invariance: a shard computes exactly the rows of the full batch
    o3 = torch.empty_like(da[1234:5678])
    mx.expm_batched(da[1234:5678].contiguous(), o3)
    torch.cuda.synchronize()
    assert torch.equal(o3, o1[1234:5678])


def test_edge_cases(cuda, oracle):
    rng = np.random.default_rng(7)
    a = rng.uniform(-1, 1, (6, 8, 8))
    a[1, 3, 4] = np.nan
    a[3, 0, 0] = -np.inf
    a[4] = 1e308                      # finite entries, overflowing norm
    a[5] = 0.0
    out, sel, st = mx.expm_batched_host(a, rounding=mx.ROUND_REFERENCE, raise_on_error=False)
    assert st == mx.ERR_NONFINITE
    assert list(sel["status"]) == [0, 1, 0, 1, 2, 0]
    assert np.isnan(out[1]).all() and np.isnan(out[3]).all() and np.isnan(out[4]).all()
    ref = oracle.expm_batch(a[[0, 2, 5]])
    assert np.array_equal(bits(out[[0, 2, 5]]), bits(ref.out))
    # empty batch
    o, s, st = mx.expm_batched_host(np.zeros((0, 8, 8)))
    assert st == mx.OK and o.shape == (0, 8, 8)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 9, 13, 16, 17, 24, 31, 32, 33, 48, 64])
def test_padded_sizes_bitwise(cuda, oracle, n):
    rng = np.random.default_rng(n)
    norms = np.array([1e-17, 1e-9, 1e-4, 0.03, 0.2, 0.9, 3.0, 60.0])
    a = rng.uniform(-1, 1, (len(norms), n, n))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    ref = oracle.expm_batch(a)
    out, sel, st = mx.expm_batched_host(a, rounding=mx.ROUND_REFERENCE)
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    assert np.array_equal(bits(out), bits(ref.out))
    out, sel, st = mx.expm_batched_host(a, rounding=mx.ROUND_FAST)
    assert rel_fro(out, ref.out).max() <= 50 * n * U53


def test_launch_counter_moves(cuda):
    before = mx.launch_count()
    mx.expm_batched_host(np.zeros((4, 8, 8)))
    assert mx.launch_count() > before


# ---- fp32 path (BASELINE cfg3): FFMA arithmetic vs the double reference ----
U24 = 2.0 ** -24


def test_cfg3_golden_slice(cuda, golden):
    g = golden("cfg_slices.npz")
    a = g["cfg3_a"]
    out, sel, st = mx.expm_batched_host(a, accuracy=mx.Accuracy.Single)
    assert st == mx.OK and out.dtype == np.float32
    assert np.array_equal(sel["degree"], g["cfg3_degree"])
    assert np.array_equal(sel["s"], g["cfg3_s"])
    assert np.array_equal(sel["norm_in"], g["cfg3_norm"])
    assert rel_fro(out, g["cfg3_out"]).max() <= 50 * 32 * U24


@pytest.fixture(scope="module")
def cfg3(oracle):
    a = workloads.generate("cfg3")
    r = oracle.expm_batch(a, accuracy=0)
    return a, r


def test_cfg3_full_batch(cuda, cfg3):
    a, ref = cfg3
    out, sel, st = mx.expm_batched_host(a, accuracy=mx.Accuracy.Single)
    assert st == mx.OK
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    assert np.array_equal(sel["norm_in"], ref.norm_in)
    err = rel_fro(out, ref.out)
    tol = 50 * 32 * U24
    assert err.max() <= tol, err.max()
    # orthogonality of e^A for the skew-symmetric half: ||X^T X - I||_F
    skew = workloads.skew_mask("cfg3", 0, a.shape[0])
    x = out[skew].astype(np.float64)
    defect = np.linalg.norm(np.einsum("bki,bkj->bij", x, x) - np.eye(32), axis=(1, 2))
    print(f"cfg3: max rel err {err.max():.3e} (tol {tol:.3e}); skew defect median "
          f"{np.median(defect):.2e} max {defect.max():.2e}")
    assert defect.max() <= tol


@pytest.mark.parametrize("n", [1, 3, 8, 13, 16, 24, 32, 40, 64])
def test_fp32_padded_sizes(cuda, oracle, n):
    rng = np.random.default_rng(100 + n)
    norms = np.array([1e-8, 1e-3, 0.04, 0.5, 1.2, 2.9, 12.0, 40.0])
    a = rng.standard_normal((len(norms), n, n))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    a = a.astype(np.float32)
    ref = oracle.expm_batch(a, accuracy=0)
    out, sel, st = mx.expm_batched_host(a, accuracy=mx.Accuracy.Single)
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    assert rel_fro(out, ref.out).max() <= 50 * n * U24


def test_fp32_non_finite(cuda):
    a = np.zeros((3, 32, 32), np.float32)
    a[1, 5, 5] = np.inf
    out, sel, st = mx.expm_batched_host(a, accuracy=mx.Accuracy.Single, raise_on_error=False)
    assert st == mx.ERR_NONFINITE and list(sel["status"]) == [0, 1, 0]
    assert np.array_equal(out[0], np.eye(32, dtype=np.float32))


@pytest.mark.parametrize("mode", ["reference", "auto", "fast"])
def test_cfg1_cluster_path(cuda, oracle, mode):
    """cfg1 (one 64x64 matrix) runs on the 4-CTA cluster kernel
    (expm_cluster.cuh): REFERENCE bit-identical, AUTO/FAST within 50 n u."""
    a = workloads.generate("cfg1", 0, 1)
    ref = oracle.expm_batch(a)
    out, sel, st = mx.expm_batched_host(a, rounding=MODES[mode])
    assert st == mx.OK and (sel["degree"][0], sel["s"][0]) == (ref.degree[0], ref.s[0])
    if mode == "reference":
        assert np.array_equal(bits(out), bits(ref.out))
    else:
        assert rel_fro(out, ref.out).max() <= 50 * 64 * U53


@pytest.mark.parametrize("batch", [3, 74, 75, 150])
def test_cluster_and_cta_paths_agree(cuda, oracle, batch):
    """np = 64 batches up to 2 * SMs / 4 use the cluster kernel, larger ones
    the one-CTA kernel; both match the reference bit for bit in REFERENCE
    rounding, across every degree and s, with n = 50 padded to 64."""
    rng = np.random.default_rng(batch)
    norms = 10.0 ** rng.uniform(-17, 2.5, batch)
    a = rng.standard_normal((batch, 50, 50))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    a[batch // 2, 3, 4] = np.inf
    ref = oracle.expm_batch(a)
    out, sel, st = mx.expm_batched_host(a, rounding=mx.ROUND_REFERENCE, raise_on_error=False)
    assert st == mx.ERR_NONFINITE and sel["status"][batch // 2] == mx.ERR_NONFINITE
    ok = sel["status"] == 0
    assert np.array_equal(sel["degree"][ok], ref.degree[ok]) and np.array_equal(sel["s"][ok], ref.s[ok])
    assert np.array_equal(bits(out[ok]), bits(ref.out[ok]))
    assert np.isnan(out[batch // 2]).all()
    out_ps, sel_ps, _ = mx.expm_batched_host(a, rounding=mx.ROUND_REFERENCE, family=mx.Family.TaylorPS,
                                             raise_on_error=False)
    ref_ps = oracle.expm_batch(a, family=1)
    assert np.array_equal(bits(out_ps[ok]), bits(ref_ps.out[ok]))


@pytest.mark.parametrize("family", [mx.Family.TaylorNew, mx.Family.PadeDiagonal])
def test_graph_capture_and_replay(cuda, oracle, family):
    """A captured mexp_expm_batched launch (the 8x8 kernels hand out work
    through a device ticket) gives the same bits on every replay of the graph."""
    import torch
    a_np = workloads.generate("cfg2", 500, 20000)
    a = torch.from_numpy(a_np).cuda()
    out = torch.empty_like(a)
    sel = torch.empty(a.shape[0] * 16, dtype=torch.uint8, device="cuda")
    mx.expm_batched(a, out, sel, rounding=mx.ROUND_REFERENCE, family=family)  # warm
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        mx.expm_batched(a, out, sel, rounding=mx.ROUND_REFERENCE, family=family,
                        stream=torch.cuda.current_stream())
    ref = oracle.expm_batch(a_np, family=int(family))
    for _ in range(3):
        out.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert np.array_equal(bits(out.cpu().numpy()), bits(ref.out))


@pytest.mark.parametrize("n", [8, 13, 50, 64])
@pytest.mark.parametrize("kind", ["pinned", "pageable"])
def test_small_call_path(cuda, oracle, n, kind):
    """Host calls up to MEXP_SMALL_CALL_KB run on one stream with the kernels
    reading/writing host memory (pinned caller buffers in place, pageable ones
    through pinned staging): same bits as the device API and the reference,
    and the first non-finite matrix reported."""
    import torch
    rng = np.random.default_rng(7 + n)
    norms = np.array([1e-9, 0.02, 0.7, 1.5, 9.0])
    a = rng.standard_normal((len(norms), n, n))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    ref = oracle.expm_batch(a)
    if kind == "pinned":
        ha = torch.from_numpy(a).pin_memory()
        ho = torch.empty_like(ha).pin_memory()
        sel_out = torch.empty(16 * len(a), dtype=torch.uint8).pin_memory()
        out, sel, st = mx.expm_batched_host(ha, ho, rounding=mx.ROUND_REFERENCE, sel_out=sel_out)
        out = out.numpy()
    else:
        out, sel, st = mx.expm_batched_host(a, rounding=mx.ROUND_REFERENCE)
    assert st == mx.OK
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    assert np.array_equal(bits(out), bits(ref.out))
    d = torch.from_numpy(a).cuda()
    od = torch.empty_like(d)
    mx.expm_batched(d, od, rounding=mx.ROUND_REFERENCE)
    assert np.array_equal(bits(out), bits(od.cpu().numpy()))
    bad = a.copy()
    bad[3, 0, n - 1] = np.nan
    _, sel, st = mx.expm_batched_host(bad, raise_on_error=False)
    assert st == mx.ERR_NONFINITE and list(sel["status"]) == [0, 0, 0, 1, 0]


@pytest.mark.parametrize("family", [mx.Family.TaylorPS, mx.Family.PadeDiagonal])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_small_call_path_families_and_fp32(cuda, family, dtype):
    """The small-call path with the other families and fp32 storage (the fp32
    Pade route pads into fp64 device buffers straight from host memory): same
    results and records as the device API."""
    import torch
    rng = np.random.default_rng(11)
    n = 24
    norms = np.array([1e-6, 0.3, 2.0, 11.0])
    a = rng.standard_normal((len(norms), n, n))
    a = (a * (norms / workloads.one_norm_batched(a))[:, None, None]).astype(dtype)
    acc = mx.Accuracy.Single if dtype == np.float32 else mx.Accuracy.Double
    out, sel, st = mx.expm_batched_host(a, accuracy=acc, family=family)
    assert st == mx.OK
    d = torch.from_numpy(a).cuda()
    od = torch.empty_like(d)
    sd = torch.empty(16 * len(a), dtype=torch.uint8, device="cuda")
    mx.expm_batched(d, od, sd, accuracy=acc, family=family)
    torch.cuda.synchronize()
    assert np.array_equal(out.view(np.uint8), od.cpu().numpy().view(np.uint8))
    assert np.array_equal(sel.view(np.uint8), sd.cpu().numpy()[: 16 * len(a)])
