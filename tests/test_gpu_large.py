"""GPU parity of the large-n path (n > 64: batched FP64 DMMA GEMMs with fused
epilogues) against the oracle: (m, s) and norm_in bit-exact, e^A within
relative Frobenius 50*n*u (BASELINE.json north_star)."""
import numpy as np
import pytest

import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads

pytestmark = pytest.mark.gpu
U53 = 2.0 ** -53


def rel_fro(got, want):
    g = got.reshape(got.shape[0], -1)
    w = want.reshape(want.shape[0], -1)
    return np.linalg.norm(g - w, axis=1) / np.linalg.norm(w, axis=1)


@pytest.mark.parametrize("n", [65, 96, 128, 130, 200, 256])
def test_large_n_every_degree(cuda, oracle, n):
    rng = np.random.default_rng(1000 + n)
    # norms hitting degrees 1, 2, 4, 8, 12, 18 and s = 0..7
    norms = np.array([1e-17, 1e-9, 1e-4, 0.03, 0.2, 0.9, 2.0, 7.0, 30.0, 100.0])
    a = rng.uniform(-1, 1, (len(norms), n, n))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    ref = oracle.expm_batch(a)
    assert set(ref.degree) == {1, 2, 4, 8, 12, 18}
    out, sel, st = mx.expm_batched_host(a)
    assert st == mx.OK
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    assert np.array_equal(sel["norm_in"], ref.norm_in)
    err = rel_fro(out, ref.out)
    assert err.max() <= 50 * n * U53, err


def test_large_n_errors_and_reference_rounding(cuda):
    a = np.zeros((3, 100, 100))
    a[1, 7, 9] = np.nan
    a[2] = 1e308
    out, sel, st = mx.expm_batched_host(a, raise_on_error=False)
    assert list(sel["status"]) == [0, 1, 2]
    assert np.array_equal(out[0], np.eye(100))
    assert np.isnan(out[1]).all() and np.isnan(out[2]).all()
    out_r, sel_r, _ = mx.expm_batched_host(a, rounding=mx.ROUND_REFERENCE, raise_on_error=False)
    assert list(sel_r["status"]) == [0, 1, 2] and np.array_equal(out_r[0], np.eye(100))


def test_cfg4_subset(cuda, oracle):
    """16 matrices of cfg4 (512 x 512, N(0,1/N), ||A||_1 log-U[0.5, 20])."""
    a = workloads.generate("cfg4", 0, 16)
    ref = oracle.expm_batch(a)
    out, sel, st = mx.expm_batched_host(a)
    assert st == mx.OK
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    err = rel_fro(out, ref.out)
    tol = workloads.CONFIGS["cfg4"].tolerance
    print(f"cfg4[0:16]: s = {sorted(set(ref.s))}, max rel err {err.max():.3e} (tol {tol:.3e})")
    assert err.max() <= tol


def test_cfg4_full_batch_properties(cuda):
    """All 1,024 cfg4 matrices at full size, through size-independent
    properties: e^A e^-A = I within 50 n u of ||e^A|| ||e^-A|| (the GEMM
    check in fp64 on the device), (m, s) of -A equal to those of A (same
    1-norm), and the selection records bit-equal to the host's mexp_select
    on the same norms."""
    import torch
    a = torch.from_numpy(workloads.generate("cfg4")).cuda()
    B, n, _ = a.shape
    e1, e2 = torch.empty_like(a), torch.empty_like(a)
    s1 = torch.empty(16 * B, dtype=torch.uint8, device="cuda")
    s2 = torch.empty_like(s1)
    mx.expm_batched(a, e1, s1)
    mx.expm_batched(-a, e2, s2)
    torch.cuda.synchronize()
    r1 = s1.cpu().numpy().view(mx.SELECTION_DTYPE)
    r2 = s2.cpu().numpy().view(mx.SELECTION_DTYPE)
    assert (r1["status"] == 0).all() and (r2["status"] == 0).all()
    assert np.array_equal(r1.view(np.uint8), r2.view(np.uint8))
    table = mx.selection_table(mx.Family.TaylorNew, mx.Accuracy.Double)
    for i in range(0, B, 97):
        assert mx.select(float(r1["norm_in"][i]), table) == (r1["degree"][i], r1["s"][i])
    tol = workloads.CONFIGS["cfg4"].tolerance
    eye = torch.eye(n, dtype=a.dtype, device="cuda")
    worst = 0.0
    for c in range(0, B, 64):
        p = torch.bmm(e1[c:c + 64], e2[c:c + 64]) - eye
        rel = torch.linalg.matrix_norm(p) / (torch.linalg.matrix_norm(e1[c:c + 64]) *
                                              torch.linalg.matrix_norm(e2[c:c + 64]))
        worst = max(worst, float(rel.max()))
    print(f"cfg4 full batch: max ||e^A e^-A - I|| / (||e^A|| ||e^-A||) = {worst:.3e} (tol {tol:.3e})")
    assert worst <= tol


def test_cfg5_full_size_inverse_property(cuda):
    """The whole 8192 x 8192 cfg5 matrix: e^A e^-A = I within 50 n u of
    ||e^A|| ||e^-A|| (cuBLAS fp64 GEMM as the checker), same (m, s) for -A."""
    import torch
    a = torch.from_numpy(workloads.generate("cfg5")).cuda()
    e1, e2 = torch.empty_like(a), torch.empty_like(a)
    s1 = torch.empty(16, dtype=torch.uint8, device="cuda")
    s2 = torch.empty_like(s1)
    mx.expm_batched(a, e1, s1)
    mx.expm_batched(-a, e2, s2)
    torch.cuda.synchronize()
    r1 = s1.cpu().numpy().view(mx.SELECTION_DTYPE)
    r2 = s2.cpu().numpy().view(mx.SELECTION_DTYPE)
    assert (r1["degree"][0], r1["s"][0]) == (r2["degree"][0], r2["s"][0]) == (18, 5)
    p = torch.matmul(e1[0], e2[0])
    p.diagonal().sub_(1.0)
    rel = float(torch.linalg.matrix_norm(p) / (torch.linalg.matrix_norm(e1[0]) * torch.linalg.matrix_norm(e2[0])))
    tol = workloads.CONFIGS["cfg5"].tolerance
    print(f"cfg5: ||e^A e^-A - I|| / (||e^A|| ||e^-A||) = {rel:.3e} (tol {tol:.3e})")
    assert rel <= tol


def test_cfg5_leading_block_and_structure(cuda, oracle):
    """cfg5 (8192^2, upper triangular + U(-5,0) diagonal, ||A||_1 = 30) is
    too large for the CPU oracle; checked through size-independent properties:
    the leading 256 x 256 block of e^A equals T_m(2^-s A_256)^(2^s) with the
    full matrix's (m, s) (exact identity for triangular A; oracle restated
    with the forced selection), the strictly lower part is exactly zero and
    the diagonal is exp(a_ii) to working accuracy."""
    import torch
    a = workloads.generate("cfg5")
    ref_norm = workloads.one_norm_batched(a)[0]
    da = torch.from_numpy(a).to(cuda)
    out = torch.empty_like(da)
    sel = torch.empty(16, dtype=torch.uint8, device=cuda)
    mx.expm_batched(da, out, sel)
    torch.cuda.synchronize()
    s = sel.cpu().numpy().view(mx.SELECTION_DTYPE)[0]
    assert s["norm_in"] == ref_norm and s["status"] == 0
    assert (s["degree"], s["s"]) == (18, 5)
    k = 256
    blk = out[0, :k, :k].cpu().numpy()
    want = oracle.expm_forced(a[0, :k, :k].copy(), int(s["degree"]), int(s["s"]))
    err = np.linalg.norm(blk - want) / np.linalg.norm(want)
    tol = workloads.CONFIGS["cfg5"].tolerance
    print(f"cfg5 leading {k}x{k} block: rel err {err:.3e} (tol {tol:.3e})")
    assert err <= tol
    assert bool((torch.tril(out[0], -1) == 0).all())
    diag = torch.diagonal(out[0]).cpu().numpy()
    assert np.max(np.abs(diag - np.exp(np.diag(a[0]))) / np.exp(np.diag(a[0]))) <= 1e-12


def test_large_n_fp32_storage(cuda, oracle):
    """fp32 storage beyond n = 64: the fp64 DMMA engine on the widened values
    (never TF32), e^A rounded once; (m, s) from the fp64 norm of the floats."""
    rng = np.random.default_rng(64)
    n = 100
    norms = np.array([1e-6, 0.3, 2.5, 40.0])
    a = rng.standard_normal((len(norms), n, n))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    a = a.astype(np.float32)
    ref = oracle.expm_batch(a, accuracy=0)
    out, sel, st = mx.expm_batched_host(a, accuracy=mx.Accuracy.Single)
    assert st == mx.OK and out.dtype == np.float32
    assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
    assert rel_fro(out.astype(np.float64), ref.out).max() <= 50 * n * 2.0 ** -24


def test_large_n_batch_beyond_grid_y(cuda, oracle):
    """More than 65,535 matrices of n > 64: every per-matrix launch of the
    large-n path is sliced along the grid's y limit."""
    n, batch = 65, 66000
    a = np.zeros((batch, n, n))
    rng = np.random.default_rng(65)
    idx = np.array([0, 1, 65534, 65535, 65536, batch - 1])
    for k, i in enumerate(idx):
        m = rng.uniform(-1, 1, (n, n))
        a[i] = m * (10.0 ** (k - 3) / np.abs(m).sum(axis=0).max())
    a[123, 4, 4] = np.nan
    out, sel, st = mx.expm_batched_host(a, raise_on_error=False)
    assert st == mx.ERR_NONFINITE and sel["status"][123] == mx.ERR_NONFINITE
    assert np.isnan(out[123]).all()
    ref = oracle.expm_batch(a[idx])
    assert np.array_equal(sel["degree"][idx], ref.degree) and np.array_equal(sel["s"][idx], ref.s)
    assert rel_fro(out[idx], ref.out).max() <= 50 * n * U53
    zero = np.setdiff1d(np.arange(batch), np.append(idx, 123))[::997]
    assert all(np.array_equal(out[i], np.eye(n)) for i in zero)


@pytest.mark.parametrize("n", [65, 96, 130, 200])
def test_large_n_reference_rounding_bitwise(cuda, oracle, n):
    """REFERENCE rounding beyond n = 64: k-ordered DMUL+DADD products over the
    true n (never a padded term) and literal lincombs -> e^A bit-identical to
    the reference for every degree and s, both Taylor families."""
    rng = np.random.default_rng(5000 + n)
    norms = np.array([1e-17, 1e-9, 1e-4, 5e-3, 0.03, 0.2, 0.9, 2.0, 7.0, 30.0, 100.0])
    a = rng.uniform(-1, 1, (len(norms), n, n))
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    for family in (0, 1):
        ref = oracle.expm_batch(a, family=family)
        out, sel, st = mx.expm_batched_host(a, rounding=mx.ROUND_REFERENCE, family=mx.Family(family))
        assert st == mx.OK
        assert np.array_equal(sel["degree"], ref.degree) and np.array_equal(sel["s"], ref.s)
        assert np.array_equal(out.view(np.uint64), ref.out.view(np.uint64)), (n, family)


def test_large_n_reference_rounding_cfg4_slice(cuda, oracle):
    a = workloads.generate("cfg4", 0, 3)
    ref = oracle.expm_batch(a)
    out, sel, st = mx.expm_batched_host(a, rounding=mx.ROUND_REFERENCE)
    assert st == mx.OK and np.array_equal(sel["s"], ref.s)
    assert np.array_equal(out.view(np.uint64), ref.out.view(np.uint64))


def test_large_n_reference_rounding_refuses_pade(cuda):
    a = np.zeros((1, 70, 70))
    with pytest.raises(ValueError, match="unsupported"):
        mx.expm_batched_host(a, rounding=mx.ROUND_REFERENCE, family=mx.Family.PadeDiagonal)


_CHUNKED_SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads
rng = np.random.default_rng(77)
n = 130
norms = np.exp(rng.uniform(np.log(1e-6), np.log(60.0), 23))
a = rng.standard_normal((23, n, n))
a *= (norms / workloads.one_norm_batched(a))[:, None, None]
a[9, 3, 4] = np.nan
a[17, 0, 0] = np.inf
out, sel, st = mx.expm_batched_host(a, raise_on_error=False)
d = torch.from_numpy(a).cuda()
od = torch.empty_like(d)
sd = torch.empty(16 * len(a), dtype=torch.uint8, device="cuda")
try:
    mx.expm_batched(d, od, sd)
except Exception:
    pass
torch.cuda.synchronize()
ref_sel = sd.cpu().numpy().view(mx.SELECTION_DTYPE)
ok = [i for i in range(len(a)) if i not in (9, 17)]
assert st == mx.ERR_NONFINITE, st
assert list(np.nonzero(sel["status"])[0]) == [9, 17]
assert np.array_equal(sel["degree"], ref_sel["degree"]) and np.array_equal(sel["s"], ref_sel["s"])
assert np.array_equal(out[ok].view(np.uint64), od.cpu().numpy()[ok].view(np.uint64))
assert np.isnan(out[9]).all() and np.isnan(out[17]).all()
print("chunked ok")
"""


def test_large_n_host_pipeline_many_chunks(cuda):
    """The large-n host pipeline over many chunks (MEXP_HOST_CHUNK_MB_LARGE=1:
    7 matrices of 130^2 per chunk, 4 chunks): selections read back through
    mapped memory and lists uploaded by the copy kernel give the same bits as
    one device call, with non-finite matrices in two different chunks."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MEXP_HOST_CHUNK_MB_LARGE="1")
    r = subprocess.run([sys.executable, "-c", _CHUNKED_SCRIPT, root], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "chunked ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("rounding", [mx.ROUND_FAST, mx.ROUND_AUTO])
def test_prep_free_path_bitwise(cuda, rounding, monkeypatch):
    """Unpadded TaylorNew batches skip the scaled copy of A: the products read
    the caller's A and scale by exact powers of two (A2 = 4^-s AA, A3 = 2^-s
    A2 A, T18's B epilogue reads 2^-s A). Same bits as the scaled-copy path
    (MEXP_LARGE_PREP=1) across every degree and s up to ~6."""
    rng = np.random.default_rng(11)
    n, b = 128, 12
    a = rng.standard_normal((b, n, n)) / np.sqrt(n)
    norms = np.array([1e-5, 3e-3, 0.03, 0.2, 0.6, 1.0, 2.0, 5.0, 12.0, 30.0, 60.0, 0.9])
    a *= (norms / workloads.one_norm_batched(a))[:, None, None]
    out0, sel0, st0 = mx.expm_batched_host(a, rounding=rounding)
    monkeypatch.setenv("MEXP_LARGE_PREP", "1")
    out1, sel1, st1 = mx.expm_batched_host(a, rounding=rounding)
    assert st0 == st1 == mx.OK
    assert set(sel0["degree"].tolist()) >= {4, 8, 12, 18} and sel0["s"].max() >= 5
    assert np.array_equal(sel0.view(np.uint8), sel1.view(np.uint8))
    assert np.array_equal(out0.view(np.uint64), out1.view(np.uint64))
