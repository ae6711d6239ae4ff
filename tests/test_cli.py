"""The `mexp` CLI over the B200 drop-in, checked the
way the reference checks its own CLI (proj/tests/cli_smoke.sh:10-50)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "bin", "mexp")


@pytest.fixture(scope="module")
def cli():
    subprocess.run(["make", "-C", ROOT, "bin/mexp"], check=True, capture_output=True)
    return BIN


def run(cli, *args):
    return subprocess.run([cli, *args], capture_output=True, text=True, timeout=300)


def test_theta_table_layout(cli):
    # cli_smoke.sh:24: '^    18    5  1.09e+00$'
    r = run(cli, "theta", "--family", "taylor", "--u", "double")
    assert r.returncode == 0
    assert "    18    5  1.09e+00" in r.stdout.splitlines()
    r = run(cli, "theta", "--family", "taylor", "--u", "single")
    assert "    18    5  3.01e+00" in r.stdout.splitlines()


def test_bad_input_and_usage_rejected(cli, tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("2\n0 inf\n0 0\n")            # cli_smoke.sh:46-50
    assert run(cli, "exp", "--in", str(bad)).returncode != 0
    assert run(cli, "exp", "--in", str(tmp_path / "missing.txt")).returncode == 1
    assert run(cli, "exp").returncode == 1       # --in required
    assert run(cli, "staircase", "--points", "0").returncode == 1  # bad norm grid
    assert run(cli, "sweep", "--kinds", "nope").returncode == 1
    assert run(cli, "bogus").returncode == 2


@pytest.mark.gpu
def test_exp_rotation_report_and_determinism(cuda, cli, tmp_path, oracle):
    # cli_smoke.sh:10-19: rotation by 1 rad -> 'taylor-new 18 0 5 1', header '2'
    rot = tmp_path / "rot.txt"
    rot.write_text("2\n0 1\n-1 0\n")
    r1 = run(cli, "exp", "--in", str(rot), "--family", "taylor-new", "--u", "double", "--report")
    assert r1.returncode == 0, r1.stderr
    assert r1.stdout.splitlines()[0] == "2"
    assert r1.stderr.split() == ["taylor-new", "18", "0", "5", "1"]
    r2 = run(cli, "exp", "--in", str(rot), "--report")
    assert r2.stdout == r1.stdout                # deterministic
    got = np.array([[float(x) for x in line.split()] for line in r1.stdout.splitlines()[1:]])
    want = oracle.expm_batch(np.array([[[0.0, 1.0], [-1.0, 0.0]]])).out[0]
    # n = 2 < 8: the AUTO policy uses reference rounding -> bit-identical
    assert np.array_equal(got, want)
    # the comparison families run on the device too: r16 for ||A|| = 1, cost 5 + 4/3
    r3 = run(cli, "exp", "--in", str(rot), "--family", "pade", "--report")
    assert r3.returncode == 0, r3.stderr
    assert r3.stderr.split() == ["pade", "16", "0", repr(19 / 3), "1"]
    got = np.array([[float(x) for x in line.split()] for line in r3.stdout.splitlines()[1:]])
    assert np.array_equal(got, oracle.expm_batch(np.array([[[0.0, 1.0], [-1.0, 0.0]]]),
                                                 family=2).out[0])
    r4 = run(cli, "exp", "--in", str(rot), "--family", "ps", "--report")
    assert r4.returncode == 0 and r4.stderr.split()[:3] == ["taylor-ps", "16", "1"]


# ---- staircase / sweep / gallery -------------------
def _ref_lib():
    import ctypes as C
    from oracle.oracle import REF_SO, Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    lib = C.CDLL(REF_SO)
    lib.ref_staircase_csv.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                      C.c_char_p, C.c_int]
    lib.ref_sweep_csv.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                  C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_char_p, C.c_int]
    lib.ref_gallery.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_void_p]
    return lib


def test_staircase_csv_equals_reference(cli):
    """cost_staircase + staircase_csv (bench.cpp:32-57) on the reference's
    default grid and on the Single tables, every family."""
    import ctypes as C
    lib = _ref_lib()
    buf = C.create_string_buffer(1 << 20)
    for fam, name in ((0, "taylor-new"), (1, "taylor-ps"), (2, "pade")):
        for acc, u in ((1, "double"), (0, "single")):
            for lo, hi, pts in ((1e-8, 64.0, 257), (1e-3, 1e3, 33)):
                k = lib.ref_staircase_csv(fam, acc, lo, hi, pts, buf, len(buf))
                r = run(cli, "staircase", "--family", name, "--u", u, "--norm-min", repr(lo),
                        "--norm-max", repr(hi), "--points", str(pts))
                assert r.returncode == 0, r.stderr
                assert r.stdout == buf.value.decode()[:k], (name, u, lo, hi)


def test_gallery_equals_reference():
    """The host gallery (gallery.cpp) reproduces the reference's matrices bit
    for bit, every kind, and refuses a zero matrix the same way."""
    lib = _ref_lib()
    subprocess.run(["make", "-C", ROOT, "tests/cpp/gallery_dump"], check=True, capture_output=True)
    specs = [(k, n, seed, norm) for k in range(9) for n, seed, norm in
             ((1, 0, 1.0), (5, 7, 0.3), (12, 12345678901, 17.5))]
    args = [str(x) if not isinstance(x, float) else repr(x) for sp in specs for x in sp]
    out = subprocess.run([os.path.join(ROOT, "tests", "cpp", "gallery_dump"), *args],
                         capture_output=True, text=True, check=True).stdout.splitlines()
    assert len(out) == len(specs)
    for (k, n, seed, norm), line in zip(specs, out):
        want = np.zeros(n * n)
        st = lib.ref_gallery(k, n, seed, norm, want.ctypes.data)
        if st:
            assert line == "error", (k, n)
            continue
        got = np.array([float.fromhex(t) for t in line.split()])
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (k, n, seed)


@pytest.mark.gpu
@pytest.mark.parametrize("n,u", [(8, "double"), (13, "double"), (16, "single")])
def test_sweep_csv_equals_reference(cuda, cli, n, u):
    """`mexp sweep` (gallery -> reference_expm and every family on the GPU,
    REFERENCE rounding for n <= 64) prints the reference's CSV byte for byte."""
    import ctypes as C
    lib = _ref_lib()
    kinds = np.arange(9, dtype=np.int32)
    fams = np.array([0, 1, 2], dtype=np.int32)
    buf = C.create_string_buffer(1 << 22)
    k = lib.ref_sweep_csv(kinds.ctypes.data, 9, fams.ctypes.data, 3, n, 36, 5, 1 if u == "double" else 0,
                          1e-3, 1e2, buf, len(buf))
    assert k > 0, buf.value
    r = run(cli, "sweep", "--n", str(n), "--count", "36", "--seed", "5", "--u", u)
    assert r.returncode == 0, r.stderr
    assert r.stdout == buf.value.decode()[:k]
