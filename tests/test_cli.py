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
    assert run(cli, "staircase").returncode == 1  # not on the B200 path
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
    assert run(cli, "exp", "--in", str(rot), "--family", "pade").returncode == 1
