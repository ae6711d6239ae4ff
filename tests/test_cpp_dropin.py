"""The C++ drop-in (include/mexp/*.hpp over libmexp_b200.so) against the
reference's own known-answer tests, re-expressed in tests/cpp/dropin_kats.cpp."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "dropin_kats")


def build():
    subprocess.run(["make", "-C", ROOT, "tests/cpp/dropin_kats"], check=True,
                   capture_output=True)


def test_dropin_builds_and_refuses_without_device():
    import torch
    build()
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: the device run covers it")
    r = subprocess.run([BIN, "--no-device"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_dropin_kats_on_device(cuda):
    build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
