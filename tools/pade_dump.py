"""Dump Pade large-n results (for bitwise comparisons between library builds).

    python tools/pade_dump.py out.npz
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1710_10989_b200 as mx  # noqa: E402
from paper_1710_10989_b200 import workloads  # noqa: E402

res = {}
for n in (130, 500, 600):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((3, n, n))
    a *= (np.array([0.4, 5.0, 40.0]) / workloads.one_norm_batched(a))[:, None, None]
    out, sel, st = mx.expm_batched_host(a, family=mx.Family.PadeDiagonal)
    res[f"o{n}"] = out
np.savez(sys.argv[1], **res)
