"""Time the 8x8 fp64 kernel per (degree, s) class: 262,144 matrices all of one
class, CUDA events around mexp_expm_batched, FAST and REFERENCE rounding.
Splits the per-matrix overhead from the marginal cost of a product / squaring.

    [MEXP_N8_VARIANT=v] python tools/n8_classes.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1710_10989_b200 as mx  # noqa: E402

B = 262144
rng = np.random.default_rng(0)
base = rng.uniform(-1, 1, (B, 8, 8))
norms = np.abs(base).sum(axis=1).max(axis=1)
SMSP = 148 * 4
for mode, rounding in [("fast", mx.ROUND_FAST), ("reference", mx.ROUND_REFERENCE)]:
    rows = []
    for label, target, prods in [("deg1", 1e-17, 0), ("deg2", 1e-9, 1), ("deg4", 1e-5, 2), ("deg8", 0.01, 3),
                                 ("deg12", 0.2, 4), ("deg18 s0", 0.8, 5), ("deg18 s1", 2.0, 6),
                                 ("deg18 s2", 4.0, 7), ("deg18 s4", 16.0, 9), ("deg18 s8", 256.0, 13)]:
        a = torch.from_numpy(base * (target / norms)[:, None, None]).cuda()
        out = torch.empty_like(a)
        sel = torch.empty(B * 16, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            mx.expm_batched(a, out, sel, rounding=rounding)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            mx.expm_batched(a, out, sel, rounding=rounding)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 50.0
        s = sel.cpu().numpy().view(mx.SELECTION_DTYPE)
        cyc = us * 1e-6 * 1.965e9 / (B / SMSP)
        rows.append((label, prods, us, cyc))
        print(f"{mode:9s} {label:10s} degree {s['degree'][0]:2d} s {s['s'].min()}-{s['s'].max()} "
              f"products {prods:2d}: {us:7.1f} us = {cyc:6.1f} SMSP cycles/matrix", flush=True)
    sq = (rows[-1][3] - rows[-3][3]) / 6.0
    print(f"{mode}: marginal squaring {sq:.1f} SMSP cycles (2 DMMAs = 32 pipe cycles in fast rounding)")
