"""Time the 32x32 fp32 path per (degree, s) class: 65,536 matrices all of one
class, CUDA events around mexp_expm_batched (pre-pass + pair kernel).
Fits time = c0 + c1 * products to split per-matrix overhead from product cost.

    python tools/pairs32_classes.py [pairs 0|1]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1710_10989_b200 as mx  # noqa: E402

if len(sys.argv) > 1:
    os.environ["MEXP_F32_PAIRS"] = sys.argv[1]
B = 65536
rng = np.random.default_rng(0)
base = rng.standard_normal((B, 32, 32)).astype(np.float32)
norms = np.abs(base.astype(np.float64)).sum(axis=1).max(axis=1)
rows = []
for label, target, prods in [("deg1", 1e-8, 0), ("deg2", 1e-4, 1), ("deg4", 0.03, 2), ("deg8", 0.3, 3), ("deg12", 1.0, 4), ("deg18 s0", 2.5, 5),
                             ("deg18 s3", 2.5 * 8, 8), ("deg18 s5", 2.5 * 32, 10), ("deg18 s10", 2.5 * 1024, 15)]:
    a = torch.from_numpy((base * (target / norms)[:, None, None]).astype(np.float32)).cuda()
    out = torch.empty_like(a)
    sel = torch.empty(B * 16, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        mx.expm_batched(a, out, sel, accuracy=mx.Accuracy.Single)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        mx.expm_batched(a, out, sel, accuracy=mx.Accuracy.Single)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 100.0
    s = sel.cpu().numpy().view(mx.SELECTION_DTYPE)
    rows.append((label, int(s["degree"][0]), int(s["s"].max()), prods, us))
    print(f"{label:10s} degree {s['degree'][0]:2d} s {s['s'].min()}-{s['s'].max()} products {prods:2d}: "
          f"{us:8.1f} us", flush=True)
P = np.array([r[3] for r in rows], float)
T = np.array([r[4] for r in rows], float)
c1, c0 = np.polyfit(P, T, 1)
print(f"fit: {c0:.1f} us + {c1:.1f} us/product; FFMA-bound product time at 70.4 TF: "
      f"{B * 32768 * 2 / 70.4e12 * 1e6:.1f} us")
