"""Run the 8x8 kernel on 262,144 matrices of one class (all the same 1-norm), for ncu.

    python tools/profile_class.py NORM [fast|auto|reference] [iters]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1710_10989_b200 as mx  # noqa: E402

target = float(sys.argv[1])
mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
rounding = {"auto": mx.ROUND_AUTO, "reference": mx.ROUND_REFERENCE, "fast": mx.ROUND_FAST}[mode]
B = 262144
rng = np.random.default_rng(0)
base = rng.uniform(-1, 1, (B, 8, 8))
norms = np.abs(base).sum(axis=1).max(axis=1)
a = torch.from_numpy(base * (target / norms)[:, None, None]).cuda()
out = torch.empty_like(a)
sel = torch.empty(B * 16, dtype=torch.uint8, device="cuda")
for _ in range(iters):
    mx.expm_batched(a, out, sel, rounding=rounding)
torch.cuda.synchronize()
print("ok")
