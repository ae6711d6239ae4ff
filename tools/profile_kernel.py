"""Run the batched expm kernel of one config a few times (for ncu / nsight).

    python tools/profile_kernel.py cfg2 auto [iters] [family]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1710_10989_b200 as mx  # noqa: E402
from paper_1710_10989_b200 import workloads  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    mode = sys.argv[2] if len(sys.argv) > 2 else "auto"
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    family = {"taylor-new": 0, "taylor-ps": 1, "pade": 2}[sys.argv[4] if len(sys.argv) > 4 else "taylor-new"]
    cfg = workloads.CONFIGS[key]
    rounding = {"auto": mx.ROUND_AUTO, "reference": mx.ROUND_REFERENCE, "fast": mx.ROUND_FAST}[mode]
    a = torch.from_numpy(workloads.generate(key)).cuda()
    out = torch.empty_like(a)
    sel = torch.empty(a.shape[0] * 16, dtype=torch.uint8, device="cuda")
    for _ in range(iters):
        mx.expm_batched(a, out, sel, accuracy=mx.Accuracy(cfg.accuracy), rounding=rounding,
                        family=mx.Family(family))
    torch.cuda.synchronize()
    print(f"{key} {mode}: {iters} launches ok")


if __name__ == "__main__":
    main()
