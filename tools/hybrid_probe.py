"""cfg3 probe: the fp32 FFMA kernel vs the fp64 DMMA engine on the same
(promoted) matrices, and both at once on two streams (half the batch each).

    python tools/hybrid_probe.py [iters]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1710_10989_b200 as mx  # noqa: E402
from paper_1710_10989_b200 import workloads  # noqa: E402


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    a32 = torch.from_numpy(workloads.generate("cfg3")).cuda()
    a64 = a32.double()
    o32, o64 = torch.empty_like(a32), torch.empty_like(a64)
    B = a32.shape[0]
    acc = mx.Accuracy.Single
    t32 = timed(lambda: mx.expm_batched(a32, o32, accuracy=acc), iters)
    res = {"fp32_us": t32}
    for name, rnd in (("fast", mx.ROUND_FAST), ("auto", mx.ROUND_AUTO)):
        res[f"fp64_{name}_us"] = timed(lambda: mx.expm_batched(a64, o64, accuracy=acc, rounding=rnd), iters)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for frac in (0.5, 0.6, 0.7):
        h = int(B * frac)

        def both():
            cur = torch.cuda.current_stream()
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            mx.expm_batched(a32[:h], o32[:h], accuracy=acc, stream=s1)
            mx.expm_batched(a64[h:], o64[h:], accuracy=acc, rounding=mx.ROUND_FAST, stream=s2)
            cur.wait_stream(s1)
            cur.wait_stream(s2)
        res[f"both_f32frac{frac}_us"] = timed(both, iters)
    print(res)


if __name__ == "__main__":
    main()
