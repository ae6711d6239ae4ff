"""Per-call latency of small host calls (mexp_expm_batched_host / mexp_expm).

    python tools/small_call_probe.py        (MEXP_SMALL_CALL_KB=0: the copy pipeline)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1710_10989_b200 as mx  # noqa: E402
from paper_1710_10989_b200 import workloads  # noqa: E402


def per_call_us(fn, iters=300):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    return (time.perf_counter() - t0) / iters * 1e6


def main():
    res = {"small_call_kb": os.environ.get("MEXP_SMALL_CALL_KB", "default")}
    a1 = workloads.generate("cfg1", 0, 1)
    p1 = torch.from_numpy(a1).pin_memory()
    o1 = torch.empty_like(p1).pin_memory()
    res["cfg1_pinned_us"] = per_call_us(lambda: mx.expm_batched_host(p1, o1))
    res["cfg1_numpy_us"] = per_call_us(lambda: mx.expm_batched_host(a1))
    res["cfg1_dropin_expm_us"] = per_call_us(lambda: mx.expm(a1[0]))
    a8 = workloads.generate("cfg2", 0, 1024)
    p8 = torch.from_numpy(a8).pin_memory()
    o8 = torch.empty_like(p8).pin_memory()
    res["n8x1024_pinned_us"] = per_call_us(lambda: mx.expm_batched_host(p8, o8))
    res["n8x1_numpy_us"] = per_call_us(lambda: mx.expm_batched_host(a8[:1]))
    # parity of the path against the device API on the same inputs
    o, sel, st = mx.expm_batched_host(a1)
    d = torch.from_numpy(a1).cuda()
    od = torch.empty_like(d)
    mx.expm_batched(d, od)
    res["cfg1_bitwise_equal_to_device_call"] = bool(np.array_equal(o, od.cpu().numpy()))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
