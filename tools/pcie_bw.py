"""Host<->device copy bandwidth on the box (pinned buffers): H2D alone, D2H
alone, and both at once on two streams -- the ceiling of the e2e path."""
import json
import os
import sys

import torch


def main():
    mb = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    n = mb << 20
    h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, fn in [
        ("h2d", lambda: d1.copy_(h1, non_blocking=True)),
        ("d2h", lambda: h2.copy_(d2, non_blocking=True)),
    ]:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name + "_gbs"] = 10 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    res["bidir_total_gbs"] = 20 * n / (time.perf_counter() - t0) / 1e9
    res["mb"] = mb
    print(json.dumps(res))


if __name__ == "__main__":
    main()
