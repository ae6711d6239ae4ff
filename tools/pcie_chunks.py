"""PCIe behaviour of chunked copies (cfg2's 268 MB each way): whole-buffer
H2D+D2H concurrently vs the same bytes in chunks, with and without the
pipeline's H2D -> D2H dependency."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1710_10989_b200 import workloads  # noqa: E402

a = torch.from_numpy(workloads.generate("cfg2")).pin_memory()
o = torch.empty_like(a).pin_memory()
d_in = torch.empty_like(a, device="cuda")
d_out = torch.empty_like(a, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
        torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def whole():
    with torch.cuda.stream(s1):
        d_in.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2):
        o.copy_(d_out, non_blocking=True)


res["whole_concurrent_ms"] = timed(whole)
B = a.shape[0]
for mb in (4, 16, 64):
    ch = (mb << 20) // 512

    def chunked(dep):
        evs = []
        for c0 in range(0, B, ch):
            with torch.cuda.stream(s1):
                d_in[c0:c0 + ch].copy_(a[c0:c0 + ch], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s1)
            with torch.cuda.stream(s2):
                if dep:
                    s2.wait_event(e)
                o[c0:c0 + ch].copy_(d_out[c0:c0 + ch], non_blocking=True)
    res[f"chunked_{mb}MB_nodep_ms"] = timed(lambda: chunked(False))
    res[f"chunked_{mb}MB_dep_ms"] = timed(lambda: chunked(True))
print(json.dumps(res))
