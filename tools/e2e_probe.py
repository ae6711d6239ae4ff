"""Break the e2e call (mexp_expm_batched_host) into its parts on the box."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time

import torch

import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads

a = torch.from_numpy(workloads.generate("cfg2")).pin_memory()
o = torch.empty_like(a).pin_memory()
res = {}
for _ in range(3):
    mx.expm_batched_host(a, o)
t0 = time.perf_counter()
for _ in range(20):
    mx.expm_batched_host(a, o)
res["e2e_ms"] = (time.perf_counter() - t0) / 20 * 1e3
# copies alone, same chunking, no kernels
d_in = torch.empty_like(a, device="cuda")
d_out = torch.empty_like(a, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    with torch.cuda.stream(s1):
        d_in.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2):
        o.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
res["h2d_plus_d2h_concurrent_ms"] = (time.perf_counter() - t0) / 20 * 1e3
t0 = time.perf_counter()
for _ in range(20):
    d_in.copy_(a, non_blocking=True)
    torch.cuda.synchronize()
res["h2d_only_ms"] = (time.perf_counter() - t0) / 20 * 1e3
t0 = time.perf_counter()
for _ in range(20):
    o.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
res["d2h_only_ms"] = (time.perf_counter() - t0) / 20 * 1e3
t0 = time.perf_counter()
for _ in range(200):
    mx.expm_batched_host(a[:64], o[:64])
res["tiny_call_overhead_us"] = (time.perf_counter() - t0) / 200 * 1e6
print(json.dumps(res))
