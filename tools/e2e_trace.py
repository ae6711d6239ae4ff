"""One traced host call (MEXP_HOST_TRACE=1 prints the chunk timeline) of a config.

    MEXP_HOST_TRACE=1 python tools/e2e_trace.py cfg4
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1710_10989_b200 as mx  # noqa: E402
from paper_1710_10989_b200 import workloads  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
cfg = workloads.CONFIGS[key]
h = torch.from_numpy(workloads.generate(key)).pin_memory()
o = torch.empty_like(h).pin_memory()
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    t0 = time.perf_counter()
    mx.expm_batched_host(h, o, accuracy=mx.Accuracy(cfg.accuracy))
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)
