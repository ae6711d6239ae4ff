"""e2e (host buffers -> e^A on host) timing of cfg2 for one pipeline setting,
taken from MEXP_HOST_STREAMS / MEXP_HOST_CHUNK_MB in the environment.

    MEXP_HOST_STREAMS=4 MEXP_HOST_CHUNK_MB=16 python tools/e2e_sweep.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1710_10989_b200 as mx  # noqa: E402
from paper_1710_10989_b200 import workloads  # noqa: E402


def main():
    a = torch.from_numpy(workloads.generate("cfg2")).pin_memory()
    out = torch.empty_like(a).pin_memory()
    for _ in range(3):
        mx.expm_batched_host(a, out)
    ts = []
    for _ in range(15):
        t0 = time.perf_counter()
        mx.expm_batched_host(a, out)
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * np.median(ts)
    print(f"streams={os.environ.get('MEXP_HOST_STREAMS', '4')} chunk_mb={os.environ.get('MEXP_HOST_CHUNK_MB', '16')} taper_kb={os.environ.get('MEXP_HOST_TAPER_KB', '-')} "
          f"median {ms:.3f} ms best {1e3 * min(ts):.3f} ms -> {a.shape[0] / (ms * 1e-3):.3e} expm/s")


if __name__ == "__main__":
    main()
