"""Small workload touching every kernel family, for compute-sanitizer runs:
8x8 (all rounding modes), padded n, 16/32/64 fp64 groups, fp32 groups,
large-n DMMA GEMM chain with ragged squarings, and per-matrix errors."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1710_10989_b200 as mx  # noqa: E402
from paper_1710_10989_b200 import workloads  # noqa: E402


def main():
    a = workloads.generate("cfg2", 0, 256)
    a[3, 1, 1] = np.nan
    for r in (mx.ROUND_AUTO, mx.ROUND_FAST, mx.ROUND_REFERENCE):
        mx.expm_batched_host(a, rounding=r, raise_on_error=False)
    rng = np.random.default_rng(0)
    for n in (5, 16, 32, 64, 100):
        norms = np.array([1e-9, 0.2, 3.0, 60.0])
        b = rng.uniform(-1, 1, (4, n, n))
        b *= (norms / workloads.one_norm_batched(b))[:, None, None]
        mx.expm_batched_host(b)
        if n <= 64:
            mx.expm_batched_host(b.astype(np.float32), accuracy=mx.Accuracy.Single)
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
