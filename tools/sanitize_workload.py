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
    # one 64x64 (4-CTA cluster kernel), every family at small and large n,
    # reference-rounded large n (exact GEMM), Pade panels on clusters of
    # 2..8 CTAs (n = 130, 500) and per-column steps (n = 600)
    mx.expm_batched_host(workloads.generate("cfg1", 0, 1))
    for fam in (mx.Family.TaylorPS, mx.Family.PadeDiagonal):
        for n in (8, 24, 64, 130):
            norms = np.array([1e-9, 0.2, 3.0, 60.0])
            b = rng.uniform(-1, 1, (4, n, n))
            b *= (norms / workloads.one_norm_batched(b))[:, None, None]
            mx.expm_batched_host(b, family=fam)
    for n in (500, 600):
        b = rng.uniform(-1, 1, (2, n, n))
        b *= (np.array([0.5, 7.0]) / workloads.one_norm_batched(b))[:, None, None]
        mx.expm_batched_host(b, family=mx.Family.PadeDiagonal)
    b = rng.uniform(-1, 1, (3, 100, 100))
    b *= (np.array([0.01, 1.0, 40.0]) / workloads.one_norm_batched(b))[:, None, None]
    mx.expm_batched_host(b, rounding=mx.ROUND_REFERENCE)
    # the multi-device host entry (shards on one device), the dense layer
    # (reference-rounded matmul, lincomb, one_norm, the exact LU) and the
    # captured-graph ticket slots
    import torch
    mx.expm_batched_host_multi(workloads.generate("cfg2", 0, 999), devices=[0, 0, 0])
    for n in (8, 50, 100):
        d = torch.from_numpy(rng.uniform(-1, 1, (3, n, n))).cuda()
        mx.matmul_batched(d, d)
        mx.matmul_batched(d, d, rounding=mx.ROUND_FAST)
        mx.lincomb_batched([1.0, -2.0, 0.5], [d, d, d])
        mx.one_norm_batched(d)
        mx.lu_solve_batched(d + n * torch.eye(n, dtype=d.dtype, device="cuda"), d)
    g = torch.from_numpy(workloads.generate("cfg2", 0, 4096)).cuda()
    o = torch.empty_like(g)
    graph = torch.cuda.CUDAGraph()
    mx.expm_batched(g, o)
    torch.cuda.synchronize()
    with torch.cuda.graph(graph):
        mx.expm_batched(g, o, stream=torch.cuda.current_stream())
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
