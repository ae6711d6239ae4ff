"""Seeded synthetic inputs for the five BASELINE.json configurations.

There is no public dataset on this path (the paper's MATLAB gallery is not in
the reference and is not reconstructed); these generators ARE the benchmark.
Both the GPU path and the CPU oracle consume the same generated arrays.

Randomness is counter-based so any shard regenerates identically:
``u = splitmix64(splitmix64(splitmix64(seed) ^ tag) ^ (matrix << 32 | element))``,
53-bit uniforms ``(u >> 11) * 2^-53`` exactly as the reference's
``uniform_pm1`` builds them (gallery.cpp:31-33), normals by Box-Muller.
Rescaling multiplies by ``target / one_norm`` in double, with the column sums
taken in the reference's row-ascending order (kernels.cpp:44-53).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def _bits(seed: int, tag: int, matrix: np.ndarray, elem: np.ndarray) -> np.ndarray:
    key = _splitmix(_splitmix(np.asarray([seed], np.uint64)) ^ np.uint64(tag))
    ctr = (matrix.astype(np.uint64) << np.uint64(32)) | elem.astype(np.uint64)
    return _splitmix(key ^ ctr)


def _u53(bits: np.ndarray) -> np.ndarray:
    return (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def uniform01(seed, tag, b0, batch, count, e0=0):
    m = np.arange(b0, b0 + batch, dtype=np.uint64)[:, None]
    e = np.arange(e0, e0 + count, dtype=np.uint64)[None, :]
    return _u53(_bits(seed, tag, m, e))


def uniform_pm1(seed, tag, b0, batch, count, e0=0):
    """U[-1, 1) from 53 bits, the reference's construction (gallery.cpp:31-33)."""
    return 2.0 * uniform01(seed, tag, b0, batch, count, e0) - 1.0


def normal(seed, tag, b0, batch, count, e0=0):
    """iid N(0, 1) by Box-Muller over two independent 53-bit streams."""
    u1 = uniform01(seed, tag, b0, batch, count, e0)
    u2 = uniform01(seed, tag + 1, b0, batch, count, e0)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


def one_norm_batched(a: np.ndarray) -> np.ndarray:
    """Exact 1-norm per matrix, rows summed in ascending order from 0.0."""
    a = a.astype(np.float64, copy=False)
    s = np.zeros((a.shape[0], a.shape[2]), np.float64)
    for i in range(a.shape[1]):
        s += np.abs(a[:, i, :])
    return s.max(axis=1)


def log_uniform(seed, tag, b0, batch, lo, hi):
    u = uniform01(seed, tag, b0, batch, 1)[:, 0]
    return np.exp(np.log(lo) + u * (np.log(hi) - np.log(lo)))


def rescale(a: np.ndarray, targets) -> np.ndarray:
    f = np.asarray(targets, np.float64) / one_norm_batched(a)
    return a * f[:, None, None]


@dataclass(frozen=True)
class Config:
    key: str
    n: int
    batch: int
    dtype: str          # storage / arithmetic type of the GPU path
    accuracy: int       # 0 = Single table (u = 2^-24), 1 = Double (u = 2^-53)
    description: str

    @property
    def unit_roundoff(self) -> float:
        return 2.0 ** -24 if self.accuracy == 0 else 2.0 ** -53

    @property
    def tolerance(self) -> float:
        """Relative Frobenius tolerance 50 * N * u from BASELINE.json."""
        return 50.0 * self.n * self.unit_roundoff


CONFIGS = {
    "cfg1": Config("cfg1", 64, 1, "f64", 1,
                   "single 64x64 fp64, N(0,1) seed 0, ||A||_1 = 2"),
    "cfg2": Config("cfg2", 8, 262144, "f64", 1,
                   "262144 x 8x8 fp64, U(-1,1), ||A||_1 log-uniform [1e-4, 1e2]"),
    "cfg3": Config("cfg3", 32, 65536, "f32", 0,
                   "65536 x 32x32 fp32, half N(0,1/N) dense, half skew B-B^T, "
                   "||A||_1 log-uniform [1e-2, 50]"),
    "cfg4": Config("cfg4", 512, 1024, "f64", 1,
                   "1024 x 512x512 fp64, N(0,1/N), ||A||_1 log-uniform [0.5, 20]"),
    "cfg5": Config("cfg5", 8192, 1, "f64", 1,
                   "single 8192x8192 fp64, strictly-upper N(0,1/N) + diag U(-5,0), "
                   "||A||_1 = 30"),
}


def generate(key: str, b0: int = 0, batch: int | None = None, seed: int = 0) -> np.ndarray:
    """Matrices [b0, b0 + batch) of config ``key`` as a (batch, n, n) array.

    Any shard [b0, b0+batch) equals the same rows of the full batch, so ranks
    can generate only their own matrices.
    """
    cfg = CONFIGS[key]
    n = cfg.n
    batch = cfg.batch - b0 if batch is None else batch
    nn = n * n
    if key == "cfg1":
        a = normal(seed, 10, b0, batch, nn).reshape(batch, n, n)
        return rescale(a, np.full(batch, 2.0))
    if key == "cfg2":
        a = uniform_pm1(seed, 20, b0, batch, nn).reshape(batch, n, n)
        return rescale(a, log_uniform(seed, 21, b0, batch, 1e-4, 1e2))
    if key == "cfg3":
        g = normal(seed, 30, b0, batch, nn).reshape(batch, n, n) / np.sqrt(n)
        idx = np.arange(b0, b0 + batch)
        skew = (idx % cfg.batch) >= cfg.batch // 2  # periodic: weak-scaling shards
        g[skew] = g[skew] - np.transpose(g[skew], (0, 2, 1))
        a = rescale(g, log_uniform(seed, 32, b0, batch, 1e-2, 50.0))
        return a.astype(np.float32)
    if key == "cfg4":
        out = np.empty((batch, n, n), np.float64)
        step = 16
        for c in range(0, batch, step):
            k = min(step, batch - c)
            a = normal(seed, 40, b0 + c, k, nn).reshape(k, n, n) / np.sqrt(n)
            out[c:c + k] = rescale(a, log_uniform(seed, 42, b0 + c, k, 0.5, 20.0))
        return out
    if key == "cfg5":
        a = np.empty((1, n, n), np.float64)
        rows = 256
        for r0 in range(0, n, rows):
            # elements of rows [r0, r0+rows), element index = i*n + j
            g = normal(seed, 50, 0, 1, rows * n, e0=r0 * n).reshape(rows, n)
            g /= np.sqrt(n)
            d = -5.0 * uniform01(seed, 52, 0, 1, rows, e0=r0)[0]
            i = np.arange(r0, r0 + rows)[:, None]
            j = np.arange(n)[None, :]
            blk = np.where(j > i, g, 0.0)
            blk[np.arange(rows), np.arange(r0, r0 + rows)] = d
            a[0, r0:r0 + rows] = blk
        return rescale(a, np.full(1, 30.0))
    raise KeyError(key)


def skew_mask(key: str, b0: int, batch: int) -> np.ndarray:
    """Which matrices of a cfg3 shard are the skew-symmetric half."""
    cfg = CONFIGS[key]
    return (np.arange(b0, b0 + batch) % cfg.batch) >= cfg.batch // 2
