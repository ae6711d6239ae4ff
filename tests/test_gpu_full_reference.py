"""Full-configuration parity of the large-n configs against the compiled
reference (oracle/_ref, the unmodified mexp library), in the same run:

* cfg4: all 1,024 matrices of 512 x 512. The reference runs one worker
  process per host core, OMP_NUM_THREADS=1, each over a contiguous shard
  (mexp::expm, expm.cpp:37-74); every (m, s) and norm_in bit-equal, every e^A
  within 50 n u = 2.84e-12.
* cfg5: the 8192 x 8192 matrix, the reference with its own OpenMP over all
  host cores (kernels.cpp:16-27); e^A within 4.55e-11. About 10-15 minutes of
  host time, so it runs only with MEXP_FULL_CFG5=1 (round-2 result:
  profiles/parity_full_cfg5_r2.json).

The reference's wall time is printed (and written to $MEXP_PARITY_OUT/*.json
when that is set): the same-run CPU baseline of these configs.
"""
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np
import pytest

import paper_1710_10989_b200 as mx
from paper_1710_10989_b200 import workloads

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _ref_shard(args):
    key, b0, count, shm_name, shape = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from multiprocessing import shared_memory
    from oracle.oracle import Reference
    a = workloads.generate(key, b0, count)
    t0 = time.perf_counter()
    r = Reference().expm_batch(a)
    secs = time.perf_counter() - t0
    shm = shared_memory.SharedMemory(name=shm_name)
    out = np.ndarray(shape, np.float64, buffer=shm.buf)
    out[b0:b0 + count] = r.out
    del out
    shm.close()
    return b0, r.degree, r.s, r.norm_in, r.status, secs


def reference_batch_parallel(key, workers):
    """The reference over the whole batch of `key`, `workers` processes."""
    import multiprocessing as mp
    from multiprocessing import shared_memory
    from paper_1710_10989_b200.sharding import shard_range
    cfg = workloads.CONFIGS[key]
    shape = (cfg.batch, cfg.n, cfg.n)
    shm = shared_memory.SharedMemory(create=True, size=int(np.prod(shape)) * 8)
    try:
        tasks = []
        for w in range(workers):
            sh = shard_range(w, workers, cfg.batch)
            if sh.count:
                tasks.append((key, sh.b0, sh.count, shm.name, shape))
        t0 = time.perf_counter()
        with mp.get_context("spawn").Pool(len(tasks)) as pool:
            res = pool.map(_ref_shard, tasks, chunksize=1)
        wall = time.perf_counter() - t0
        out = np.ndarray(shape, np.float64, buffer=shm.buf).copy()
    finally:
        shm.close()
        shm.unlink()
    deg = np.zeros(cfg.batch, np.int32)
    s = np.zeros(cfg.batch, np.int32)
    norm = np.zeros(cfg.batch)
    status = np.zeros(cfg.batch, np.int32)
    for b0, d, ss, nn, st, _ in res:
        deg[b0:b0 + len(d)] = d
        s[b0:b0 + len(d)] = ss
        norm[b0:b0 + len(d)] = nn
        status[b0:b0 + len(d)] = st
    return out, deg, s, norm, status, wall, max(r[5] for r in res)


def rel_fro(got, want):
    g = got.reshape(got.shape[0], -1)
    w = want.reshape(want.shape[0], -1)
    return np.linalg.norm(g - w, axis=1) / np.linalg.norm(w, axis=1)


def _record(name, rec):
    d = os.environ.get("MEXP_PARITY_OUT")
    print(json.dumps(rec))
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, name), "w") as f:
            json.dump(rec, f, indent=1)


def test_cfg4_full_batch_vs_reference(cuda, reference):
    cfg = workloads.CONFIGS["cfg4"]
    cores = _cores()
    ref_out, deg, s, norm, status, wall, busy = reference_batch_parallel("cfg4", cores)
    assert (status == 0).all()
    a = workloads.generate("cfg4")
    t0 = time.perf_counter()
    out, sel, st = mx.expm_batched_host(a)
    gpu_wall = time.perf_counter() - t0
    assert st == mx.OK
    assert np.array_equal(sel["degree"], deg) and np.array_equal(sel["s"], s)
    assert np.array_equal(sel["norm_in"].view(np.uint64), norm.view(np.uint64))
    err = rel_fro(out, ref_out)
    _record("parity_full_cfg4_r2.json", {
        "config": "cfg4", "matrices": int(cfg.batch), "n": cfg.n,
        "selection_bit_equal": True, "max_rel_err": float(err.max()),
        "median_rel_err": float(np.median(err)), "tolerance": cfg.tolerance,
        "s_values": sorted(int(x) for x in set(s)),
        "reference": {"wall_s": wall, "slowest_worker_s": busy, "workers": cores,
                      "omp_num_threads": 1, "expm_per_s": cfg.batch / wall,
                      "what": "oracle/_ref (unmodified mexp), one process per core over "
                              "contiguous shards of all 1024 matrices"},
        "gpu_host_call_s": gpu_wall})
    assert err.max() <= cfg.tolerance


_CFG5_SCRIPT = r"""
import os, sys, time, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle.oracle import Reference
from paper_1710_10989_b200 import workloads
a = workloads.generate("cfg5")
t0 = time.perf_counter()
r = Reference().expm_batch(a)
secs = time.perf_counter() - t0
np.save(sys.argv[2], r.out[0])
print(int(r.degree[0]), int(r.s[0]), repr(float(r.norm_in[0])), int(r.status[0]), secs)
"""


@pytest.mark.skipif(os.environ.get("MEXP_FULL_CFG5") != "1",
                    reason="~10-15 min of host time: set MEXP_FULL_CFG5=1")
def test_cfg5_full_vs_reference(cuda, reference):
    import torch
    cfg = workloads.CONFIGS["cfg5"]
    cores = _cores()
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "ref_cfg5.npy")
        env = dict(os.environ, OMP_NUM_THREADS=str(cores))
        t0 = time.perf_counter()
        r = subprocess.run([sys.executable, "-c", _CFG5_SCRIPT, ROOT, path], env=env,
                           capture_output=True, text=True, timeout=4 * 3600)
        wall = time.perf_counter() - t0
        assert r.returncode == 0, r.stderr[-2000:]
        d, s, nrm, st, secs = r.stdout.split()
        want = np.load(path)
    a = workloads.generate("cfg5")
    da = torch.from_numpy(a).cuda()
    out = torch.empty_like(da)
    sel = torch.empty(16, dtype=torch.uint8, device="cuda")
    mx.expm_batched(da, out, sel)
    torch.cuda.synchronize()
    rec = sel.cpu().numpy().view(mx.SELECTION_DTYPE)[0]
    assert (int(rec["degree"]), int(rec["s"]), int(rec["status"])) == (int(d), int(s), 0)
    assert float(rec["norm_in"]) == float(nrm)
    got = out[0].cpu().numpy()
    err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    _record("parity_full_cfg5_r2.json", {
        "config": "cfg5", "n": cfg.n, "degree": int(d), "s": int(s),
        "selection_bit_equal": True, "rel_err": err, "tolerance": cfg.tolerance,
        "reference": {"expm_s": float(secs), "process_wall_s": wall, "omp_num_threads": cores,
                      "expm_per_s": 1.0 / float(secs),
                      "what": "oracle/_ref (unmodified mexp) mexp::expm on the 8192^2 matrix, "
                              "its OpenMP row split over all host cores"}})
    assert err <= cfg.tolerance
