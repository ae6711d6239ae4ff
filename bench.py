"""Benchmark: batched scaling-and-squaring expm (arXiv 1710.10989 TaylorNew) on B200.

Default workload = BASELINE.json configs[1] (cfg2): 262,144 fp64 8x8 matrices,
U(-1,1) rescaled to a log-uniform 1-norm in [1e-4, 1e2]. A step is one
batched expm over the job's 262,144 matrices, inputs resident in HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfgX]
                    [--impl ours|reference] [--rounding auto|reference|fast]
                    [--weak] [--dry-run]

Multi-GPU: one process per GPU over NCCL. With
``--gpus N`` and no torchrun environment, bench.py re-launches itself under
``torch.distributed.run`` with N ranks. The config's batch is split by matrix
(rank r owns [r*B/N + min(r, B%N), ...), ``"scaling": "strong"``); ``--weak``
gives every rank its own full batch instead. No collective runs on the data
path; an NCCL gather of e^A and the selection records to rank 0 (grouped
ncclSend/ncclRecv) is timed separately on the device ("gather") and checked
bit for bit against rank 0 recomputing the whole batch.

Prints ONE JSON line on rank 0. `value` = expm/s over all ranks (device time,
CUDA events, max over ranks); `e2e` = the same metric through the host C-ABI
call (mexp_expm_batched_host: pinned H2D + kernels + D2H inside the timed
region, max over ranks). --impl reference times the reference's own CPU
implementation (oracle/_ref, the unmodified mexp library) on all host cores,
the same way as the `cpu_baseline` leg of our arm (one worker process per core,
each owning a contiguous shard of the config's batch; a step's time is the
slowest worker's, like the max over GPU ranks).

--dry-run checks the multi-rank plumbing on CPU (gloo): launch, shard split,
gather and the rank-0 JSON line, with the per-rank compute replaced by a copy.
It measures nothing and says so ("dry_run": true, "value": null).
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1710_10989_b200 import workloads  # noqa: E402
from paper_1710_10989_b200.sharding import gather_to_root, max_over_ranks, shard_range  # noqa: E402

METRIC = "matrix exponentials/sec and effective TFLOP/s (fraction of HBM/FP64 roofline)"
UNIT = "expm/s"
L2_BYTES = 126 * 2 ** 20


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


def compute_peak_tflops(dtype):
    """FP64 (DMMA) / FP32 (FFMA) peak measured on a B200 of this pool by
    tools/fp64_peak.cu (profiles/fp64_peak.json); datasheet-class otherwise."""
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    if dtype == "f64":
        if "dmma_tflops" in d:
            return d["dmma_tflops"], "measured (tools/fp64_peak.cu, DMMA m8n8k4)"
        return 37.2, "datasheet-class (148 SM x 64 FMA/clk x 2 x 1.965 GHz)"
    if "ffma_tflops" in d:
        return d["ffma_tflops"], "measured (tools/fp64_peak.cu, FFMA)"
    return 74.4, "datasheet-class (148 SM x 128 FFMA/clk x 2 x 1.965 GHz)"


# Which roofline binds each workload: the batched
# small-n configs are quoted against HBM (BASELINE.json), the large-n ones
# against the FP64 tensor-core peak.
ROOFLINE_BOUND = {"cfg1": "tensor", "cfg2": "hbm", "cfg3": "hbm", "cfg4": "tensor",
                  "cfg5": "tensor"}
KERNEL_NAME = {
    "cfg1": "expm64_cluster_kernel (1 launch per step)",
    "cfg2": "expm8_pipe_kernel (1 launch per step)",
    "cfg3": "select32 + scatter32 pre-pass, expm32_pairs_kernel (3 launches per step; "
            "the pair kernel ~92% of the step)",
    "cfg4": "gemm_dmma_kernel<*> chain (all launches of the step; GEMMs dominate)",
    "cfg5": "gemm_dmma_kernel<*> chain (all launches of the step; GEMMs dominate)",
}


FAMILIES = {"taylor-new": 0, "taylor-ps": 1, "pade": 2}
# products per degree of each family's table (theta_tables.cpp:45-73); the
# Pade solve counts 4/3 of a product (expm.cpp:70-72)
PRODUCTS = {0: {1: 0, 2: 1, 4: 2, 8: 3, 12: 4, 18: 5},
            1: {1: 0, 2: 1, 4: 2, 6: 3, 9: 4, 16: 6},
            2: {2: 0, 4: 1, 6: 2, 8: 3, 10: 3, 12: 4, 14: 4, 16: 5, 18: 5, 20: 5, 22: 6, 24: 6,
                26: 6}}


def flops_per_matrix(n, degree, s, family=0):
    prods = np.vectorize(PRODUCTS[family].get)(degree) + (4.0 / 3.0 if family == 2 else 0.0)
    return 2.0 * n ** 3 * (prods + s)


class ClockSampler:
    """NVML clock/throttle sampling during the timed region (1-2 ms period)."""

    def __init__(self, device_index=0):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
            "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            # the first sample is taken before the timed work starts
            t0 = time.perf_counter()
            while not self.samples and time.perf_counter() - t0 < 0.05:
                time.sleep(0.0005)
        return self

    def __exit__(self, *a):
        if self.nv:
            try:  # one sample at the end of the timed region as well
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            except Exception:
                pass
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------ CPU reference --
# The reference's CPU path (oracle/_ref = the unmodified mexp library), timed
# the way the GPU ranks are: P worker processes, each owning a contiguous
# shard of the config's batch, generated before timing; one step = every
# worker runs mexp::expm over (a sample of) its shard; the step's time is the
# slowest worker's. OMP_NUM_THREADS=1 per worker for the batched configs (the
# reference parallelises only inside one product for n > 64,
# kernels.cpp:16-27); a single large matrix (cfg5) runs in one process with
# the reference's own OpenMP over all cores.
def _cpu_worker(conn, key, b0, count, family, omp):
    os.environ["OMP_NUM_THREADS"] = str(omp)
    from oracle.oracle import Reference
    ref = Reference()
    cfg = workloads.CONFIGS[key]
    a = workloads.generate(key, b0, count) if count else None
    conn.send("ready")
    while True:
        msg = conn.recv()
        if msg is None:
            break
        k = min(int(msg), count)
        t0 = time.perf_counter()
        if k:
            ref.expm_batch(a[:k], accuracy=cfg.accuracy, family=family)
        conn.send((k, time.perf_counter() - t0))
    conn.close()


class CpuReference:
    """Persistent reference workers over a contiguous split of matrices
    [0, total) of config `key` (total <= the config's batch)."""

    def __init__(self, key, workers, total, family=0, omp=1):
        ctx = mp.get_context("spawn")
        self.procs, self.conns, self.counts = [], [], []
        for w in range(workers):
            sh = shard_range(w, workers, total)
            parent, child = ctx.Pipe()
            p = ctx.Process(target=_cpu_worker, args=(child, key, sh.b0, sh.count, family, omp),
                            daemon=True)
            p.start()
            self.procs.append(p)
            self.conns.append(parent)
            self.counts.append(sh.count)
        for c in self.conns:
            assert c.recv() == "ready"

    def step(self, per_worker=None):
        """One step over `per_worker` matrices per worker (default: the whole
        shard). Returns (matrices done, slowest worker's seconds)."""
        for c, cnt in zip(self.conns, self.counts):
            c.send(cnt if per_worker is None else per_worker)
        res = [c.recv() for c in self.conns]
        return sum(r[0] for r in res), max(r[1] for r in res)

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except Exception:
                pass
        for p in self.procs:
            p.join(timeout=30)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_reference_measure(key, family, steps, warmup, sample="default", budget_s=120.0):
    """The reference's CPU rate on this host for config `key`, shared by
    --impl reference and the cpu_baseline leg. Returns (rate, record)."""
    cfg = workloads.CONFIGS[key]
    cores = host_cores()
    fam_name = {v: k for k, v in FAMILIES.items()}[family]
    if key == "cfg1":
        # one 64x64 matrix: the reference runs it on one core (no OpenMP for
        # n <= 64, kernels.cpp:13,18); the rate is 1 / per-call latency
        os.environ["OMP_NUM_THREADS"] = "1"
        from oracle.oracle import Reference
        ref = Reference()
        a = workloads.generate(key, 0, 1)
        for _ in range(max(warmup, 1) * 10):
            ref.expm_batch(a, accuracy=cfg.accuracy, family=family)
        lat = []
        t_end = time.perf_counter() + min(budget_s, 5.0)
        for _ in range(max(steps, 1)):
            calls = 50
            t0 = time.perf_counter()
            for _ in range(calls):
                ref.expm_batch(a, accuracy=cfg.accuracy, family=family)
            lat.append((time.perf_counter() - t0) / calls)
            if time.perf_counter() > t_end:
                break
        v = 1.0 / statistics.median(lat)
        return v, {"value": v, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"{len(lat)} x 50 mexp::expm calls on the cfg1 matrix, one core "
                             f"(median per-call latency {1e6 * statistics.median(lat):.1f} us)",
                   "steps": len(lat), "cpu": cpu_model(), "family": fam_name}
    if key == "cfg5":
        if sample == "full":
            # the whole expm of the 8192^2 matrix with the reference's OpenMP
            os.environ["OMP_NUM_THREADS"] = str(cores)
            w = CpuReference(key, 1, 1, family, omp=cores)
            try:
                done, secs = w.step()
            finally:
                w.close()
            v = done / secs
            return v, {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                       "sample": f"the full cfg5 expm (one 8192^2 matrix), mexp::expm with "
                                 f"OMP_NUM_THREADS={cores}: {secs:.1f} s",
                       "steps": 1, "cpu": cpu_model(), "family": fam_name}
        # bounded sample: one reference product (kernels::matmul, OpenMP row
        # split, kernels.cpp:16-27) of two 2048^2 blocks of the cfg5 matrix,
        # scaled by flops to the cfg5 expm (10 products of 8192^2)
        os.environ["OMP_NUM_THREADS"] = str(cores)
        from oracle.oracle import Reference
        ref = Reference()
        nb = 2048
        a = workloads.generate(key, 0, 1)[0, :nb, :nb].copy()
        ref.matmul(a, a)
        t0 = time.perf_counter()
        ref.matmul(a, a)
        secs = time.perf_counter() - t0
        gflops = 2.0 * nb ** 3 / secs / 1e9
        expm_flops = 2.0 * 8192 ** 3 * 10
        v = gflops * 1e9 / expm_flops
        return v, {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"one reference kernels::matmul of a 2048^2 block of the cfg5 matrix "
                             f"({gflops:.1f} GFLOP/s, OMP_NUM_THREADS={cores}), scaled to the "
                             f"cfg5 expm's 10 products of 8192^2 (bench.py --cpu-sample full "
                             f"times the whole expm)",
                   "steps": 1, "cpu": cpu_model(), "family": fam_name}
    # batched configs: one worker process per core over the config's batch
    total = cfg.batch
    per = None
    if key == "cfg4" and sample != "full":
        per = 1  # one 512^2 matrix per worker per step (~0.3-0.6 s)
    w = CpuReference(key, cores, total, family, omp=1)
    try:
        for _ in range(max(warmup, 1)):
            w.step(per)
        rates, secs_all = [], []
        t_end = time.perf_counter() + budget_s
        for _ in range(max(steps, 1)):
            done, secs = w.step(per)
            rates.append(done / secs)
            secs_all.append(secs)
            if time.perf_counter() > t_end:
                break
    finally:
        w.close()
    v = statistics.median(rates)
    what = (f"the full {total}-matrix batch per step" if per is None else
            f"{per} matrix per worker per step ({per * cores} of the {total})")
    return v, {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
               "sample": f"{cores} worker processes (OMP_NUM_THREADS=1), each owning a contiguous "
                         f"shard of {key}; {what}; rate = matrices / slowest worker's time, "
                         f"median of {len(rates)} steps",
               "steps": len(rates), "step_s_median": statistics.median(secs_all),
               "cpu": cpu_model(), "family": fam_name}


# ---------------------------------------------------------------- main ----
def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None,
                   help="timed steps (default per config: a timed region of ~0.1-1 s so clock samples "
                        "and transients average out; the reference arm: 20)")
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--config", default="cfg2", choices=sorted(workloads.CONFIGS))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--rounding", default="auto", choices=["auto", "reference", "fast"])
    p.add_argument("--family", default="taylor-new", choices=sorted(FAMILIES),
                   help="Family (theta_tables.hpp:8); the headline is taylor-new")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample", default="default", choices=["default", "full"],
                   help="cfg4/cfg5 CPU baseline over the whole workload instead of a bounded sample")
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--weak", action="store_true",
                   help="every rank owns a full config-sized batch (weak scaling) instead of the "
                        "split of one batch (the default)")
    p.add_argument("--strong", action="store_true", help=argparse.SUPPRESS)  # the default
    p.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                   help="capture the timed steps in one CUDA graph (auto: n <= 64)")
    p.add_argument("--no-verify-gather", action="store_true")
    p.add_argument("--dry-run", action="store_true",
                   help="multi-rank plumbing check on CPU (gloo); compute replaced by a copy")
    p.add_argument("--dry-batch", type=int, default=None, help="dry run: matrices in the job")
    a = p.parse_args()
    if a.steps is None:
        a.steps = 20 if a.impl == "reference" else {"cfg1": 1000, "cfg2": 1000, "cfg3": 300,
                                                     "cfg4": 10, "cfg5": 3}[a.config]
    if a.dry_run:
        a.steps = min(a.steps, 3)
    return a


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args):
    """`--gpus N` without a torchrun environment: run N ranks of this script."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def workload_config(args, world, per_rank, batch=None):
    """The `config` object of both arms' JSON lines (same keys and values)."""
    cfg = workloads.CONFIGS[args.config]
    batch = cfg.batch if batch is None else batch
    total = world * batch if args.weak else batch
    esz = 8 if cfg.dtype == "f64" else 4
    io = 2 * per_rank * cfg.n * cfg.n * esz
    small = io < L2_BYTES // 8
    return {"workload": args.config, "description": cfg.description, "n": cfg.n,
            "batch_per_rank": per_rank, "global_batch": total, "rounding": args.rounding,
            "family": args.family,
            "parallelism": f"matrix-sharded x{world}" + (" (weak: a full batch per rank)" if args.weak
                                                        else " (one batch split by matrix)"),
            "l2": (f"L2 flushed before every step (write of {2 * L2_BYTES >> 20} MiB); steps captured "
                   f"in one CUDA graph, expm part timed by in-graph events" if small else
                   f"inputs larger than L2 (in+out {io / 2 ** 20:.0f} MiB per rank, two alternating "
                   f"buffer pairs when they fit)")}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = workloads.CONFIGS[args.config]
    if cfg.batch == 1 and world > 1:
        args.weak = True  # single-matrix configs run as replicas (as our arm does)
    value, rec = cpu_reference_measure(args.config, FAMILIES[args.family], args.steps, args.warmup,
                                       args.cpu_sample)
    per_rank = cfg.batch if args.weak else shard_range(0, world, cfg.batch).count
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": rec["steps"], "warmup": args.warmup,
        "ms_per_step": 1e3 * cfg.batch / value,
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None,
        "dtype": cfg.dtype, "data": "synthetic (seeded, counter-based; see workloads.py)",
        "config": workload_config(args, world, per_rank),
        "cpu_baseline": rec,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "execution": "the unmodified reference library (oracle/_ref) on the host cores",
    }
    print(json.dumps(line), flush=True)


def nccl_comm_lines(path_prefix):
    """NCCL's own INIT log lines of this process (rank / nRanks / comm)."""
    import glob
    lines = []
    for f in glob.glob(path_prefix + "*"):
        try:
            for ln in open(f):
                if ("nRanks" in ln and "comm" in ln) or "Init COMPLETE" in ln:
                    lines.append(ln.strip())
        except OSError:
            pass
    return lines


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    dry = args.dry_run
    if dry:
        mx = None
        dev = torch.device("cpu")
    else:
        import paper_1710_10989_b200 as mx
        if not torch.cuda.is_available():
            raise SystemExit("bench.py: no CUDA device (there is no CPU fallback; --dry-run checks "
                             "the multi-rank plumbing only)")
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
    nccl_prefix = None
    if world > 1:
        if dry:
            dist.init_process_group("gloo")
        else:
            if "NCCL_DEBUG" not in os.environ:
                nccl_prefix = f"/tmp/mexp_bench_nccl_r{rank}_{os.getpid()}"
                os.environ["NCCL_DEBUG"] = "INFO"
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                os.environ["NCCL_DEBUG_FILE"] = nccl_prefix + ".%h.%p.log"
            dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
    cfg = workloads.CONFIGS[args.config]
    n = cfg.n
    B = cfg.batch if not (dry and args.dry_batch) else args.dry_batch
    if B == 1 and world > 1 and not args.weak:
        # a single matrix (cfg1, cfg5) does not shard: replicas only
        args.weak = True
        if rank == 0:
            print("bench.py: single-matrix config -> one replica per rank (--weak)", file=sys.stderr)
    shard = shard_range(rank, world, B, weak=args.weak)
    Bl = shard.count
    total = world * B if args.weak else B
    counts = [shard_range(r, world, B, weak=args.weak).count for r in range(world)]
    a_host = workloads.generate(args.config, shard.b0, shard.count)
    fam = FAMILIES[args.family]
    esz = 8 if cfg.dtype == "f64" else 4
    mat_bytes = n * n * esz
    # two input/output buffer pairs alternate so the working set exceeds L2
    pairs = 2 if 2 * Bl * mat_bytes < 4 * L2_BYTES else 1
    ins = [torch.from_numpy(a_host).to(dev) for _ in range(pairs)]
    outs = [torch.empty_like(ins[0]) for _ in range(pairs)]
    sel = torch.zeros(max(Bl, 1) * 16, dtype=torch.uint8, device=dev)
    if not dry:
        rounding = {"auto": mx.ROUND_AUTO, "reference": mx.ROUND_REFERENCE,
                    "fast": mx.ROUND_FAST}[args.rounding]
        stream = torch.cuda.current_stream(dev)
        kw = dict(accuracy=mx.Accuracy(cfg.accuracy), rounding=rounding, family=mx.Family(fam))

    def step(i, st=None):
        if dry:
            outs[i % pairs].copy_(ins[i % pairs])
            return
        mx.expm_batched(ins[i % pairs], outs[i % pairs], sel, stream=st or stream, **kw)

    for i in range(max(args.warmup, 3)):
        step(i)
    if not dry:
        torch.cuda.synchronize()
    flops = 0.0
    if not dry and Bl:
        sels = sel.cpu().numpy().view(mx.SELECTION_DTYPE)[:Bl]
        flops = float(flops_per_matrix(n, sels["degree"], sels["s"], fam).sum())

    small = 2 * Bl * mat_bytes < L2_BYTES // 8
    use_graph = (not dry) and (args.graph == "on" or (args.graph == "auto" and n <= 64))
    if world > 1:
        dist.barrier()
    if not dry:
        torch.cuda.synchronize()
    launches0 = 0 if dry else mx.launch_count()
    clk = ClockSampler(local) if not dry else None
    timing = ""
    if dry:
        t0 = time.perf_counter()
        for i in range(args.steps):
            step(i)
        ms = 1e3 * (time.perf_counter() - t0)
        launches = 0
        timing = "dry run: wall clock of the copies (measures nothing)"
    elif use_graph:
        # The K steps are captured in one CUDA graph (no host launch gaps:
        # at 8 ranks a cfg2 shard is ~15 us of kernel, less than a Python +
        # ctypes launch). Few, small matrices (cfg1): an L2 flush (a write of
        # 2x L2) before every step and only the expm part of each step timed,
        # by CUDA events recorded inside the graph.
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if small else None
        evs = [(torch.cuda.Event(enable_timing=True, external=True),
                torch.cuda.Event(enable_timing=True, external=True))
               for _ in range(args.steps)] if small else None
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            gs = torch.cuda.current_stream(dev)
            for i in range(args.steps):
                if small:
                    flush.fill_(float(i))
                    evs[i][0].record(gs)
                step(i, gs)
                if small:
                    evs[i][1].record(gs)
        launches = mx.launch_count() - launches0
        graph.replay()  # warm the graph
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with clk:
            ev0.record(stream)
            graph.replay()
            ev1.record(stream)
            torch.cuda.synchronize()
        ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) if small else ev0.elapsed_time(ev1)
        timing = ("CUDA graph of the K steps; CUDA events " +
                  ("inside the graph around each expm (L2 flushed before each)" if small else
                   "on the launching stream around the graph replay"))
    else:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with clk:
            ev0.record(stream)
            for i in range(args.steps):
                step(i)
            ev1.record(stream)
            torch.cuda.synchronize()
        launches = mx.launch_count() - launches0
        ms = ev0.elapsed_time(ev1)
        timing = "CUDA events on the launching stream around the K steps"
    rank_ms = ms
    flops_total = flops
    if world > 1:
        ms = max_over_ranks(ms, dev)
        t = torch.tensor([flops], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        flops_total = float(t.item())
        dist.barrier()
    ms_step = ms / args.steps
    value = total / (ms_step * 1e-3)

    # ---- e2e through the host C-ABI call (pinned buffers), max over ranks ----
    e2e_value, e2e_how = None, None
    if not dry and Bl:
        h_in = torch.from_numpy(a_host).pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        for _ in range(2):
            mx.expm_batched_host(h_in, h_out, **kw)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            mx.expm_batched_host(h_in, h_out, **kw)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        e2e_how = ("mexp_expm_batched_host (each rank its own shard over its own PCIe link), "
                   "pinned host buffers, wall clock per call, max over ranks")
        # A single double matrix under the TaylorNew family (cfg1): the
        # reference's caller makes one mexp::expm call per matrix from C++, so
        # the per-call time is taken natively (bin/call_latency: the C++
        # drop-in on a host DenseMatrix, 2000 calls) instead of through
        # Python's ctypes overhead.
        native = os.path.join(ROOT, "bin", "call_latency")
        if Bl == 1 and n <= 64 and cfg.dtype == "f64" and fam == 0 and args.rounding == "auto" \
                and os.path.exists(native):
            import tempfile
            with tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as tf:
                a_host[0].astype("<f8").tofile(tf.name)
            try:
                r = subprocess.run([native, tf.name, str(n), "2000"], capture_output=True, text=True,
                                   timeout=120)
                e2e_s = json.loads(r.stdout.strip().splitlines()[-1])["us_per_call"] * 1e-6
                e2e_how = ("mexp::expm (C++ drop-in, expm.hpp:37) on a host DenseMatrix, 2000 calls "
                           "timed natively by bin/call_latency")
            except Exception as exc:  # keep the Python-timed value
                e2e_how += f" (native timing unavailable: {exc})"
            finally:
                os.unlink(tf.name)
        if world > 1:
            e2e_s = max_over_ranks(e2e_s, dev)
        e2e_value = total / e2e_s
    elif world > 1 and not dry:
        max_over_ranks(0.0, dev)

    # ---- gather of e^A and the records to rank 0, timed on the device ----
    gather = None
    if world > 1:
        if not dry:
            torch.cuda.synchronize()
        dist.barrier()
        root_out = None
        if rank == 0:
            root_out = torch.empty((sum(counts), n, n), dtype=outs[0].dtype, device=dev)
        sel_l = sel[:16 * Bl]
        if dry:
            g0 = time.perf_counter()
            got = gather_to_root(outs[0], counts, out=root_out)
            gsel = gather_to_root(sel_l.view(-1, 16), counts)
            g_ms = 1e3 * (time.perf_counter() - g0)
        else:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            got = gather_to_root(outs[0], counts, out=root_out)
            gsel = gather_to_root(sel_l.view(-1, 16), counts)
            e1.record()
            torch.cuda.synchronize()
            g_ms = e0.elapsed_time(e1)
        g_ms = max_over_ranks(g_ms, dev if not dry else None)
        gather = {"ms": g_ms, "bytes_to_root": (sum(counts) - counts[0]) * (mat_bytes + 16),
                  "how": "grouped send/recv to rank 0 (torch.distributed.batch_isend_irecv: "
                         "ncclGroupStart, ncclSend/ncclRecv per rank, ncclGroupEnd), "
                         "receiving in place into rank 0's result; " +
                         ("wall clock (dry run)" if dry else "CUDA events, max over ranks")}
        # the gathered job result must equal the whole batch computed in one place
        if rank == 0 and not args.weak and not args.no_verify_gather:
            full = workloads.generate(args.config, 0, B)
            if dry:
                ok = np.array_equal(got.numpy(), full)
            else:
                fa = torch.from_numpy(full).to(dev)
                fo = torch.empty_like(fa)
                fs = torch.empty(B * 16, dtype=torch.uint8, device=dev)
                mx.expm_batched(fa, fo, fs, **kw)
                torch.cuda.synchronize()
                ok = torch.equal(fo.view(torch.uint8), got.view(torch.uint8)) and \
                    torch.equal(fs.view(-1, 16), gsel)
                del fa, fo, fs
            gather["verified_bitwise_vs_one_gpu"] = bool(ok)
        del got, gsel, root_out

    # ---- per-rank evidence ----
    me = {"rank": rank, "b0": shard.b0, "count": Bl, "ms": rank_ms,
          "device": "cpu (dry run)" if dry else torch.cuda.get_device_name(dev),
          "pci_bus_id": None if dry else _pci_bus_id(local)}
    if nccl_prefix:
        me["nccl"] = nccl_comm_lines(nccl_prefix)[:4]
    ranks = [me]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, me)
    for r in ranks if rank == 0 else []:
        print(f"bench.py rank {r['rank']}/{world}: shard [{r['b0']}, {r['b0'] + r['count']}) on "
              f"{r['device']} {r['pci_bus_id'] or ''}, {r['ms'] / args.steps:.3f} ms/step", file=sys.stderr)
        for ln in r.get("nccl", []):
            print(f"  {ln}", file=sys.stderr)

    if rank == 0:
        line = {
            "metric": METRIC, "value": None if dry else value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None,
            "dtype": cfg.dtype, "data": "synthetic (seeded, counter-based; see workloads.py)",
            "config": workload_config(args, world, Bl, B),
            "timing": timing,
            "ranks": [{k: r[k] for k in ("rank", "b0", "count", "ms", "device", "pci_bus_id")}
                      for r in ranks],
        }
        if nccl_prefix:
            line["nccl"] = {"version": ".".join(map(str, torch.cuda.nccl.version())),
                            "comm_init": [r.get("nccl", [])[:1] for r in ranks]}
        if dry:
            line["dry_run"] = True
        else:
            peaks = load_peaks()
            alg_bytes = 2.0 * Bl * mat_bytes  # one read of A, one write of e^A per matrix (this rank)
            hbm_gbs = alg_bytes / (ms_step * 1e-3) / 1e9
            traffic = None
            tpath = os.path.join(ROOT, "profiles", "traffic.json")
            if os.path.exists(tpath):
                key = f"{args.config}_{args.rounding}" + ("" if fam == 0 else f"_{args.family}")
                traffic = json.load(open(tpath)).get(key)
            peakc, peakc_src = compute_peak_tflops(cfg.dtype)
            tflops = flops / (ms_step * 1e-3) / 1e12
            if ROOFLINE_BOUND[args.config] == "hbm":
                roof = {"bound": "hbm", "achieved": hbm_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": hbm_gbs / peaks["hbm_gbs"], "traffic": traffic,
                        "peak_source": peaks["source"] + " (MEASURED_PEAKS.json hbm_gbs)"}
            else:
                roof = {"bound": "tensor", "achieved": tflops, "peak": peakc, "unit": "TFLOP/s",
                        "frac": tflops / peakc, "traffic": traffic, "peak_source": peakc_src}
            roof["kernel"] = KERNEL_NAME[args.config] if fam == 0 else f"{args.family} kernels"
            roof["algorithmic"] = (f"{alg_bytes / 1e6:.1f} MB (A in + e^A out) and "
                                   f"{flops / 1e9:.2f} GFLOP (sum 2 n^3 (pi_m + s)) per step, rank 0")
            line.update({
                "effective_tflops": flops_total / (ms_step * 1e-3) / 1e12,
                "compute_peak": {"tflops": peakc, "source": peakc_src, "frac": tflops / peakc},
                "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": peaks["hbm_gbs"],
                        "frac": hbm_gbs / peaks["hbm_gbs"]},
                "roofline": roof,
                "e2e": {"value": e2e_value, "unit": UNIT,
                        "h2d_bytes_per_step": total * mat_bytes,
                        "d2h_bytes_per_step": total * (mat_bytes + 16),
                        "how": e2e_how},
                "gpu_launches": int(launches),
                "clocks": clk.summary(),
            })
            if not args.no_cpu_baseline and world == 1:
                _, rec = cpu_reference_measure(args.config, fam, steps=3, warmup=1,
                                               sample=args.cpu_sample, budget_s=30.0)
                line["cpu_baseline"] = rec
        if gather:
            line["gather"] = gather
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _pci_bus_id(local):
    try:
        import torch
        p = torch.cuda.get_device_properties(local)
        return f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}"
    except Exception:
        return None


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    rank, world, _ = dist_env()
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE",
              file=sys.stderr)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
