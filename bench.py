"""Benchmark: batched scaling-and-squaring expm (arXiv 1710.10989 TaylorNew) on B200.

Default workload = BASELINE.json configs[1] (cfg2): 262,144 fp64 8x8 matrices,
U(-1,1) rescaled to a log-uniform 1-norm in [1e-4, 1e2]. A step is one
batched expm over the rank's 262,144 matrices, inputs resident in HBM. With N
GPUs every rank runs its own 262,144 matrices (global indices
[rank*B, (rank+1)*B)), no collective on the data path -> "scaling": "weak";
an NCCL gather of the results to rank 0 is timed separately ("gather").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfgX]
                    [--impl ours|reference] [--rounding auto|reference|fast]

Prints ONE JSON line on rank 0. `value` = expm/s over all ranks (device time,
CUDA events, max over ranks); `e2e` = the same metric through the host C-ABI
call (mexp_expm_batched_host: pinned H2D + kernels + D2H inside the timed
region). --impl reference times the reference's own CPU implementation
(oracle/_ref, the unmodified mexp library) on all host cores.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
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
    "cfg1": "expm_small_f64_kernel<64,1> (1 launch per step)",
    "cfg2": "expm8_f64_kernel (1 launch per step)",
    "cfg3": "expm_small_f32_kernel<32,2> (1 launch per step)",
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


# ---------------------------------------------------------------- CPU arms --
def _ref_worker(args):
    key, b0, count, chunk, family = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle.oracle import Reference
    ref = Reference()
    a = workloads.generate(key, b0, count)
    cfg = workloads.CONFIGS[key]
    t0 = time.perf_counter()
    done = 0
    for c in range(0, count, chunk):
        ref.expm_batch(a[c:c + chunk], accuracy=cfg.accuracy, family=family)
        done += min(chunk, count - c)
    return done, time.perf_counter() - t0


def cpu_reference_rate(key, matrices_per_worker, workers, pool=None, family=0):
    """Aggregate expm/s of the compiled reference over `workers` processes."""
    cfg = workloads.CONFIGS[key]
    tasks = [(key, (w * matrices_per_worker) % max(cfg.batch - matrices_per_worker, 1),
              matrices_per_worker, 256, family) for w in range(workers)]
    own = pool is None
    if own:
        pool = mp.get_context("spawn").Pool(workers)
    try:
        t0 = time.perf_counter()
        res = pool.map(_ref_worker, tasks)
        wall = time.perf_counter() - t0
    finally:
        if own:
            pool.close()
            pool.join()
    done = sum(r[0] for r in res)
    busy = max(r[1] for r in res)
    return done / busy, done, wall


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


def per_worker_sample(key):
    # ~2-4 s of single-core work per worker (survey probe: cfg2 ~130k/s/core,
    # cfg3 ~9k/s, cfg1 ~1.1k/s); keeps the whole CPU leg well under a minute
    return {"cfg1": 256, "cfg2": 32768, "cfg3": 2048, "cfg4": 1, "cfg5": 1}[key]


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
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--strong", action="store_true",
                   help="split the config's batch across the ranks (strong scaling) instead of "
                        "one full batch per rank (weak, the default)")
    a = p.parse_args()
    if a.steps is None:
        a.steps = 20 if a.impl == "reference" else {"cfg1": 1000, "cfg2": 1000, "cfg3": 300,
                                                     "cfg4": 10, "cfg5": 3}[a.config]
    return a


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = workloads.CONFIGS[args.config]
    cores = host_cores()
    per = per_worker_sample(args.config)
    pool = mp.get_context("spawn").Pool(cores)
    try:
        for _ in range(max(args.warmup, 1)):
            cpu_reference_rate(args.config, max(per // 8, 1), cores, pool, FAMILIES[args.family])
        rates = []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r, done, wall = cpu_reference_rate(args.config, max(per // 8, 1), cores, pool,
                                               FAMILIES[args.family])
            rates.append(r)
            if time.perf_counter() - t0 > 120:  # bound the arm to ~2 minutes
                break
    finally:
        pool.close()
        pool.join()
    value = statistics.median(rates)
    sample = (f"{cores} worker processes x {max(per // 8, 1)} {cfg.n}x{cfg.n} matrices of "
              f"{args.config} per step, OMP_NUM_THREADS=1, rate = matrices / slowest worker's compute time")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": len(rates), "warmup": args.warmup,
        "ms_per_step": 1e3 * (max(per // 8, 1) * cores) / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": cfg.dtype, "data": "synthetic (seeded, counter-based; see workloads.py)",
        "config": {"workload": args.config, "description": cfg.description, "n": cfg.n,
                   "batch": cfg.batch, "family": args.family, "parallelism": "host processes"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1710_10989_b200 as mx

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = workloads.CONFIGS[args.config]
    n = cfg.n
    B = cfg.batch
    # weak scaling (default): each rank owns a full config-sized batch of its
    # own matrices; --strong: the config's batch split by matrix across ranks
    shard = shard_range(rank, world, B, weak=not args.strong)
    Bl = shard.count
    total = B if args.strong else world * B
    a_host = workloads.generate(args.config, shard.b0, shard.count)
    torch_dtype = torch.float64 if cfg.dtype == "f64" else torch.float32
    rounding = {"auto": mx.ROUND_AUTO, "reference": mx.ROUND_REFERENCE,
                "fast": mx.ROUND_FAST}[args.rounding]
    fam = FAMILIES[args.family]
    esz = 8 if cfg.dtype == "f64" else 4
    mat_bytes = n * n * esz
    # two input/output buffer pairs alternate so the working set exceeds L2
    pairs = 2 if 2 * Bl * mat_bytes < 4 * L2_BYTES else 1
    ins = [torch.from_numpy(a_host).to(dev) for _ in range(pairs)]
    outs = [torch.empty_like(ins[0]) for _ in range(pairs)]
    sel = torch.empty(Bl * 16, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(i):
        mx.expm_batched(ins[i % pairs], outs[i % pairs], sel, accuracy=mx.Accuracy(cfg.accuracy),
                        rounding=rounding, stream=stream, family=mx.Family(fam))

    for i in range(max(args.warmup, 3)):
        step(i)
    torch.cuda.synchronize()
    sels = sel.cpu().numpy().view(mx.SELECTION_DTYPE)
    flops = float(flops_per_matrix(n, sels["degree"], sels["s"], fam).sum())

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = mx.launch_count()
    # a working set far inside L2 (cfg1: one matrix): flush + graph timing
    small = 2 * Bl * mat_bytes < L2_BYTES // 8
    if small:
        # Few, small matrices (cfg1): the steps are captured in one CUDA graph
        # (no host launch gaps between them) with an L2 flush -- a write of
        # 2x L2 -- before every step; only the expm part of each step is
        # timed, by CUDA events recorded inside the graph.
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
        evs = [(torch.cuda.Event(enable_timing=True, external=True),
                torch.cuda.Event(enable_timing=True, external=True))
               for _ in range(args.steps)]
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            gs = torch.cuda.current_stream(dev)
            for i in range(args.steps):
                flush.fill_(float(i))
                evs[i][0].record(gs)
                mx.expm_batched(ins[i % pairs], outs[i % pairs], sel, accuracy=mx.Accuracy(cfg.accuracy),
                                rounding=rounding, stream=gs, family=mx.Family(fam))
                evs[i][1].record(gs)
        launches = mx.launch_count() - launches0
        graph.replay()  # warm the graph
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            graph.replay()
            torch.cuda.synchronize()
        ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    else:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            ev0.record(stream)
            for i in range(args.steps):
                step(i)
            ev1.record(stream)
            torch.cuda.synchronize()
        launches = mx.launch_count() - launches0
        ms = ev0.elapsed_time(ev1)
    if world > 1:
        ms = max_over_ranks(ms, dev)
        dist.barrier()
    ms_step = ms / args.steps
    value = total / (ms_step * 1e-3)

    # ---- e2e through the host C-ABI call (pinned buffers) ----
    h_in = torch.from_numpy(a_host).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    for _ in range(2):
        mx.expm_batched_host(h_in, h_out, accuracy=mx.Accuracy(cfg.accuracy), rounding=rounding,
                             family=mx.Family(fam))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        mx.expm_batched_host(h_in, h_out, accuracy=mx.Accuracy(cfg.accuracy), rounding=rounding,
                             family=mx.Family(fam))
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    e2e_how = "mexp_expm_batched_host, pinned host buffers, wall clock"
    # A single double matrix under the TaylorNew family (cfg1): the reference's
    # caller makes one mexp::expm call per matrix from C++, so the per-call
    # time is taken natively (bin/call_latency: the C++ drop-in on a host
    # DenseMatrix, 2000 calls) instead of through Python's ctypes overhead.
    native = os.path.join(ROOT, "bin", "call_latency")
    if Bl == 1 and cfg.dtype == "f64" and fam == 0 and rounding == mx.ROUND_AUTO and os.path.exists(native):
        import subprocess
        import tempfile
        with tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as tf:
            a_host[0].astype("<f8").tofile(tf.name)
        try:
            r = subprocess.run([native, tf.name, str(n), "2000"], capture_output=True, text=True, timeout=120)
            e2e_s = json.loads(r.stdout.strip().splitlines()[-1])["us_per_call"] * 1e-6
            e2e_how = ("mexp::expm (C++ drop-in, expm.hpp:37) on a host DenseMatrix, 2000 calls timed "
                       "natively by bin/call_latency")
        except Exception as exc:  # keep the Python-timed value
            e2e_how += f" (native timing unavailable: {exc})"
        finally:
            os.unlink(tf.name)
    if world > 1:
        e2e_s = max_over_ranks(e2e_s, dev)
    e2e_value = total / e2e_s

    # ---- gather of the results to rank 0 (NCCL), timed separately ----
    gather = None
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
        g0 = time.perf_counter()
        counts = [shard_range(r, world, B, weak=not args.strong).count for r in range(world)]
        gathered = gather_to_root(outs[0], counts)
        torch.cuda.synchronize()
        del gathered
        gather = {"ms": 1e3 * (time.perf_counter() - g0),
                  "bytes_to_root": (sum(counts) - counts[0]) * mat_bytes,
                  "how": "torch.distributed.gather (NCCL)"}

    if rank == 0:
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
                               f"{flops / 1e9:.2f} GFLOP (sum 2 n^3 (pi_m + s)) per step")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None,
            "dtype": cfg.dtype, "data": "synthetic (seeded, counter-based; see workloads.py)",
            "config": {"workload": args.config, "description": cfg.description, "n": n,
                       "batch_per_rank": Bl, "global_batch": total, "rounding": args.rounding,
                       "family": args.family,
                       "parallelism": f"matrix-sharded x{world}",
                       "l2": (f"L2 flushed before every step (write of {2 * L2_BYTES >> 20} MiB); "
                              f"steps captured in one CUDA graph, expm part timed by in-graph events"
                              if small else
                              f"inputs larger than L2 ({pairs} x {2 * Bl * mat_bytes / 2**20:.0f} MiB "
                              f"in+out, alternating buffers)")},
            "effective_tflops": tflops,
            "compute_peak": {"tflops": peakc, "source": peakc_src, "frac": tflops / peakc},
            "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": peaks["hbm_gbs"],
                    "frac": hbm_gbs / peaks["hbm_gbs"]},
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": Bl * mat_bytes,
                    "d2h_bytes_per_step": Bl * mat_bytes + 16 * Bl,
                    "how": e2e_how},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if gather:
            line["gather"] = gather
        if not args.no_cpu_baseline and world == 1:
            cores = host_cores()
            per = per_worker_sample(args.config)
            rate, done, wall = cpu_reference_rate(args.config, per, cores, family=fam)
            line["cpu_baseline"] = {
                "value": rate, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"{done} matrices of {args.config} ({per} per worker process, "
                          f"OMP_NUM_THREADS=1), oracle/_ref = unmodified mexp library",
                "cpu": cpu_model()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
