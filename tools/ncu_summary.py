"""Summarise an ncu --set full report for profiles/.

    python tools/ncu_summary.py gpurun_out/prof_cfg2.ncu-rep "cfg2 auto" > profiles/...txt
Prints duration, DRAM traffic, pipe utilisations, occupancy, stall mix and the
opcode mix per launch; with --traffic KEY also merges {KEY: dram bytes per
launch} into profiles/traffic.json (bench.py's roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else rep
    traffic_key = None
    if "--traffic" in sys.argv:
        traffic_key = sys.argv[sys.argv.index("--traffic") + 1]
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, vals = rows[0], rows[2]
    d = dict(zip(hdr, vals))
    name = d.get("Kernel Name", "?")

    def f(k):
        try:
            return float(d[k])
        except (KeyError, ValueError):
            return float("nan")

    dur_ns = f("gpu__time_duration.sum")
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    # ncu reports these in the unit of its header row
    units = dict(zip(hdr, rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
    wr *= scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
    tunit = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9,
             "us": 1e-6, "ms": 1e-3, "s": 1}
    dur = dur_ns * tunit.get(units.get("gpu__time_duration.sum", "nsecond"), 1e-9)
    print(f"# ncu --set full summary: {label}")
    print(f"kernel: {name}")
    print(f"grid {d.get('launch__grid_size')} x block {d.get('launch__block_size')}, "
          f"registers/thread {d.get('launch__registers_per_thread')}, "
          f"SM clock {d.get('smsp__cycles_elapsed.avg.per_second', '?')}")
    print(f"duration: {dur * 1e6:.1f} us (under ncu, --clock-control none)")
    print(f"DRAM: read {rd / 1e6:.1f} MB, write {wr / 1e6:.1f} MB, "
          f"total {(rd + wr) / 1e6:.1f} MB -> {(rd + wr) / dur / 1e9:.0f} GB/s")
    for k in ["sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__throughput.avg.pct_of_peak_sustained_elapsed",
              "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]:
        if k in d:
            print(f"{k}: {d[k]}")
    items = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                items.append((float(v), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in items) or 1
    print("stalls: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for v, k in sorted(items, reverse=True)[:8]))
    src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv",
                                          "--print-source", "sass"))))
    if len(src) > 2:
        h = src[1]
        ix, isrc = h.index("Instructions Executed"), h.index("Source")
        cnt = collections.Counter()
        for r in src[2:]:
            try:
                n = int(r[ix] or 0)
            except (ValueError, IndexError):
                continue
            toks = r[isrc].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            cnt[op.split(".")[0]] += n
        total = sum(cnt.values())
        print(f"warp instructions executed: {total}")
        print("opcode mix: " + ", ".join(f"{op} {100 * n / total:.1f}%" for op, n in cnt.most_common(16)))
    if traffic_key:
        p = os.path.join(ROOT, "profiles", "traffic.json")
        t = json.load(open(p)) if os.path.exists(p) else {}
        t[traffic_key] = rd + wr
        json.dump(t, open(p, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
