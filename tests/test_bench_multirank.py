"""bench.py's multi-rank path on CPU (no GPU): `--gpus 2` re-launches itself
under torch.distributed.run, splits the config's batch by matrix across the
two ranks, gathers e^A and the selection records to rank 0
with grouped send/recv and prints one JSON line with n_gpus = 2. The dry run
(gloo, per-rank compute replaced by a copy) checks exactly that plumbing; the
gathered result must equal the whole batch.

Also: the reference arm prints the same `config` object as our arm, so the
two lines describe the same workload.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_line(stdout):
    lines = [ln for ln in stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus,batch", [(2, 1001), (3, 10)])
def test_bench_dry_run_ranks_split_gather(gpus, batch):
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
                        "--dry-run", "--dry-batch", str(batch), "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _json_line(r.stdout)
    assert line["n_gpus"] == gpus and line["dry_run"] is True and line["value"] is None
    assert line["scaling"] == "strong"
    assert line["config"]["global_batch"] == batch
    ranks = line["ranks"]
    assert [x["rank"] for x in ranks] == list(range(gpus))
    # contiguous split, the first batch % gpus ranks one matrix more
    base, extra = divmod(batch, gpus)
    pos = 0
    for x in ranks:
        assert x["b0"] == pos and x["count"] == base + (x["rank"] < extra)
        pos += x["count"]
    assert pos == batch
    g = line["gather"]
    assert g["verified_bitwise_vs_one_gpu"] is True
    assert g["bytes_to_root"] == (batch - ranks[0]["count"]) * (8 * 8 * 8 + 16)
    # every rank reported itself on stderr
    for k in range(gpus):
        assert f"bench.py rank {k}/{gpus}: shard" in r.stderr


def test_reference_arm_config_matches_ours():
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "cfg2", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _json_line(r.stdout)
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert "full 262144-matrix batch" in line["cpu_baseline"]["sample"]
    args = argparse.Namespace(config="cfg2", weak=False, rounding="auto", family="taylor-new")
    assert line["config"] == bench.workload_config(args, 1, 262144)


def test_bench_dry_run_single_matrix_config_runs_replicas():
    """cfg1 / cfg5 are one matrix: under N ranks each rank runs a replica
    (replicas only), reported as weak scaling."""
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                        "--config", "cfg1", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _json_line(r.stdout)
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert [x["count"] for x in line["ranks"]] == [1, 1]
    assert line["config"]["global_batch"] == 2
