#!/bin/bash
# fp32 tests + cfg3 bench (quick iteration)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "fp32 or cfg3 or f32" -s > gpurun_out/pytest_f32.log 2>&1; echo "exit $?" >> gpurun_out/pytest_f32.log
timeout 600 python bench.py --config cfg3 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_cfg3.log
