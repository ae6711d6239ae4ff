#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ps.py tests/test_gpu_pade.py -m gpu -q -x > gpurun_out/pytest_q.log 2>&1; echo "exit $?" >> gpurun_out/pytest_q.log
for m in auto fast reference; do
  timeout 300 python bench.py --steps 200 --warmup 10 --rounding $m --no-cpu-baseline > gpurun_out/bench_cfg2_$m.log 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 3 --config cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1
