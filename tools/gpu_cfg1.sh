#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ps.py -m gpu -q -x > gpurun_out/pytest_cfg1.log 2>&1; echo "exit $?" >> gpurun_out/pytest_cfg1.log
for m in auto reference; do
  timeout 300 python bench.py --config cfg1 --steps 200 --warmup 10 --rounding $m --no-cpu-baseline > gpurun_out/bench_cfg1_$m.log 2>&1
done
MEXP_CLUSTER_MAX=0 timeout 300 python bench.py --config cfg1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_cfg1_nocluster.log 2>&1
