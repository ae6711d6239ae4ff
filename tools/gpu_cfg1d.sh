#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 120 python tools/profile_kernel.py cfg1 auto 3 > gpurun_out/cfg1_try.log 2>&1; echo "try exit $?" >> gpurun_out/cfg1_try.log
if grep -q "try exit 0" gpurun_out/cfg1_try.log; then
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cluster or cfg1 or golden or padded" > gpurun_out/pytest_cfg1.log 2>&1; echo "exit $?" >> gpurun_out/pytest_cfg1.log
  for m in auto reference; do
    timeout 300 python bench.py --config cfg1 --steps 200 --warmup 10 --rounding $m --no-cpu-baseline > gpurun_out/bench_cfg1_$m.log 2>&1
  done
fi
