#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -s -k "cfg2 or golden or edge or padded or device" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for v in 0 1 2 3; do
  for m in auto fast; do
    MEXP_N8_VARIANT=$v timeout 300 python bench.py --steps 200 --warmup 10 --rounding $m --no-cpu-baseline > gpurun_out/bench_v${v}_$m.log 2>&1
  done
done
echo done
