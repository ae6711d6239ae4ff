#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in 0 4 5; do
  for m in auto fast; do
    MEXP_N8_VARIANT=$v timeout 300 python bench.py --steps 200 --warmup 10 --rounding $m --no-cpu-baseline --e2e-steps 10 > gpurun_out/bench_v${v}_$m.log 2>&1
  done
done
echo done
