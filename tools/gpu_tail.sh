#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for k in 0 2 3 4; do
  MEXP_FAST_TAIL=$k timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "cfg2_full_batch and auto" > gpurun_out/tail_$k.log 2>&1
  MEXP_FAST_TAIL=$k timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 10 > gpurun_out/bench_tail_$k.log 2>&1
done
echo done
