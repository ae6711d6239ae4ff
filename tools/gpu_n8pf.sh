#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in 0 8 0 8; do for m in auto fast; do
  MEXP_N8_VARIANT=$v timeout 300 python bench.py --steps 300 --warmup 10 --rounding $m --no-cpu-baseline --e2e-steps 1 > gpurun_out/n8v_${v}_$m.log 2>&1
  echo "variant $v $m $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/n8v_${v}_$m.log)" >> gpurun_out/n8pf.txt
done; done
MEXP_N8_VARIANT=8 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cfg2 or golden" > gpurun_out/pytest_pf.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pf.log
