#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -s -k "cfg2 or golden or edge or padded or cfg3 or large" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for mb in 8 16 32; do
  MEXP_HOST_CHUNK_MB=$mb timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 20 > gpurun_out/e2e_$mb.log 2>&1
done
echo done
