#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 --config cfg4 --family pade --no-cpu-baseline > gpurun_out/fam_cfg4_pade.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --config cfg5 --family pade --no-cpu-baseline > gpurun_out/fam_cfg5_pade.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --config cfg5 --family taylor-ps --no-cpu-baseline > gpurun_out/fam_cfg5_taylor-ps.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
