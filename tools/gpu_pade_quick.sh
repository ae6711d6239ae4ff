#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pade.py -m gpu -q -x > gpurun_out/pytest_pade.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pade.log
timeout 300 python bench.py --steps 50 --warmup 5 --family pade --no-cpu-baseline > gpurun_out/fam_cfg2_pade.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --config cfg3 --family pade --no-cpu-baseline > gpurun_out/fam_cfg3_pade.log 2>&1
