#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 120 python tools/profile_kernel.py cfg2 auto 2 pade > gpurun_out/pade_try.log 2>&1; echo "try exit $?" >> gpurun_out/pade_try.log
timeout 900 python -m pytest tests/test_gpu_pade.py tests/test_cli.py -m gpu -q -x > gpurun_out/pytest_pade.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pade.log
for m in auto reference; do
  timeout 300 python bench.py --steps 50 --warmup 5 --family pade --rounding $m --no-cpu-baseline > gpurun_out/fam_cfg2_pade_$m.log 2>&1
done
MEXP_PADE8_GENERIC=1 timeout 300 python bench.py --steps 50 --warmup 5 --family pade --no-cpu-baseline > gpurun_out/fam_cfg2_pade_generic.log 2>&1
