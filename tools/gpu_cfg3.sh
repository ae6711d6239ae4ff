#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -s -k "cfg3 or fp32" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config cfg3 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_cfg3.log 2>&1
if [ -n "$1" ]; then
python tools/profile_kernel.py cfg3 auto 2 > gpurun_out/p3.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:expm_small -s 1 -c 1 -o gpurun_out/prof_cfg3 -f python tools/profile_kernel.py cfg3 auto 2 > gpurun_out/ncu_cfg3.log 2>&1
fi
echo done
