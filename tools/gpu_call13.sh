#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 20 > gpurun_out/e2e_pinned.log 2>&1
for i in 1 2; do timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/cfg4_run$i.log 2>&1; done
python tools/profile_kernel.py cfg4 auto 2 > gpurun_out/p4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python tools/profile_kernel.py cfg4 auto 2 > gpurun_out/ncu_l4.log 2>&1
echo done
