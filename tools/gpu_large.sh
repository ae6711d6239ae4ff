#!/bin/bash
# large-n tests and benches (cfg4, cfg5)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_ps.py tests/test_gpu_pade.py -m gpu -q -x > gpurun_out/pytest_large.log 2>&1; echo "exit $?" >> gpurun_out/pytest_large.log
timeout 600 python bench.py --steps 10 --warmup 3 --config cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --config cfg5 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1
