#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_large.py tests/test_cpp_dropin.py tests/test_gpu_ps.py -m gpu -q -x > gpurun_out/pytest_large.log 2>&1; echo "exit $?" >> gpurun_out/pytest_large.log
timeout 600 python bench.py --steps 3 --warmup 1 --config cfg4 --rounding reference --no-cpu-baseline > gpurun_out/bench_cfg4_ref.log 2>&1
timeout 900 python bench.py --steps 1 --warmup 1 --config cfg5 --rounding reference --no-cpu-baseline > gpurun_out/bench_cfg5_ref.log 2>&1
