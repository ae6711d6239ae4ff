#!/bin/bash
# first GPU call: tests, smoke, bench, fp64 peak
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 120 ./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 300 python bench.py --steps 100 --warmup 10 --rounding reference --no-cpu-baseline > gpurun_out/bench_ref.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 10 --rounding fast --no-cpu-baseline > gpurun_out/bench_fast.log 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
