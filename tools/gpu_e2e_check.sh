#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ps.py -m gpu -q -x > gpurun_out/pytest_parity.log 2>&1; echo "exit $?" >> gpurun_out/pytest_parity.log
for mb in 8 16 32; do MEXP_HOST_CHUNK_MB=$mb timeout 120 python tools/e2e_sweep.py >> gpurun_out/e2e_sweep.txt 2>&1; done
MEXP_HOST_PIPE=streams timeout 120 python tools/e2e_sweep.py >> gpurun_out/e2e_sweep.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_default.log 2>&1
