#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_pade.py -m gpu -q -x > gpurun_out/pytest_large.log 2>&1; echo "exit $?" >> gpurun_out/pytest_large.log
