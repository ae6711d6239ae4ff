cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pade.py tests/test_gpu_ps.py tests/test_cpp_dropin.py -m gpu -x -q -s > gpurun_out/pytest_pade.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pade.log
