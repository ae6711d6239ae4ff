#!/bin/bash
# cfg2 iteration: parity tests for the 8x8 path + benches in the three modes
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -s -k "cfg2 or golden or edge or padded or device or kats" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for m in auto fast reference; do
  timeout 300 python bench.py --steps 200 --warmup 10 --rounding $m --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_cfg2_$m.log 2>&1
done
if [ -n "$1" ]; then
python tools/profile_kernel.py cfg2 auto 3 > gpurun_out/p2.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:expm8 -s 1 -c 1 -o gpurun_out/prof_cfg2 -f python tools/profile_kernel.py cfg2 auto 3 > gpurun_out/ncu_cfg2.log 2>&1
fi
echo done
