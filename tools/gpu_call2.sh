#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for m in auto fast reference; do
  timeout 300 python bench.py --steps 100 --warmup 10 --rounding $m --no-cpu-baseline > gpurun_out/bench_cfg2_$m.log 2>&1
done
timeout 300 python bench.py --steps 50 --warmup 5 --config cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1
python tools/profile_kernel.py cfg2 auto 3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:expm_small -s 1 -c 1 -o gpurun_out/prof_cfg2_auto -f python tools/profile_kernel.py cfg2 auto 3 > gpurun_out/ncu_cfg2.log 2>&1
python tools/profile_kernel.py cfg3 auto 3 > gpurun_out/prof_plain3.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:expm_small -s 1 -c 1 -o gpurun_out/prof_cfg3 -f python tools/profile_kernel.py cfg3 auto 3 > gpurun_out/ncu_cfg3.log 2>&1
echo done
