#!/bin/bash
# Standard GPU iteration: tests, benches, optional ncu of one config.
#   bash tools/gpu_cycle.sh "<configs>" "<ncu config list>"
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CONFIGS=${1:-cfg2}
NCU=${2:-}
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for c in $CONFIGS; do
  if [ "$c" = "cfg2" ]; then
    for m in auto fast reference; do
      timeout 300 python bench.py --steps 200 --warmup 10 --rounding $m --no-cpu-baseline > gpurun_out/bench_cfg2_$m.log 2>&1
    done
  else
    timeout 600 python bench.py --steps 20 --warmup 3 --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  fi
done
for c in $NCU; do
  python tools/profile_kernel.py $c auto 3 > gpurun_out/prof_plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:expm -s 1 -c 1 -o gpurun_out/prof_$c -f python tools/profile_kernel.py $c auto 3 > gpurun_out/ncu_$c.log 2>&1
done
echo done
