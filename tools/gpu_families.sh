#!/bin/bash
# cfg2 (and cfg3/cfg4 for TaylorPS) throughput of the comparison families
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for f in taylor-ps pade; do
  timeout 300 python bench.py --steps 100 --warmup 5 --family $f > gpurun_out/fam_cfg2_${f}_auto.log 2>&1
  for m in reference fast; do
    timeout 300 python bench.py --steps 100 --warmup 5 --family $f --rounding $m --no-cpu-baseline > gpurun_out/fam_cfg2_${f}_$m.log 2>&1
  done
done
timeout 300 python bench.py --steps 20 --warmup 3 --config cfg3 --family taylor-ps --no-cpu-baseline > gpurun_out/fam_cfg3_taylor-ps.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --config cfg3 --family pade --no-cpu-baseline > gpurun_out/fam_cfg3_pade.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --config cfg4 --family taylor-ps --no-cpu-baseline > gpurun_out/fam_cfg4_taylor-ps.log 2>&1
echo done
