#!/bin/bash
# Every family x rounding on every config (device time, e2e, CPU reference for the
# auto lines of cfg2/cfg3); one JSON line per log under gpurun_out/fam_*.log
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for f in taylor-new taylor-ps pade; do
  for m in auto reference fast; do
    [ "$f" = pade ] && [ "$m" = fast ] && continue
    cpu="--no-cpu-baseline"; [ "$m" = auto ] && [ "$f" != taylor-new ] && cpu=""
    timeout 300 python bench.py --steps 100 --warmup 5 --family $f --rounding $m $cpu > gpurun_out/fam_cfg2_${f}_$m.log 2>&1
  done
  cpu=""; [ "$f" = taylor-new ] && cpu="--no-cpu-baseline"
  timeout 300 python bench.py --steps 20 --warmup 3 --config cfg3 --family $f $cpu > gpurun_out/fam_cfg3_$f.log 2>&1
  timeout 600 python bench.py --steps 5 --warmup 3 --config cfg4 --family $f --no-cpu-baseline > gpurun_out/fam_cfg4_$f.log 2>&1
  timeout 900 python bench.py --steps 2 --warmup 3 --e2e-steps 2 --config cfg5 --family $f --no-cpu-baseline > gpurun_out/fam_cfg5_$f.log 2>&1
done
for c in cfg4 cfg5; do
  timeout 900 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --config $c --rounding reference --no-cpu-baseline > gpurun_out/fam_${c}_taylor-new_reference.log 2>&1
done
echo done
