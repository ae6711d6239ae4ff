#!/bin/bash
# Variant sweep: each variants/*.so in place of the library, then
#   bench.py --config $1 --steps $2 --warmup 3 $3
# (device time only), twice in alternating order to expose box noise.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
cfg=${1:-cfg2}; steps=${2:-50}; extra=${3:-}
cp paper_1710_10989_b200/_lib/libmexp_b200.so /tmp/lib_keep.so
for pass in 1 2; do
for v in variants/*.so; do
  n=$(basename $v .so)
  cp $v paper_1710_10989_b200/_lib/libmexp_b200.so
  timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 $extra > gpurun_out/var_${cfg}_${n}_$pass.log 2>&1
  echo "$cfg $n pass$pass $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/var_${cfg}_${n}_$pass.log)" >> gpurun_out/variants.txt
done; done
cp /tmp/lib_keep.so paper_1710_10989_b200/_lib/libmexp_b200.so
