#!/bin/bash
# cfg3 variant sweep: each variants/*.so in place of the library, cfg3 bench;
# then ncu --set full of the kernel for the variant named in $1.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
cp paper_1710_10989_b200/_lib/libmexp_b200.so /tmp/lib_keep.so
for v in variants/*.so; do
  n=$(basename $v .so)
  cp $v paper_1710_10989_b200/_lib/libmexp_b200.so
  timeout 300 python bench.py --config cfg3 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg3_$n.log 2>&1
done
if [ -n "$1" ]; then
  cp variants/$1.so paper_1710_10989_b200/_lib/libmexp_b200.so
  python tools/profile_kernel.py cfg3 auto 2 > gpurun_out/p3.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:expm_small -s 1 -c 1 -o gpurun_out/prof_cfg3_$1 -f python tools/profile_kernel.py cfg3 auto 2 > gpurun_out/ncu_cfg3.log 2>&1
fi
cp /tmp/lib_keep.so paper_1710_10989_b200/_lib/libmexp_b200.so
