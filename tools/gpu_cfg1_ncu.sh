#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/profile_kernel.py cfg1 auto 5 > gpurun_out/cfg1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/profile_kernel.py cfg1 auto 5 > gpurun_out/cfg1_launches.csv 2>&1
MEXP_CLUSTER_MAX=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/profile_kernel.py cfg1 auto 5 > gpurun_out/cfg1_launches_cta.csv 2>&1
ncu --set full --import-source on --clock-control none -k regex:cluster -s 2 -c 1 -o gpurun_out/prof_cfg1 -f python tools/profile_kernel.py cfg1 auto 4 > gpurun_out/ncu_cfg1.log 2>&1
