#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/profile_kernel.py cfg2 fast 2 > gpurun_out/p2f.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:expm8 -s 1 -c 1 -o gpurun_out/prof_cfg2_fast -f python tools/profile_kernel.py cfg2 fast 2 > gpurun_out/ncu_cfg2_fast.log 2>&1
