#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/profile_kernel.py cfg2 auto 2 pade > gpurun_out/pade_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:expm_small -s 1 -c 1 -o gpurun_out/prof_pade8 -f python tools/profile_kernel.py cfg2 auto 2 pade > gpurun_out/ncu_pade8.log 2>&1
