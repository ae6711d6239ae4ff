#!/bin/bash
# ncu --set full of the 8x8 kernel in REFERENCE rounding (all products k-ordered exact)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/profile_kernel.py cfg2 reference 2 > gpurun_out/p2r.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:expm8 -s 1 -c 1 -o gpurun_out/prof_cfg2_ref -f python tools/profile_kernel.py cfg2 reference 2 > gpurun_out/ncu_cfg2_ref.log 2>&1
