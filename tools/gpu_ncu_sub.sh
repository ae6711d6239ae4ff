#!/bin/bash
# ncu --set full of one Pade LU/solve trailing-update launch (gemm_sub_kernel) on cfg4
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/profile_kernel.py cfg4 auto 1 pade > gpurun_out/p4p.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_sub -s ${1:-10} -c 1 -o gpurun_out/prof_sub -f python tools/profile_kernel.py cfg4 auto 1 pade > gpurun_out/ncu_sub.log 2>&1
