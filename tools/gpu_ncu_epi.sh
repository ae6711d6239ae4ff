#!/bin/bash
# ncu --set full of cfg4's epilogue GEMMs (EPI_T18_B = <3>, EPI_AL = <2>)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/profile_kernel.py cfg4 auto 1 > gpurun_out/p4.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -s 2 -c 1 -o gpurun_out/prof_cfg4_epi3 -f python tools/profile_kernel.py cfg4 auto 1 > gpurun_out/ncu_epi3.log 2>&1
