#!/bin/bash
# launch list of one Pade cfg4 expm call
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/profile_kernel.py cfg4 auto 1 pade > gpurun_out/p4p.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_pade.csv python tools/profile_kernel.py cfg4 auto 1 pade > gpurun_out/ncu4p.log 2>&1
