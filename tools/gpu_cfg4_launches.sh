#!/bin/bash
# launch list (per-kernel device time) of one cfg4 and one cfg5 expm call
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/profile_kernel.py cfg4 auto 1 > gpurun_out/p4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python tools/profile_kernel.py cfg4 auto 1 > gpurun_out/ncu4.log 2>&1
python tools/profile_kernel.py cfg5 auto 1 > gpurun_out/p5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python tools/profile_kernel.py cfg5 auto 1 > gpurun_out/ncu5.log 2>&1
