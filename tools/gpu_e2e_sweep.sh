#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for st in 2 3 4 6 8; do for mb in 4 8 16 32; do
  MEXP_HOST_STREAMS=$st MEXP_HOST_CHUNK_MB=$mb timeout 120 python tools/e2e_sweep.py >> gpurun_out/e2e_sweep.txt 2>&1
done; done
timeout 120 python tools/e2e_probe.py > gpurun_out/e2e_probe.json 2>&1
