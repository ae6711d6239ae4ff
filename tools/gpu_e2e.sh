#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/pcie_bw.py 128 > gpurun_out/pcie.json 2>&1
for mb in 4 8 16 32 64; do
  MEXP_HOST_CHUNK_MB=$mb timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/e2e_$mb.log 2>&1
done
echo done
