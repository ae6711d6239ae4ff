#!/bin/bash
# Evidence run: tests, smoke, benches for every config, ncu launch list of the
# default bench, ncu --set full of the top kernel of cfg2/cfg3/cfg4.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
[ -x tools/fp64_peak ] && ./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_reference_arm.log 2>&1
for c in cfg1 cfg3; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/bench_$c.log 2>&1; done
for c in cfg4 cfg5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launches.log 2>&1
python tools/profile_kernel.py cfg2 auto 2 > gpurun_out/p2.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:expm8 -s 1 -c 1 -o gpurun_out/prof_cfg2_auto -f python tools/profile_kernel.py cfg2 auto 2 > gpurun_out/ncu_cfg2.log 2>&1
python tools/profile_kernel.py cfg1 auto 3 > gpurun_out/p1.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cluster -s 1 -c 1 -o gpurun_out/prof_cfg1 -f python tools/profile_kernel.py cfg1 auto 3 > gpurun_out/ncu_cfg1.log 2>&1
python tools/profile_kernel.py cfg3 auto 2 > gpurun_out/p3.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:expm_small -s 1 -c 1 -o gpurun_out/prof_cfg3 -f python tools/profile_kernel.py cfg3 auto 2 > gpurun_out/ncu_cfg3.log 2>&1
python tools/profile_kernel.py cfg4 auto 1 > gpurun_out/p4.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -s 0 -c 1 -o gpurun_out/prof_cfg4 -f python tools/profile_kernel.py cfg4 auto 1 > gpurun_out/ncu_cfg4.log 2>&1
echo done
