#!/bin/bash
# The maintained GPU-box driver (run under gpurun from the repo root):
#
#   tools/gpu.sh tests                 pytest -m gpu + smoke()
#   tools/gpu.sh bench CFG [ROUND..]   bench.py lines for a config (default: auto)
#   tools/gpu.sh cfg2                  cfg2 in auto / fast / reference rounding
#   tools/gpu.sh evidence              tests, smoke, every config's bench line,
#                                      the reference arm, launch lists, ncu
#   tools/gpu.sh launches CFG          ncu launch list (gpu__time_duration) of bench.py
#   tools/gpu.sh ncu CFG [ROUND]       ncu --set full of the config's top kernel
#   tools/gpu.sh sanitize              compute-sanitizer memcheck/racecheck/synccheck/initcheck
#   tools/gpu.sh e2e                   e2e variants of the host pipeline (cfg2, cfg3)
#   tools/gpu.sh envbench CFG R ENV..  one bench line per environment string (knob A/B)
#
# Everything lands in gpurun_out/ (scratch); summaries worth keeping are
# copied to profiles/ by hand.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}" || exit 1
mkdir -p gpurun_out
out=gpurun_out

line() {  # the JSON line of a bench log, summarised
    python - "$1" <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
r = d.get("roofline", {})
print(f"{sys.argv[1]}: {d['ms_per_step'] * 1e3:.1f} us/step  {d['value']:.4g} {d['unit']}  "
      f"{r.get('bound')} frac {r.get('frac', 0):.3f}  e2e {d['e2e']['value']:.4g}  "
      f"clk {d.get('clocks', {}).get('sm_mhz')}")
PY
}

case "$1" in
tests)
    timeout 1800 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
    tail -3 $out/pytest_gpu.log
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
    tail -2 $out/smoke.log ;;
bench)
    cfg=${2:-cfg2}; shift 2; rounds=${*:-auto}
    for r in $rounds; do
        timeout 1200 python bench.py --config $cfg --rounding $r --no-cpu-baseline --e2e-steps 3 > $out/bench_${cfg}_$r.log 2>&1
        line $out/bench_${cfg}_$r.log
    done ;;
cfg2)
    for r in auto fast reference; do
        python bench.py --rounding $r --no-cpu-baseline --e2e-steps 3 > $out/bench_cfg2_$r.log 2>&1
        line $out/bench_cfg2_$r.log
    done ;;
evidence)
    "$0" tests
    [ -x tools/fp64_peak ] && ./tools/fp64_peak > $out/fp64_peak.json 2>&1
    timeout 900 python bench.py > $out/bench_default.log 2>&1; line $out/bench_default.log
    timeout 600 python bench.py --impl reference > $out/bench_reference_arm.log 2>&1
    for c in cfg1 cfg3 cfg4 cfg5; do
        timeout 1200 python bench.py --config $c > $out/bench_$c.log 2>&1; line $out/bench_$c.log
    done
    for c in cfg2 cfg3 cfg4 cfg5; do "$0" launches $c; done
    for c in cfg2 cfg3 cfg4 cfg5; do "$0" ncu $c; done
    "$0" ncu cfg2 fast
    "$0" ncu cfg2 reference ;;
envbench)  # envbench CFG ROUNDING "VAR=x VAR2=y" ... : one bench line per environment
    cfg=$2; r=$3; shift 3
    for e in "$@"; do
        tag=$(echo "$e" | tr ' =' '_-')
        env $e timeout 600 python bench.py --config $cfg --rounding $r --no-cpu-baseline --e2e-steps 1 \
            > $out/envbench_${cfg}_${r}_$tag.log 2>&1
        echo -n "[$e] "; line $out/envbench_${cfg}_${r}_$tag.log
    done ;;
launches)
    cfg=${2:-cfg2}
    python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $out/plain_$cfg.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file $out/launches_$cfg.csv python bench.py --config $cfg --steps 2 --warmup 3 \
        --no-cpu-baseline --e2e-steps 1 > $out/ncu_launches_$cfg.log 2>&1
    echo "launches_$cfg.csv: $(grep -c gpu__time_duration $out/launches_$cfg.csv) rows" ;;
ncu)
    cfg=${2:-cfg2}; r=${3:-auto}
    case $cfg in cfg1) k=regex:cluster;; cfg2) k=regex:expm8_;; cfg3) k=regex:expm32_pairs;;
                 *) k=regex:gemm_dmma;; esac
    python tools/profile_kernel.py $cfg $r 2 > $out/prof_plain_$cfg.log 2>&1 && \
    timeout 900 ncu --set full --import-source on --clock-control none -k $k -s 1 -c 1 \
        -o $out/prof_${cfg}_$r -f python tools/profile_kernel.py $cfg $r 2 > $out/ncu_${cfg}_$r.log 2>&1
    python tools/ncu_summary.py $out/prof_${cfg}_$r.ncu-rep > $out/ncu_${cfg}_$r.txt 2>&1
    head -5 $out/ncu_${cfg}_$r.txt ;;
sanitize)
    for t in memcheck racecheck synccheck initcheck; do
        timeout 1200 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_workload.py \
            > $out/sanitize_$t.log 2>&1
        echo "$t exit $?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/sanitize_$t.log | tail -1)"
    done ;;
e2e)
    for zc in 0 1; do
        MEXP_HOST_OUT_ZC=$zc python bench.py --steps 50 --no-cpu-baseline --e2e-steps 20 > $out/e2e_cfg2_zc$zc.log 2>&1
        line $out/e2e_cfg2_zc$zc.log
        MEXP_HOST_OUT_ZC=$zc python bench.py --config cfg3 --steps 20 --no-cpu-baseline --e2e-steps 10 > $out/e2e_cfg3_zc$zc.log 2>&1
        line $out/e2e_cfg3_zc$zc.log
    done ;;
*)
    sed -n 2,17p "$0"; exit 2 ;;
esac
