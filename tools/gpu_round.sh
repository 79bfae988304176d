#!/bin/bash
# One GPU measurement round (run under gpurun from the repo root).
# usage: tools/gpu_round.sh TAG [what...]   what in: build tests smoke bench launches ncu sanitize
set -u
TAG=${1:-r}; shift || true
WHAT=${*:-"build tests smoke bench launches ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
for w in $WHAT; do
  case $w in
    build) make -j8 all > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; } ;;
    tests) timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $OUT/smoke.log ;;
    bench) timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json; tail -3 $OUT/bench.err ;;
    launches) timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $OUT/launches.csv \
        python bench.py --steps 1 --warmup 3 --pw-apps 4 --j3-sweeps 10 --gs-sweeps 10 --no-e2e --no-cpu > $OUT/launches_bench.log 2>&1; echo "launches rc=$?" ;;
    ncu) timeout 900 $NCU --set full --clock-control none --import-source on -k regex:'jacobi2d_tb|jacobi2d_stream|pw_advect3d_kernel|jacobi3d_kernel|jacobi3d_t2_kernel|gauss_seidel2d|stencil2d_kernel' -s ${NCU_SKIP:-1} -c 10 \
        -o $OUT/prof python tools/prof_kernels.py --sweeps ${NCU_SWEEPS:-4} --tblock ${NCU_TBLOCK:-1} --apps 3 > $OUT/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $OUT/ncu.log ;;
    sanitize) echo "compute-sanitizer is closed on this pool (r02f); the last sanitizer results are profiles/r02d_sanitize.txt"; continue; for tool in memcheck racecheck synccheck; do
        RC=""; [ $tool = racecheck ] && RC="ST_GS_MS=0"; timeout 900 env $RC /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > $OUT/sanitize_$tool.log 2>&1
        echo "sanitize $tool rc=$?"; tail -3 $OUT/sanitize_$tool.log; done ;;
  esac
done
# tuning sweeps (quick bench lines, no e2e / cpu legs)
if [ -n "${TUNE:-}" ]; then
  for cfg in $TUNE; do
    env $(echo $cfg | tr ',' ' ') timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu $BENCH_ARGS > $OUT/tune_$cfg.json 2>&1
    echo "$cfg: $(python -c "import json,sys;d=json.load(open('$OUT/tune_$cfg.json'));p=d['pw_advect3d'] or {};j=d.get('jacobi3d') or {};print(d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'],'| pw',p.get('value'),p.get('roofline',{}).get('frac'),'| j3',j.get('value'),j.get('roofline',{}).get('frac'))" 2>&1 | tail -1)"
  done
fi
