#!/bin/bash
# A/B of two prebuilt libraries (build_ab/libstencil_{base,new}.so, no rebuild on the box):
# locked-clock ncu time of one launch of $KREG, then a short bench line, alternating.
# usage: KREG=jacobi3d_t2 BENCH_ARGS="--no-pw --no-gs ..." PROF_ARGS="..." TESTS="..." bash tools/exp/gpu_ablib.sh
OUT=gpurun_out/ablib; mkdir -p $OUT
LIB=paper_2310_01882_b200/libstencil.so
NCU=/usr/local/cuda/bin/ncu
cp build_ab/libstencil_new.so $LIB
if [ -n "${TESTS:-}" ]; then timeout 900 python -m pytest $TESTS -x -q > $OUT/pytest.log 2>&1; echo "pytest(new) rc=$?"; tail -1 $OUT/pytest.log; fi
for rep in 1 2; do for v in base new; do
  cp build_ab/libstencil_$v.so $LIB
  t=$(timeout 300 $NCU --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__inst_executed.sum -k regex:$KREG -s ${SKIP:-0} -c 1 --csv \
      python tools/prof_kernels.py ${PROF_ARGS:---sweeps 4 --tblock 1 --apps 0} 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]; h=rows[0]
print(' '.join(r[h.index('Metric Name')].split('__')[-1]+'='+r[h.index('Metric Value')] for r in rows[1:]))")
  b=$(timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-scaling $BENCH_ARGS 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k='${LEG:-jacobi3d}'; x=d.get(k) or d
print(x['value'], x['roofline']['frac'], d['clocks']['sm_mhz'])")
  echo "$rep $v | ncu: $t | bench: $b"
done; done
