#!/bin/bash
# A/B of kernel variants selected by environment settings: one T-blocked C2 launch under
# ncu at locked base clocks (cycles per launch, no power-cap noise), then a short bench line.
# usage: CFGS="ST_JACOBI_TB4_ROWS=0 ST_JACOBI_TB4_ROWS=512,ST_JACOBI_TB4_EDGE_COST=200" bash tools/exp/gpu_ab.sh
OUT=gpurun_out/ab; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
if [ -n "${TESTS:-}" ]; then timeout 900 python -m pytest $TESTS -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log; fi
NCU=/usr/local/cuda/bin/ncu
for cfg in $CFGS; do
  envs=$(echo $cfg | tr ',' ' ')
  env $envs timeout 300 $NCU --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__inst_executed.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio \
    -k regex:${KREG:-jacobi2d_tb4} -s ${SKIP:-1} -c 1 --csv python tools/prof_kernels.py --sweeps ${SWEEPS:-20} --tblock ${TB:-10} --apps 0 > $OUT/ncu_$cfg.csv 2> $OUT/ncu_$cfg.err
  m=$(python - "$OUT/ncu_$cfg.csv" <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; out={}
for r in rows[1:]:
    out[r[h.index("Metric Name")]]=r[h.index("Metric Value")]
print(" ".join(f"{k.split('__')[-1][:40]}={v}" for k,v in out.items()))
PY
)
  echo "$cfg ncu: $m"
  if [ -z "${NOBENCH:-}" ]; then
    env $envs timeout 300 python bench.py --steps 3 --warmup 3 --tblock ${TB:-10} --no-e2e --no-cpu --no-scaling --no-pw --no-j3 --no-gs --no-generic > $OUT/b_$cfg.json 2> $OUT/b_$cfg.err
    echo "$cfg bench: $(python -c "import json;d=json.load(open('$OUT/b_$cfg.json'));print(d['value'],d['roofline']['ms_per_pass'],d['clocks']['sm_mhz'],d['clocks']['power_w_median'])" 2>&1 | tail -1)"
  fi
done
