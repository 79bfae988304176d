# scratch GPU step (edited per experiment); run under gpurun from the repo root
OUT=gpurun_out/${TAG:-r2e}; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
q() { python -c "import json,sys;d=json.load(open('$1'));print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1; }
tune() {
for cfg in "$@"; do
  env $(echo $cfg | tr ',' ' ') timeout 300 python bench.py --steps 3 --warmup 3 --sweeps 400 --no-e2e --no-cpu --no-pw --no-j3 --no-gs --no-generic > $OUT/t_$cfg$SUF.json 2>$OUT/t_$cfg$SUF.err
  echo "$cfg$SUF: $(q $OUT/t_$cfg$SUF.json)"
done; }
tune ST_JACOBI_TB4_EDGE_COST=220 ST_JACOBI_TB4_EDGE_COST=260 ST_JACOBI_TB4_EDGE_COST=300 ST_JACOBI_TB4_EDGE_COST=360 ST_JACOBI_TB4_EDGE_COST=260,ST_JACOBI_TB4_ROWS=357
