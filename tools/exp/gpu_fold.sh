# sustained C2 bench: power-of-two folding of the level multiplies on/off (alternating, twice)
OUT=gpurun_out/fold; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
q() { python -c "import json,sys;d=json.load(open('$1'));print(d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['clocks'].get('power_w_median'))" 2>&1 | tail -1; }
i=0
for cfg in ST_JACOBI_FOLD=0 ST_JACOBI_FOLD=1 ST_JACOBI_FOLD=0 ST_JACOBI_FOLD=1; do
  i=$((i+1))
  env $cfg timeout 300 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu --no-pw --no-j3 --no-gs --no-generic --no-scaling > $OUT/t_$i.json 2>$OUT/t_$i.err
  echo "$cfg: $(q $OUT/t_$i.json)"
done
