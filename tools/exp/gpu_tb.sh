OUT=gpurun_out/${TAG:-tb}; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_jacobi.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
q() { python -c "import json,sys;d=json.load(open('$1'));print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['clocks'].get('power_w_median'), d.get('c4',{}).get('value'))" 2>&1 | tail -1; }
i=0
for cfg in ${CFGS:-ST_JACOBI_TB4_CTA=1 ST_JACOBI_TB4_CTA=0}; do
  i=$((i+1))
  env $(echo $cfg | tr ',' ' ') timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-pw --no-j3 --no-gs --no-generic ${BARGS:---no-scaling} > $OUT/t_$i.json 2>$OUT/t_$i.err
  echo "$cfg: $(q $OUT/t_$i.json)"
done
