OUT=gpurun_out/j3; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "jacobi3d or pen" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for rep in 1 2; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-pw --no-gs --no-generic --no-scaling > $OUT/b_$rep.json 2>$OUT/b_$rep.err
  python -c "import json;d=json.load(open('$OUT/b_$rep.json'));j=d['jacobi3d'];print('j3', j['value'], j['roofline']['frac'])"
done
