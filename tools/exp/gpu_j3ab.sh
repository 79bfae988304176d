# 3-D Jacobi T=2: ddiv6_vote (default build) vs per-lane ddiv6 (-DST_J3_VOTE=0)
OUT=gpurun_out/j3ab; mkdir -p $OUT
for v in 1 0; do
  touch paper_2310_01882_b200/csrc/jacobi3d.cu
  make -j8 all EXTRA_NVFLAGS="-DST_J3_VOTE=$v" > $OUT/build_$v.log 2>&1 || { tail -20 $OUT/build_$v.log; exit 1; }
  [ $v = 1 ] && { timeout 600 python -m pytest tests -x -q -m gpu -k "jacobi3d" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest.log; }
  for rep in 1 2; do
    timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-pw --no-gs --no-generic --no-scaling > $OUT/b_${v}_$rep.json 2>$OUT/b_${v}_$rep.err
    python -c "import json;d=json.load(open('$OUT/b_${v}_$rep.json'));j=d['jacobi3d'];print('vote=$v', j['value'], j['roofline']['frac'])"
  done
done
