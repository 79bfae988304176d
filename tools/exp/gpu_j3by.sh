OUT=gpurun_out/j3by; mkdir -p $OUT
for cfg in "16 4" "8 4" "16 2"; do
  set -- $cfg; by=$1; r=$2
  touch paper_2310_01882_b200/csrc/jacobi3d.cu
  make -j8 all EXTRA_NVFLAGS="-DST_J3T2_BY=$by -DST_J3T2_R=$r" > $OUT/build_$by$r.log 2>&1 || { tail -20 $OUT/build_$by$r.log; exit 1; }
  grep -A2 'jacobi3d_t2_kernelILi128ELi'$by'ELi5ELi'$r'ELb0' build/jacobi3d.ptxas.txt | grep -E 'registers|spill' | tr '\n' ' '; echo
  timeout 600 python -m pytest tests -x -q -m gpu -k "jacobi3d" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest.log
  timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-pw --no-gs --no-generic --no-scaling > $OUT/b_$by$r.json 2>$OUT/b_$by$r.err
  python -c "import json;d=json.load(open('$OUT/b_$by$r.json'));j=d['jacobi3d'];print('BY=$by R=$r', j['value'], j['roofline']['frac'])"
done
