# 3-D Jacobi T=2 build variants (EXTRA_NVFLAGS) and run-time knobs, timed by bench.py's jacobi3d leg
j3() { timeout 300 env $2 python bench.py --sweeps 8 --no-pw --no-gs --no-generic --no-e2e --no-cpu --steps 3 > gpurun_out/j3v.json 2>/dev/null
  echo "variant [$1] [$2]: $(python -c "import json;d=json.load(open('gpurun_out/j3v.json'))['jacobi3d'];print(d['value'],d['roofline']['frac'])")"; }
for v in "-DST_J3T2_UNROLL=6" "-DST_J3T2_UNROLL=2" ""; do
  touch paper_2310_01882_b200/csrc/jacobi3d.cu
  make -j8 all EXTRA_NVFLAGS="$v" > /dev/null 2>&1 || echo "build $v failed"
  j3 "$v" ""
done
for k in ST_J3T2_PLANES=64 ST_J3T2_PLANES=128 ST_J3T2_PLANES=171 ST_J3T2_VARIANT=3; do j3 "" $k; done
timeout 300 python -m pytest tests/test_gpu_jacobi3d.py -q -x 2>&1 | tail -1
