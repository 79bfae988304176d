# PW build variants (EXTRA_NVFLAGS), timed by bench.py's PW leg
for v in "-DST_PW_UNROLL=3" "-DST_PW_UNROLL=2" ""; do
  touch paper_2310_01882_b200/csrc/pw_advect3d.cu
  make -j8 all EXTRA_NVFLAGS="$v" > /dev/null 2>&1 || echo "build $v failed"
  timeout 300 python bench.py --sweeps 8 --no-j3 --no-gs --no-generic --no-e2e --no-cpu --steps 3 > gpurun_out/pwv.json 2>/dev/null
  echo "variant [$v]: $(python -c "import json;d=json.load(open('gpurun_out/pwv.json'))['pw_advect3d'];print(d['value'],d['roofline']['frac'])")"
done
