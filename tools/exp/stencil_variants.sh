# generic stencil2d kernel build variants (EXTRA_NVFLAGS), timed by bench.py's stencil2d_generic leg
for v in "" "-DST_STENCIL_SX=64 -DST_STENCIL_SY=2" "-DST_STENCIL_SX=128 -DST_STENCIL_SY=1" "-DST_STENCIL_SX=64 -DST_STENCIL_SY=2 -DST_STENCIL_RPT=2" "-DST_STENCIL_SX=64 -DST_STENCIL_SY=4" "-DST_STENCIL_SX=32 -DST_STENCIL_SY=2" "-DST_STENCIL_SX=64 -DST_STENCIL_SY=2 -DST_STENCIL_TU=8"; do
  touch paper_2310_01882_b200/csrc/stencil2d.cu
  make -j8 all EXTRA_NVFLAGS="$v" > /dev/null 2>&1 || echo "build $v failed"
  timeout 300 python bench.py --sweeps 8 --no-pw --no-j3 --no-gs --no-e2e --no-cpu --steps 2 > gpurun_out/sv.json 2>/dev/null
  echo "variant [$v]: $(python -c "import json;d=json.load(open('gpurun_out/sv.json'))['stencil2d_generic'];print(d['value'],d['roofline']['frac'])")"
done
touch paper_2310_01882_b200/csrc/stencil2d.cu; make -j8 all > /dev/null 2>&1
