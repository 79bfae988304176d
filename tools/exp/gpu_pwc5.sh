# PW on C5 (1024x1024x512) and C3: planes per CTA chunk
OUT=gpurun_out/pwc5; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for ppc in 128 64 256 512 32; do
  ST_PW_PLANES=$ppc timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-j3 --no-gs --no-generic > $OUT/p_$ppc.json 2>$OUT/p_$ppc.err
  python -c "import json;d=json.load(open('$OUT/p_$ppc.json'));print('ppc=$ppc', 'C5', d['c5']['value'], d['c5']['roofline']['frac'], 'C3', d['pw_advect3d']['value'], d['pw_advect3d']['roofline']['frac'])"
done
