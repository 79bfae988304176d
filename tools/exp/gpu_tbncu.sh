#!/bin/bash
# ncu --set full (source-level stalls) of the T-blocked Jacobi kernel, one launch per variant.
OUT=gpurun_out/tbncu; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
NCU=/usr/local/cuda/bin/ncu
for sk in 0; do  # (the skewed variant it compared is gone: DESIGN.md §6.2)
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:jacobi2d_tb4 -c 1 \
     -o $OUT/tb_s$sk python tools/prof_kernels.py --sweeps 10 --tblock ${TB:-10} --apps 0 > $OUT/ncu_s$sk.log 2>&1
  echo "ncu s$sk rc=$?"
  $NCU -i $OUT/tb_s$sk.ncu-rep --page source --csv --print-source sass > $OUT/src_s$sk.csv 2> $OUT/src_s$sk.err
  $NCU -i $OUT/tb_s$sk.ncu-rep --page raw --csv > $OUT/raw_s$sk.csv 2>/dev/null
  ls -la $OUT/tb_s$sk.ncu-rep $OUT/src_s$sk.csv
done
