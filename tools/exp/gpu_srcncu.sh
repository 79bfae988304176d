#!/bin/bash
# ncu --set full with source-level stall sampling of one launch of the kernel matching $KREG
# (launched by tools/prof_kernels.py), exported as the source-page CSV.
OUT=gpurun_out/srcncu; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
NCU=/usr/local/cuda/bin/ncu
TAG=${TAG:-k}
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$KREG -s ${SKIP:-0} -c 1 \
   -o $OUT/$TAG python tools/prof_kernels.py ${PROF_ARGS:---sweeps 2 --tblock 1 --apps 0} > $OUT/$TAG.log 2>&1
echo "ncu rc=$?"
$NCU -i $OUT/$TAG.ncu-rep --page source --csv --print-source sass > $OUT/src_$TAG.csv 2> /dev/null
$NCU -i $OUT/$TAG.ncu-rep --page raw --csv > $OUT/raw_$TAG.csv 2>/dev/null
python tools/ncu_source_stalls.py $OUT/src_$TAG.csv
