OUT=gpurun_out/gsncu; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
ST_GS_MS_K=${K:-4} timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:gauss_seidel2d_ms -s ${SKIP:-2} -c 1 \
  -o $OUT/prof python tools/exp/gs_ms_perf.py --sweeps 4,${SW:-100} > $OUT/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $OUT/ncu.log
