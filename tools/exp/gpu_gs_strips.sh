OUT=gpurun_out/gsstrips; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for ny in 32 16384; do
  for probe in 0 1 3; do
    ST_GS_MS_PROBE=$probe ST_GS_MS_K=4 timeout 120 python tools/exp/gs_ms_perf.py --ny $ny --sweeps 40,200 > $OUT/s_${ny}_$probe.log 2>&1
    echo "ny=$ny probe=$probe: $(tail -1 $OUT/s_${ny}_$probe.log)"
  done
done
