OUT=gpurun_out/gstrace; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for ny in 32 16384; do
ST_GS_MS_TRACE=1 ST_GS_MS_K=4 timeout 120 python tools/exp/gs_ms_perf.py --ny $ny --sweeps 200 > $OUT/trace_$ny.log 2>&1; echo rc=$?; grep -v 'nan' $OUT/trace_$ny.log | tail -9
done
