OUT=gpurun_out/gsprobe; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for k in 1 2 3 4; do
  ST_GS_MS_PROBE=1 ST_GS_MS_K=$k timeout 120 python tools/exp/gs_ms_perf.py --sweeps 8,200 > $OUT/probe_$k.log 2>&1; echo "probe K=$k rc=$?"; tail -1 $OUT/probe_$k.log
done
