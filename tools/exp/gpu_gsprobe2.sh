OUT=gpurun_out/gsprobe2; mkdir -p $OUT
for f in "-DST_GS_MS_PROBE_NOLOAD" "-DST_GS_MS_PROBE_NOSTORE" "-DST_GS_MS_PROBE_NOLOAD -DST_GS_MS_PROBE_NOSTORE" ""; do
  touch paper_2310_01882_b200/csrc/gauss_seidel2d_ms.cu
  make -j8 all EXTRA_NVFLAGS="$f" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
  ST_GS_MS_K=4 timeout 240 python tools/exp/gs_ms_perf.py --sweeps 100,400 > $OUT/perf.log 2>&1; echo "[$f]: $(tail -1 $OUT/perf.log)"
done
