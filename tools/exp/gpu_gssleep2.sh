OUT=gpurun_out/gssleep2; mkdir -p $OUT
for f in "-DST_GS_MS_LSLEEP=500 -DST_GS_MS_PSLEEP=200" "-DST_GS_MS_LSLEEP=1000 -DST_GS_MS_PSLEEP=500" "-DST_GS_MS_LSLEEP=200 -DST_GS_MS_PSLEEP=100"; do
  touch paper_2310_01882_b200/csrc/gauss_seidel2d_ms.cu
  make -j8 all EXTRA_NVFLAGS="$f" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
  ST_GS_MS_K=4 timeout 240 python tools/exp/gs_ms_perf.py --sweeps 100,400 > $OUT/perf.log 2>&1; echo "$f: $(tail -3 $OUT/perf.log | tr '\n' ' ')"
done
