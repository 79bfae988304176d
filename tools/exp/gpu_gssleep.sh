OUT=gpurun_out/gssleep; mkdir -p $OUT
for a in 2000 500 100; do
  touch paper_2310_01882_b200/csrc/gauss_seidel2d_ms.cu
  make -j8 all EXTRA_NVFLAGS="-DST_GS_MS_SSLEEP=$a" > $OUT/build_$a.log 2>&1 || { tail -20 $OUT/build_$a.log; exit 1; }
  ST_GS_MS_K=4 timeout 240 python tools/exp/gs_ms_perf.py --sweeps 100,400 > $OUT/perf_$a.log 2>&1; echo "sleep=$a: $(tail -3 $OUT/perf_$a.log | tr '\n' ' ')"
done
