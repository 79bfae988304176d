OUT=gpurun_out/gspub; mkdir -p $OUT
for pub in ${PUBS:-1 2 4}; do
  touch paper_2310_01882_b200/csrc/gauss_seidel2d_ms.cu
  make -j8 all EXTRA_NVFLAGS="-DST_GS_MS_PUB=$pub" > $OUT/build_$pub.log 2>&1 || { tail -20 $OUT/build_$pub.log; exit 1; }
  [ $pub = 1 ] && { ST_GS_MS_K=4 timeout 240 python tests/gs_ms_cases.py 4 | tail -1; }
  ST_GS_MS_K=4 timeout 240 python tools/exp/gs_ms_perf.py --sweeps 100,400 > $OUT/perf_$pub.log 2>&1; echo "pub=$pub: $(tail -2 $OUT/perf_$pub.log | tr '\n' ' ')"
done
