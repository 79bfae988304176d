OUT=gpurun_out/gsp; mkdir -p $OUT
for p in 4 8 2; do
  touch paper_2310_01882_b200/csrc/gauss_seidel2d_ms.cu
  make -j8 all EXTRA_NVFLAGS="-DST_GS_MS_P=$p" > $OUT/build_$p.log 2>&1 || { tail -20 $OUT/build_$p.log; exit 1; }
  grep -A2 'ms_kernelILi4' build/gauss_seidel2d_ms.ptxas.txt | grep -E 'registers|spill' | tr '\n' ' '
  [ $p = 4 ] && { ST_GS_MS_K=4 timeout 240 python tests/gs_ms_cases.py 4 | tail -1; }
  ST_GS_MS_K=4 timeout 240 python tools/exp/gs_ms_perf.py --sweeps 100,400 > $OUT/perf_$p.log 2>&1; echo "P=$p: $(tail -3 $OUT/perf_$p.log | tr '\n' ' ')"
done
