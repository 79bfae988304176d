OUT=gpurun_out/gsncu2; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for probe in ${PROBES:-0 1}; do
ST_GS_MS_PROBE=$probe ST_GS_MS_K=4 timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:gauss_seidel2d_ms -s 1 -c 1 \
  -o $OUT/prof_$probe python tools/exp/gs_ms_perf.py --sweeps 200 > $OUT/ncu_$probe.log 2>&1; echo "ncu $probe rc=$?"
done
