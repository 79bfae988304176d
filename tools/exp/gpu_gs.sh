# multi-sweep Gauss-Seidel: parity for K = 1..4, then throughput per K (each step under its own timeout)
OUT=gpurun_out/${TAG:-gs}; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for k in ${KS:-4 2 3 1}; do
  ST_GS_MS_K=$k timeout 240 python tests/gs_ms_cases.py $k > $OUT/cases_$k.log 2>&1; echo "cases K=$k rc=$?"; tail -3 $OUT/cases_$k.log
done
for k in ${PK:-4 3 2}; do
  ST_GS_MS_K=$k timeout 240 python tools/exp/gs_ms_perf.py > $OUT/perf_$k.log 2>&1; echo "perf K=$k rc=$?"; cat $OUT/perf_$k.log | tail -4
done
ST_GS_MS=0 timeout 240 python tools/exp/gs_ms_perf.py --sweeps 4,100 > $OUT/perf_old.log 2>&1; echo "old rc=$?"; tail -2 $OUT/perf_old.log
