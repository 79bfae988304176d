OUT=gpurun_out/gscheck; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "gauss or seidel" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > $OUT/sanitize_$tool.log 2>&1
  echo "sanitize $tool rc=$?"; tail -2 $OUT/sanitize_$tool.log
done
