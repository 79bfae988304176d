OUT=gpurun_out/${TAG:-pen}; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu -k "pen or jacobi3d or pw or local or ipc" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
timeout 900 python tools/exp/local_overhead.py pencils > $OUT/pencils.json 2> $OUT/pencils.err; echo "pencils rc=$?"; cat $OUT/pencils.err | tail -12
