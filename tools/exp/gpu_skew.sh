#!/bin/bash
# Skewed vs plain rotated steady state of the T-blocked Jacobi kernel: parity, then C2 bench lines.
OUT=gpurun_out/skew; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_full_size.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for t in ${TBS:-10 8}; do for sk in ${SKEWS:-1 0}; do
  ST_JACOBI_TB_SKEW=$sk timeout 300 python bench.py --steps 3 --warmup 3 --tblock $t --no-e2e --no-cpu --no-scaling --no-pw --no-j3 --no-gs --no-generic > $OUT/b_t${t}_s${sk}.json 2> $OUT/b_t${t}_s${sk}.err
  echo "T=$t skew=$sk: $(python -c "import json;d=json.load(open('$OUT/b_t${t}_s${sk}.json'));print(d['value'],d['roofline']['ms_per_pass'],d['clocks'])" 2>&1 | tail -1)"
done; done
