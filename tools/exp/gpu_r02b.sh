# copy6 ceiling of the PW access pattern + ncu of the T=10 headline kernel
OUT=gpurun_out/r02b; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o $OUT/copy6 tools/exp/copy6.cu && \
  { $OUT/copy6 512 512; $OUT/copy6 1024 512; } > $OUT/copy6.txt 2>&1; cat $OUT/copy6.txt
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:'jacobi2d_tb4' -s 2 -c 2 \
  -o $OUT/prof python tools/prof_kernels.py --sweeps 40 --tblock 0 --apps 1 --gs-sweeps 1 > $OUT/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 $OUT/ncu.log
