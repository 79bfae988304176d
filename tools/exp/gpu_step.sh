# scratch GPU step (edited per experiment); run under gpurun from the repo root
OUT=gpurun_out/${TAG:-r2g}; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
PYTHONFAULTHANDLER=1 CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --same-gpu --steps 1 --warmup 3 --sweeps 16 --pw-apps 2 --scale-steps 1 --j3-sweeps 6 --no-e2e --no-cpu > $OUT/n2.out 2> $OUT/n2.err
echo "rc=$?"; tail -c 1500 $OUT/n2.out; grep -v "^\s*$" $OUT/n2.err | grep -A25 "Fatal\|Error\|error" | head -60
