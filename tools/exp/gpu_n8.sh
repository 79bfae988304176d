# the driver's N>1 launch with every rank on the one GPU (functional: IPC with 4 and 8 processes)
OUT=gpurun_out/n8; mkdir -p $OUT
make -j8 all > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
for n in 4 8; do
  CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) \
    bench.py --gpus $n --same-gpu --steps 1 --warmup 3 --sweeps 20 --pw-apps 2 --scale-steps 1 --j3-sweeps 6 --no-e2e --no-cpu > $OUT/n$n.json 2> $OUT/n$n.err
  echo "N=$n rc=$?"; python -c "
import json;d=json.load(open('$OUT/n$n.json'))
print(d['n_gpus'], d['value'], d.get('per_gpu'), d.get('efficiency'), d['config'].get('transport'), d['config'].get('ipc_probe'), d['config']['workload'])
print('c5', d['c5']['workload'], d['c5'].get('per_gpu'), 'j3', d['jacobi3d']['workload'])" 2>&1 | tail -3
  tail -2 $OUT/n$n.err
done
