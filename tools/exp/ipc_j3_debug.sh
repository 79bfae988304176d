# IPC 3-D slab debug runs (world, fused, halo, iters, tblock, dims) with per-plane mismatch reports
run() { # world fused h it tb dims
  P=$(python -c "import socket;s=socket.socket();s.bind(('127.0.0.1',0));print(s.getsockname()[1])")
  for r in $(seq 0 $(($1-1))); do
    RANK=$r WORLD_SIZE=$1 LOCAL_RANK=$r MASTER_ADDR=127.0.0.1 MASTER_PORT=$P ST_FUSED_HALO=$2 J3_H=$3 J3_IT=$4 J3_TB=$5 J3_DIMS=$6 timeout 120 python tests/ipc_cases.py j3_dbg > gpurun_out/dbg/r$r.log 2>&1 &
  done; wait; echo "== w=$1 fused=$2 h=$3 it=$4 tb=$5 dims=$6"; grep -h "rank\|CASE" gpurun_out/dbg/r0.log | cut -c1-200
}
mkdir -p gpurun_out/dbg
for ST in 0 1; do ST_FUSED_HALO=$ST CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 120 python tests/local_group_cases.py j3_p2_h2_t2_b | tail -1; done
run 2 1 2 3 2 70,33,29
run 2 1 2 4 2 70,33,29
run 2 1 2 5 2 70,33,29
run 2 1 2 6 2 70,33,29
run 2 1 2 4 2 140,33,29
run 2 1 2 4 2 70,40,29
run 2 1 2 4 2 64,32,29
run 2 1 2 4 2 70,33,60
