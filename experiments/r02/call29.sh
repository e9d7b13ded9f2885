#!/bin/bash
# round 2, call 29 (4 GPUs): tcgen05 consumers hand an item over at its last tile: c5 / c3 at N=4
O=gpurun_out/r02c29; mkdir -p $O
timeout 600 python -m pytest tests/test_step_gpu.py tests/test_decode_gpu.py -q -x -p no:cacheprovider -m "gpu and not slow" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() { local n=$1 np=$2; shift 2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus $np "$@" --no-cpu-baseline > $O/$n.json 2> $O/$n.err; }
export LAM_SPIN_TIMEOUT_MS=1000
run c5_n4 4 --workload c5 --steps 5 --warmup 2
run c3_n4 4 --workload c3 --steps 10 --warmup 3
run c3_n4_mb4 4 --workload c3 --steps 10 --warmup 3 --micro-batches 4
run c4_n4 4 --workload c4 --steps 5 --warmup 2
