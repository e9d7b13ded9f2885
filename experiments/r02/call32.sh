#!/bin/bash
# round 2, call 32 (4 GPUs): per-micro-batch model streams + length-capped items: c3 / c5 at N=4,
# micro-batches 2 and 4; c2 N=4
O=gpurun_out/r02c32; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
run c3_mb2 4 --workload c3 --steps 10 --warmup 2
run c3_mb4 4 --workload c3 --steps 10 --warmup 2 --micro-batches 4
run c5_mb2 4 --workload c5 --steps 5 --warmup 2
run c5_mb4 4 --workload c5 --steps 5 --warmup 2 --micro-batches 4
run c2_mb2 4 --workload c2 --steps 10 --warmup 2
