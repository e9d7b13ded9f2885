#!/bin/bash
# round 2, call 40 (4 GPUs): where does c3 at N=4 lose? dependency-free diagnostic, item size,
# micro-batches, weak scaling
O=gpurun_out/r02c40; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
run base 4 --workload c3 --steps 10 --warmup 2
LAM_PEER_AHEAD=1 run ahead 4 --workload c3 --steps 10 --warmup 2
LAM_STEP_ITEM_TOKENS=1024 run item1k 4 --workload c3 --steps 10 --warmup 2
run mb8 4 --workload c3 --steps 10 --warmup 2 --micro-batches 8
run weak 4 --workload c3 --steps 5 --warmup 2 --scaling weak
LAM_PEER_AHEAD=1 run c2_ahead 4 --workload c2 --steps 10 --warmup 2
