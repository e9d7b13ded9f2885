#!/bin/bash
# round 2, call 41 (4 GPUs): c3 N=4 relay cost: model-side wait on 1 flag instead of 4
# (diagnostic, wrong semantics), 4 micro-batches, per-layer launches for comparison
O=gpurun_out/r02c41; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
run base 4 --workload c3 --steps 10 --warmup 2
LAM_PEER_WAITN=1 run wait1 4 --workload c3 --steps 10 --warmup 2
run mb4 4 --workload c3 --steps 10 --warmup 2 --micro-batches 4
LAM_PEER_WAITN=1 run mb4_wait1 4 --workload c3 --steps 10 --warmup 2 --micro-batches 4
run layer 4 --workload c3 --steps 10 --warmup 2 --launch layer
run n2 2 --workload c3 --steps 10 --warmup 2
