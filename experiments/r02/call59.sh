#!/bin/bash
# round 2, call 59 (4 GPUs): c3 at N=4: split count of the dependent step launch (LAM_STEP_SPLITS)
O=gpurun_out/r02c59; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
for s in 1 2 4; do
  for mb in 2 4; do
    LAM_STEP_SPLITS=$s run c3_s${s}_mb$mb 4 --workload c3 --steps 5 --warmup 3 --micro-batches $mb
  done
done
