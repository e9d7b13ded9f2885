#!/bin/bash
# round 2, call 61 (4 GPUs): split policy, continued: larger item caps, 4 micro-batches
O=gpurun_out/r02c61; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
export LAM_STEP_ROUNDS=0
for w in c4 c5; do
  LAM_STEP_ITEM_TOKENS=16384 run ${w}_t16k 4 --workload $w --steps 5 --warmup 3
  LAM_STEP_ITEM_TOKENS=32768 run ${w}_t32k 4 --workload $w --steps 5 --warmup 3
  LAM_STEP_ITEM_TOKENS=8192 run ${w}_t8k 4 --workload $w --steps 5 --warmup 3
done
for w in c3 c5 c2; do
  LAM_STEP_ITEM_TOKENS=8192 run ${w}_t8k_mb4 4 --workload $w --steps 5 --warmup 3 --micro-batches 4
done
LAM_STEP_ITEM_TOKENS=8192 run c2_t8k 4 --workload c2 --steps 5 --warmup 3
