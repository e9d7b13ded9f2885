#!/bin/bash
# round 2, call 60 (4 GPUs): split policy of dependent step launches: rounds rule on/off, item cap
O=gpurun_out/r02c60; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
for w in c4 c5 c3; do
  LAM_STEP_ROUNDS=1 LAM_STEP_ITEM_TOKENS=4096 run ${w}_r1_t4k 4 --workload $w --steps 5 --warmup 3
  LAM_STEP_ROUNDS=0 LAM_STEP_ITEM_TOKENS=4096 run ${w}_r0_t4k 4 --workload $w --steps 5 --warmup 3
  LAM_STEP_ROUNDS=0 LAM_STEP_ITEM_TOKENS=8192 run ${w}_r0_t8k 4 --workload $w --steps 5 --warmup 3
done
LAM_STEP_ROUNDS=0 run c3_r0_t4k_n2 2 --workload c3 --steps 5 --warmup 3
LAM_STEP_ROUNDS=0 run c4_r0_t4k_n2 2 --workload c4 --steps 5 --warmup 3
LAM_STEP_ROUNDS=0 run c5_r0_t4k_n2 2 --workload c5 --steps 5 --warmup 3
