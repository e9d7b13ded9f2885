#!/bin/bash
# round 2, call 30 (4 GPUs): c3 at N=4: step (S auto / S=1 / 128 CTAs), per-layer, mma.sync kernel
O=gpurun_out/r02c30; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
run c3_step 4 --workload c3 --steps 10 --warmup 3
LAM_BENCH_SPLIT_TOKENS=4096 run c3_step_s1 4 --workload c3 --steps 10 --warmup 3
LAM_DECODE_CTAS=128 LAM_BENCH_SPLIT_TOKENS=4096 run c3_step_s1_128 4 --workload c3 --steps 10 --warmup 3
run c3_layer 4 --workload c3 --steps 10 --warmup 3 --launch layer
LAM_GQA_TC=0 run c3_step_mma 4 --workload c3 --steps 10 --warmup 3
LAM_GQA_TC=0 run c3_layer_mma 4 --workload c3 --steps 10 --warmup 3 --launch layer
