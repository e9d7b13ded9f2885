#!/bin/bash
# round 2, call 28 (4 GPUs): diagnose c5 / c3 at N=4 with the step launch
O=gpurun_out/r02c28; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
export LAM_SPIN_TIMEOUT_MS=1000 LAM_BENCH_VERBOSE=1
run c5_n4 4 --workload c5 --steps 2 --warmup 2
run c3_n4 4 --workload c3 --steps 5 --warmup 2
LAM_BENCH_SPLIT_TOKENS=4096 run c3_n4_s1 4 --workload c3 --steps 5 --warmup 2
run c3_n4_layer 4 --workload c3 --steps 5 --warmup 2 --launch layer
