#!/bin/bash
# round 2, call 44 (4 GPUs): stream memop latencies; c3 N=4 relay with/without the signal barrier
O=gpurun_out/r02c44; mkdir -p $O
timeout 200 python experiments/r02/memop_latency.py > $O/memop_default.txt 2>&1
LAM_SIGNAL_NO_BARRIER=1 timeout 200 python experiments/r02/memop_latency.py > $O/memop_nobarrier.txt 2>&1
run() { local n=$1 np=$2; shift 2
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
LAM_BENCH_SEQ=128 LAM_SIGNAL_NO_BARRIER=1 run l128_nob 4 --workload c3 --steps 10 --warmup 3
LAM_SIGNAL_NO_BARRIER=1 run full_nob 4 --workload c3 --steps 10 --warmup 3
