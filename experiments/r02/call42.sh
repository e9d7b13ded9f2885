#!/bin/bash
# round 2, call 42 (4 GPUs): relay latency probe: c3 geometry at l=128 (attention ~free), so the
# per-layer time is the qkv -> attention -> out -> model relay
O=gpurun_out/r02c42; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
export LAM_BENCH_SEQ=128
run n4 4 --workload c3 --steps 10 --warmup 3
LAM_PEER_WAITN=1 run n4_wait1 4 --workload c3 --steps 10 --warmup 3
LAM_PEER_AHEAD=1 run n4_ahead 4 --workload c3 --steps 10 --warmup 3
run n4_layer 4 --workload c3 --steps 10 --warmup 3 --launch layer
run n2 2 --workload c3 --steps 10 --warmup 3
run n1 1 --workload c3 --steps 10 --warmup 3 --engine peer
run n4_mb1 4 --workload c3 --steps 10 --warmup 3 --micro-batches 1
