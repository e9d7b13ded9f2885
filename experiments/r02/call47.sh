#!/bin/bash
# round 2, call 47 (4 GPUs): in-kernel model-worker relay (--relay kernel), strong scaling
O=gpurun_out/r02c47; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  LAM_STEP_TRACE=$O/tr_$n timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e > $O/$n.json 2> $O/$n.err
  python experiments/r02/trace_report.py $O/tr_$n 2 > $O/$n.trace.txt 2>&1; }
run c3n4 4 --workload c3 --steps 10 --warmup 3 --relay kernel
run c3n2 2 --workload c3 --steps 10 --warmup 3 --relay kernel
run c2n4 4 --workload c2 --steps 10 --warmup 3 --relay kernel
run c4n4 4 --workload c4 --steps 5 --warmup 3 --relay kernel
run c5n4 4 --workload c5 --steps 5 --warmup 3 --relay kernel
run c3n4_stream 4 --workload c3 --steps 10 --warmup 3
