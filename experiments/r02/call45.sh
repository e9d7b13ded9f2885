#!/bin/bash
# round 2, call 45 (4 GPUs): per-launch stamps of the c3 step (LAM_STEP_TRACE)
O=gpurun_out/r02c45; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  LAM_STEP_TRACE=$O/tr_$n timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err
  python experiments/r02/trace_report.py $O/tr_$n 2 > $O/$n.trace.txt 2>&1; }
run n4 4 --workload c3 --steps 5 --warmup 3
LAM_BENCH_SEQ=128 run n4_l128 4 --workload c3 --steps 5 --warmup 3
run n2 2 --workload c3 --steps 5 --warmup 3
