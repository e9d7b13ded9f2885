#!/bin/bash
# round 2, call 72 (2 GPUs): where C5 loses at N=2: per-launch stamps and claim records
O=gpurun_out/r02c72; mkdir -p $O
LAM_STEP_TRACE=$O/tr_c5n2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 2 --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/c5n2.json 2> $O/c5n2.err
python experiments/r02/trace_report.py $O/tr_c5n2 2 > $O/c5n2.trace.txt 2>&1
LAM_STEP_TRACE=$O/tr_c3n2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 2 --workload c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/c3n2.json 2> $O/c3n2.err
python experiments/r02/trace_report.py $O/tr_c3n2 2 > $O/c3n2.trace.txt 2>&1
