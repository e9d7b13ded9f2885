#!/bin/bash
# round 2, call 58 (4 GPUs): does 4 micro-batches help whenever a rank's layer is ~0.5 GB?
# c2 with l=2048 at N=4 has C2@N=8's per-rank layer size; c3 repeated; c2 full for contrast
O=gpurun_out/r02c58; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
for mb in 2 4; do
  LAM_BENCH_SEQ=2048 run c2l2k_mb$mb 4 --workload c2 --steps 5 --warmup 3 --micro-batches $mb
  run c3_mb$mb 4 --workload c3 --steps 5 --warmup 3 --micro-batches $mb
  run c2_mb$mb 4 --workload c2 --steps 5 --warmup 3 --micro-batches $mb
  run c4_mb$mb 4 --workload c4 --steps 5 --warmup 3 --micro-batches $mb
done
LAM_BENCH_SEQ=2048 timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/c2l2k_n1.json 2> $O/c2l2k_n1.err
