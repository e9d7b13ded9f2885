#!/bin/bash
# round 2, call 57 (4 GPUs): c3 at N=4 after the single-fence publication: micro-batches x relay
O=gpurun_out/r02c57; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e --check 0 > $O/$n.json 2> $O/$n.err; }
for mb in 2 4 8; do
  run c3_mb${mb}_stream 4 --workload c3 --steps 5 --warmup 3 --micro-batches $mb
  run c3_mb${mb}_kernel 4 --workload c3 --steps 5 --warmup 3 --micro-batches $mb --relay kernel
done
run c5_mb4_stream 4 --workload c5 --steps 5 --warmup 3 --micro-batches 4
run c5_mb8_stream 4 --workload c5 --steps 5 --warmup 3 --micro-batches 8
