#!/bin/bash
# round 2, call 27 (4 GPUs): strong scaling with the step launch (full grid, splits), N=1,2,4, one box
O=gpurun_out/r02c27; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  if [ $np = 1 ]; then timeout 600 python bench.py "$@" --no-cpu-baseline > $O/$n.json 2> $O/$n.err
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29516 bench.py --gpus $np "$@" --no-cpu-baseline > $O/$n.json 2> $O/$n.err; fi; }
export LAM_SPIN_TIMEOUT_MS=3000
for wl in c3 c2; do for np in 1 2 4; do run ${wl}_n$np $np --workload $wl --steps 10 --warmup 3; done; done
for wl in c4 c5; do for np in 1 2 4; do run ${wl}_n$np $np --workload $wl --steps 5 --warmup 2; done; done
run c3_n4_mb4 4 --workload c3 --steps 10 --warmup 3 --micro-batches 4
