#!/bin/bash
# round 2, call 62 (4 GPUs): final same-box strong-scaling table, default flags (step launch,
# peer transport, 2 micro-batches, stream relay, output check on)
O=gpurun_out/r02c62; mkdir -p $O
run() { local n=$1 np=$2; shift 2
  if [ $np = 1 ]; then timeout 400 python bench.py "$@" --no-cpu-baseline > $O/$n.json 2> $O/$n.err
  else timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline > $O/$n.json 2> $O/$n.err; fi; }
for w in c2 c3 c4 c5; do
  for n in 1 2 4; do
    run ${w}_n$n $n --workload $w --steps 5 --warmup 3
  done
done
