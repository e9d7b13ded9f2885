#!/bin/bash
# round 2, call 66 (4 GPUs): C5 over the request partition (peer transport) vs the head
# partition (bench.py), same box
O=gpurun_out/r02c66; mkdir -p $O
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29524 experiments/r02/req_partition_bench.py > $O/req_n$n.json 2> $O/req_n$n.err
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $n --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/head_n$n.json 2> $O/head_n$n.err
done
timeout 400 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --check 0 > $O/head_n1.json 2> $O/head_n1.err
