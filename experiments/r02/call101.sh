#!/bin/bash
# round 2 (session 3), call 101 (4 GPUs): strong scaling of the default workload (C2) with the
# final kernels, one box: N = 1, 2, 4
O=gpurun_out/r02c101; mkdir -p $O
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/c2_n1.json 2> $O/c2_n1.err
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline > $O/c2_n$n.json 2> $O/c2_n$n.err
done
echo done
