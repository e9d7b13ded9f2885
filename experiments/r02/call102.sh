#!/bin/bash
# round 2 (session 3), call 102 (4 GPUs): strong scaling of C3 / C4 / C5 with the final kernels,
# one box: N = 1 and N = 4
O=gpurun_out/r02c102; mkdir -p $O
for w in c3 c4 c5; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${w}_n1.json 2> $O/${w}_n1.err
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2958${w:1:1} bench.py --gpus 4 --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${w}_n4.json 2> $O/${w}_n4.err
done
echo done
