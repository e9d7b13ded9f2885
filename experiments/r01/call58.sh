#!/bin/bash
# 4 GPUs, current build: multi-GPU tests (head / request / peer), default bench at N=1/2/4 (C2), C3 at N=2/4
mkdir -p gpurun_out
exec > gpurun_out/call58.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -k "dist or peer or request" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/b58_c2_n1.json 2>/dev/null; echo "N=1 c2 rc=$?"
for N in 2 4; do
  for WL in c2 c3; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --workload $WL > gpurun_out/b58_${WL}_n$N.json 2> gpurun_out/b58_${WL}_n$N.err; echo "N=$N $WL rc=$?"
  done
done
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/b58_c3_n1.json 2>/dev/null; echo "N=1 c3 rc=$?"
