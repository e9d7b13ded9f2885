#!/bin/bash
# round 2, call 24 (4 GPUs): strong scaling c3 / c2 / c5 / c4 with the step launch at N=1,2,4 on one box;
# 4-rank multi-GPU tests
O=gpurun_out/r02c24; mkdir -p $O
timeout 900 python -m pytest tests/test_dist_gpu.py -q -p no:cacheprovider -rf > $O/pytest_dist.log 2>&1; echo "rc=$?" >> $O/pytest_dist.log
run() { # name, nproc, args...
  local n=$1 np=$2; shift 2
  if [ $np = 1 ]; then timeout 900 python bench.py "$@" --no-cpu-baseline > $O/$n.json 2> $O/$n.err
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $np "$@" --no-cpu-baseline > $O/$n.json 2> $O/$n.err; fi
}
for wl in c3 c2 c5 c4; do
  for np in 1 2 4; do run ${wl}_n$np $np --workload $wl --steps 10 --warmup 3; done
done
