#!/bin/bash
# round 2, call 22 (2 GPUs): strong scaling with the step launch (c3, c2), N=1 and N=2 on one box;
# multi-GPU tests; c3 step with the tcgen05 kernel
O=gpurun_out/r02c22; mkdir -p $O
timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_peer_gpu.py tests/test_step_gpu.py -q -p no:cacheprovider -rf > $O/pytest_dist.log 2>&1; echo "rc=$?" >> $O/pytest_dist.log
run() { # name, nproc, args...
  local n=$1 np=$2; shift 2
  if [ $np = 1 ]; then timeout 900 python bench.py "$@" --no-cpu-baseline > $O/$n.json 2> $O/$n.err
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $np "$@" --no-cpu-baseline > $O/$n.json 2> $O/$n.err; fi
}
for wl in c3 c2; do
  run ${wl}_n1 1 --workload $wl --steps 10 --warmup 3
  run ${wl}_n2 2 --workload $wl --steps 10 --warmup 3
  run ${wl}_n2_layer 2 --workload $wl --steps 10 --warmup 3 --launch layer
done
LAM_GQA_TC=1 run c3_n1_tc 1 --workload c3 --steps 10 --warmup 3
LAM_GQA_TC=1 run c3_n2_tc 2 --workload c3 --steps 10 --warmup 3
