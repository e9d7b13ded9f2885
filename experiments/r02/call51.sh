#!/bin/bash
# round 2, call 51 (4 GPUs): step / relay modes in the multi-GPU tests; strong scaling with the
# stream relay (default) and the in-kernel relay after the single-fence publication
O=gpurun_out/r02c51; mkdir -p $O
timeout 1200 python -m pytest tests/test_dist_gpu.py tests/test_step_gpu.py -x -q > $O/tests.txt 2>&1
run() { local n=$1 np=$2; shift 2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e > $O/$n.json 2> $O/$n.err; }
for w in c2 c3 c4 c5; do
  for n in 2 4; do
    run ${w}n${n}_stream $n --workload $w --steps 5 --warmup 3
    run ${w}n${n}_kernel $n --workload $w --steps 5 --warmup 3 --relay kernel
  done
done
run c5n4_kernel_mb4 4 --workload c5 --steps 5 --warmup 3 --relay kernel --micro-batches 4
