#!/bin/bash
# round 2, call 26 (2 GPUs): micro-batches 2 vs 4 for c4 / c3 strong at N=2; step tests
O=gpurun_out/r02c26; mkdir -p $O
timeout 900 python -m pytest tests/test_step_gpu.py -q -p no:cacheprovider -rf -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() { local n=$1 np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e > $O/$n.json 2> $O/$n.err; }
for mb in 4 2 8; do
  LAM_SPIN_TIMEOUT_MS=2000 run c4_mb$mb 2 --workload c4 --steps 5 --warmup 2 --micro-batches $mb
done
for mb in 4 2; do
  LAM_SPIN_TIMEOUT_MS=2000 run c3_mb$mb 2 --workload c3 --steps 10 --warmup 3 --micro-batches $mb
done
