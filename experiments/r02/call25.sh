#!/bin/bash
# round 2, call 25 (2 GPUs): step-launch splits: tests, then c4 / c3 / c5 strong N=2 with status
O=gpurun_out/r02c25; mkdir -p $O
timeout 900 python -m pytest tests/test_step_gpu.py tests/test_dist_gpu.py -q -p no:cacheprovider -rf -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() { local n=$1 np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus $np "$@" --no-cpu-baseline > $O/$n.json 2> $O/$n.err; }
LAM_SPIN_TIMEOUT_MS=2000 run c4_n2 2 --workload c4 --steps 5 --warmup 2
LAM_SPIN_TIMEOUT_MS=2000 run c5_n2 2 --workload c5 --steps 5 --warmup 2
LAM_SPIN_TIMEOUT_MS=2000 run c3_n2 2 --workload c3 --steps 10 --warmup 3
