#!/bin/bash
# round 2, call 46 (4 GPUs): single-fence publication + remote qkv polling: multi-GPU tests,
# c3 N=4 / N=2 with stamps and the output check
O=gpurun_out/r02c46; mkdir -p $O
timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_step_gpu.py tests/test_peer_gpu.py -x -q > $O/tests.txt 2>&1
run() { local n=$1 np=$2; shift 2
  LAM_STEP_TRACE=$O/tr_$n timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus $np "$@" --no-cpu-baseline --no-e2e > $O/$n.json 2> $O/$n.err
  python experiments/r02/trace_report.py $O/tr_$n 2 > $O/$n.trace.txt 2>&1; }
run n4 4 --workload c3 --steps 10 --warmup 3
run n2 2 --workload c3 --steps 10 --warmup 3
