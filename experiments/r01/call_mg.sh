#!/bin/bash
mkdir -p gpurun_out
N=${NGPU:-2}
timeout 600 python -m pytest tests/test_dist_gpu.py -q > gpurun_out/pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.log
for WL in ${WORKLOADS:-c2}; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps ${STEPS:-10} --warmup 3 --workload $WL --no-cpu-baseline > gpurun_out/bench_${WL}_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${WL}_n$N.log
done
for f in gpurun_out/pytest_dist.log gpurun_out/bench_*_n$N.log; do tail -n 2 $f; done
