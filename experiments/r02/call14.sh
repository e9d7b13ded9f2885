#!/bin/bash
# round 2, call 14 (2 GPUs): multi-GPU tests, strong-scaling bench lines N=1 and N=2 for c3 / c2
O=gpurun_out/r02c14; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_peer_gpu.py -q -p no:cacheprovider -rf > $O/pytest_dist.log 2>&1; echo "rc=$?" >> $O/pytest_dist.log
for wl in c3 c2; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > $O/${wl}_n1.json 2> $O/${wl}_n1.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > $O/${wl}_n2.json 2> $O/${wl}_n2.err
done
