#!/bin/bash
# round 2, call 38 (2 GPUs): NVLink peer-transport preset (latency + bandwidth)
O=gpurun_out/r02c38; mkdir -p $O
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 experiments/r02/nvlink_preset.py > $O/nvlink.json 2> $O/nvlink.err
