#!/bin/bash
# round 2, call 65 (4 GPUs): row map (request partition on the peer transport): 1-GPU oracle
# test, multi-GPU engine tests (request partition over NCCL and peer, every head-shard mode)
O=gpurun_out/r02c65; mkdir -p $O
timeout 1500 python -m pytest tests/test_peer_gpu.py tests/test_step_gpu.py tests/test_dist_gpu.py -x -q > $O/tests.txt 2>&1
