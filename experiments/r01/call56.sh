#!/bin/bash
# 2 GPUs: request-partitioned pool with NCCL + real kernels; C1 split sweep
mkdir -p gpurun_out
exec > gpurun_out/call56.log 2>&1
timeout 900 python -m pytest tests/test_dist_gpu.py -q -k request 2>&1 | tail -3
for R in 1 2; do
  PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c1 --splits 1024,512,256,128 --iters 50 2>&1 | grep -v Warn
  LAM_DECODE_CTAS=128 PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c1 --splits 1024,256 --iters 50 2>&1 | grep -v Warn | sed "s/^/ctas128 /"
done
