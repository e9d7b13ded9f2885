#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/sweep.log 2>&1
for V in 0 1 3 4; do
  LAM_GQA_VARIANT=$V timeout 300 python scripts/exp_decode.py --cfg c3 --splits 0,512,1024,2048,4096 | sed "s/^/v$V /"
done
for V in 0 2 5; do
  LAM_GQA_VARIANT=$V timeout 300 python scripts/exp_decode.py --cfg c3 --P 128 --splits 0,1024,2048 | sed "s/^/v$V P128 /"
done
for V in 0 1 3 4; do
  LAM_GQA_VARIANT=$V timeout 300 python scripts/exp_decode.py --cfg c3n8 --splits 0,1024,2048 | sed "s/^/v$V /"
  LAM_GQA_VARIANT=$V timeout 300 python scripts/exp_decode.py --cfg c4 --splits 0,2048,4096,8192 | sed "s/^/v$V /"
done
timeout 300 python scripts/exp_decode.py --cfg c1 --splits 0,512,256,128 --iters 50
timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0,1024,2048,4096
echo done
