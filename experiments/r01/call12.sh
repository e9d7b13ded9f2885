#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/sweep8.log 2>&1
for V in 0 2; do
  for C in c3 c3n8 c4; do
    LAM_GQA_VARIANT=$V timeout 300 python scripts/exp_decode.py --cfg $C --P 128 --splits 0,2048,1024 | sed "s/^/v$V P128 /"
  done
done
echo done
