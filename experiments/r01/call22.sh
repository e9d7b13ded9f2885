#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/sweep14.log 2>&1
for F in 0 8; do
  LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c3 --splits 4096,2048,1024 | sed "s/^/f$F /"
  LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c2 --splits 4096,1024 | sed "s/^/f$F /"
done
