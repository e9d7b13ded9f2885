#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/sweep18.log 2>&1
for F in 0 8; do
  LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c5 --splits 0,4096,2048 | sed "s/^/f$F /"
  LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c5 --splits 0 --no-order | sed "s/^/f$F noorder /"
  LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c3 --splits 0 | sed "s/^/f$F /"
done
