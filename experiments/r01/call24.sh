#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/sweep16.log 2>&1
for F in 0 64 8; do
  LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c3 --splits 2048,1024,512 | sed "s/^/f$F /"
done
for F in 0 64; do LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c3n8 --splits 2048,1024 | sed "s/^/f$F /"; LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c4 --splits 8192,4096 | sed "s/^/f$F /"; done
