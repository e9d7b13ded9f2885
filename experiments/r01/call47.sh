#!/bin/bash
# streaming-only diagnostic (consumers skip the math): does the item count cost the producer?
mkdir -p gpurun_out
exec > gpurun_out/call47.log 2>&1
cd ab/cur
for F in 0 16; do
  LAM_DECODE_FLAGS=$F PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c3n8 --splits 4096,2048,1024,512 --iters 30 2>&1 | grep -v Warn | sed "s/^/flags$F /"
  LAM_DECODE_FLAGS=$F PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c3 --splits 4096,2048,1024 --iters 30 2>&1 | grep -v Warn | sed "s/^/flags$F /"
  LAM_DECODE_FLAGS=$F PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c2 --splits 4096,1024 --iters 30 2>&1 | grep -v Warn | sed "s/^/flags$F /"
  LAM_DECODE_FLAGS=$F PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c4 --splits 32768,8192,2048 --iters 30 2>&1 | grep -v Warn | sed "s/^/flags$F /"
done
