#!/bin/bash
# where does the per-item cost of the tensor-core kernel go?  flags: 16 = no consumer math,
# 32 = no epilogue work, 48 = neither
mkdir -p gpurun_out
exec > gpurun_out/call53.log 2>&1
cd ab/cur
for F in 0 16 32 48; do
  LAM_DECODE_FLAGS=$F PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c3 --splits 4096,1024 --iters 30 2>&1 | grep -v Warn | sed "s/^/flags$F /"
  LAM_DECODE_FLAGS=$F PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c3n8 --splits 4096,2048 --iters 30 2>&1 | grep -v Warn | sed "s/^/flags$F /"
  LAM_DECODE_FLAGS=$F PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c2 --splits 4096,1024 --iters 30 2>&1 | grep -v Warn | sed "s/^/flags$F /"
done
