#!/bin/bash
# claim-ahead A/B (LAM_CLAIM_AHEAD = 0 / 4 / 8 / 16), same box; correctness first
mkdir -p gpurun_out
exec > gpurun_out/call52.log 2>&1
LAM_CLAIM_AHEAD=8 timeout 600 python -m pytest tests/test_decode_gpu.py -x -q 2>&1 | tail -2
cd ab/cur
for R in 1 2; do
for A in 0 4 8 16; do
  for C in c2 c3 c5 c3n8 c1; do
    LAM_CLAIM_AHEAD=$A PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/A$A /"
  done
done
done
for A in 0 8; do
  LAM_DECODE_FLAGS=16 LAM_CLAIM_AHEAD=$A PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c3 --splits 4096,1024 --iters 30 2>&1 | grep -v Warn | sed "s/^/stream A$A /"
  LAM_CLAIM_AHEAD=$A PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c3 --splits 1024 --iters 30 2>&1 | grep -v Warn | sed "s/^/A$A /"
  LAM_CLAIM_AHEAD=$A PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c4 --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/A$A /"
done
