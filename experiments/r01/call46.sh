#!/bin/bash
# split path: batched merge (cur) vs sequential merge (om) vs e970b95; split-tail knobs on cur
mkdir -p gpurun_out
exec > gpurun_out/call46.log 2>&1
for R in 1 2; do
for h in e970b95 cur om; do
  for C in c3n8 c4 c4n8 c3; do
    (cd ab/$h && PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/$h /")
  done
done
done
cd ab/cur
for C in c3 c5 c2 c3n8; do
  for T in "148 2" "148 4" "296 2" "296 4"; do
    set -- $T
    LAM_TAIL_UNITS=$1 LAM_TAIL_SPLITS=$2 PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/tail $1x$2 /"
  done
done
PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c3n8 --splits 4096,2048,1024 --iters 30 2>&1 | grep -v Warn | sed "s/^/uniform /"
PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg c4 --splits 32768,16384,8192,4096 --iters 30 2>&1 | grep -v Warn | sed "s/^/uniform /"
