#!/bin/bash
# batched split merge: split tail + uniform splits, sustained
mkdir -p gpurun_out
exec > gpurun_out/call41.log 2>&1
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_peer_gpu.py -x -q 2>&1 | tail -3
for C in c2 c3 c3n8 c1; do
  for T in "0 4" "148 2" "148 4" "296 4"; do
    set -- $T
    LAM_TAIL_UNITS=$1 LAM_TAIL_SPLITS=$2 PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 --iters 200 --warm 50 2>&1 | grep -v Warn | sed "s/^/tail $1 x$2 /"
  done
done
PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c3n8 --splits 4096,2048,1024 --iters 200 --warm 50 2>&1 | grep -v Warn | sed "s/^/uniform /"
PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c4 --splits 32768,16384,8192,4096 --iters 100 --warm 20 2>&1 | grep -v Warn | sed "s/^/uniform /"
PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c5 --splits 0 --iters 100 --warm 20 2>&1 | grep -v Warn | sed "s/^/auto /"
LAM_TAIL_UNITS=148 LAM_TAIL_SPLITS=4 PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c5 --splits 0 --iters 100 --warm 20 2>&1 | grep -v Warn | sed "s/^/tail148x4 /"
