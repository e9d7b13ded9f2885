#!/bin/bash
# same-box bisect of the S=1 regression: e970b95, 37c31e1, HEAD without the flags check, HEAD
mkdir -p gpurun_out
exec > gpurun_out/call44.log 2>&1
for R in 1 2; do
for h in e970b95 37c31e1 noflag HEAD; do
  for C in c2 c3 c4; do
    (cd ab/$h && PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/$h /")
  done
done
done
