#!/bin/bash
# same-box A/B of decode kernels: older builds vs HEAD (the re-entry bench was lower than r01)
mkdir -p gpurun_out
exec > gpurun_out/call43.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for R in 1; do
for h in 6dc8b57 8793e33 e970b95 HEAD; do
  for C in c2 c3 c4 c5 c1; do
    (cd ab/$h && PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/$h /")
  done
done
done
