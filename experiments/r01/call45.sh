#!/bin/bash
# launch_bounds(...,1) (no register cap) and two S-accumulation chains vs e970b95, same box
mkdir -p gpurun_out
exec > gpurun_out/call45.log 2>&1
timeout 600 python -m pytest tests/test_decode_gpu.py -x -q 2>&1 | tail -2
for R in 1 2; do
for h in e970b95 lb new; do
  for C in c2 c3 c4 c5 c1 c3n8; do
    (cd ab/$h && PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/$h /")
  done
done
done
