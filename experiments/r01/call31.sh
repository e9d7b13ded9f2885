#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/bisect.log 2>&1
for R in 1 2; do
for h in 6dc8b57 1b03a2e bb680eb 7bd42db b762168; do
  for C in c2 c3 c3n8; do
    (cd ab/$h && PYTHONPATH=$PWD timeout 300 python exp_decode.py --cfg $C --splits 0 2>&1 | grep -v Warn | sed "s/^/$h /")
  done
done
done
