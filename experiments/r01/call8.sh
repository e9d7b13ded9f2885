#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/sweep6.log 2>&1
for R in 1 2; do
for F in 0 2; do
  for C in c3 c3n8 c4 c2; do
  LAM_DECODE_FLAGS=$F LAM_ITEMS_PER_CTA=1 timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 | sed "s/^/f$F /"
  done
  LAM_DECODE_FLAGS=$F LAM_ITEMS_PER_CTA=8 timeout 300 python scripts/exp_decode.py --cfg c4 --splits 0 | sed "s/^/f$F i8 /"
done
done
echo done
