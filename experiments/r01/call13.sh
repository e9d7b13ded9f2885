#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/sweep9.log 2>&1
for N in 148 128 132 136 140 144 120 112; do
  LAM_DECODE_CTAS=$N timeout 300 python scripts/exp_decode.py --cfg c3n8 --splits 0 | sed "s/^/ctas$N /"
  LAM_DECODE_CTAS=$N timeout 300 python scripts/exp_decode.py --cfg c3 --splits 0 | sed "s/^/ctas$N /"
  LAM_DECODE_CTAS=$N timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 | sed "s/^/ctas$N /"
done
LAM_DECODE_CTAS=128 timeout 300 python scripts/exp_decode.py --cfg c4 --splits 8192,4096 | sed "s/^/ctas128 /"
echo done
