#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/sweep10.log 2>&1
for C in c1 c2 c3 c3n8 c4 c4n8; do
  timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 | sed "s/^/auto /"
done
LAM_DECODE_CTAS=128 timeout 300 python scripts/exp_decode.py --cfg c3 --splits 0 | sed "s/^/ctas128 /"
LAM_DECODE_CTAS=128 timeout 300 python scripts/exp_decode.py --cfg c4 --splits 8192 | sed "s/^/ctas128 /"
LAM_DECODE_CTAS=128 timeout 300 python scripts/exp_decode.py --cfg c4n8 --splits 0,16384,8192 | sed "s/^/ctas128 /"
LAM_DECODE_CTAS=148 timeout 300 python scripts/exp_decode.py --cfg c4n8 --splits 4096 | sed "s/^/ctas148 /"
LAM_DECODE_CTAS=148 timeout 300 python scripts/exp_decode.py --cfg c1 --splits 0 --iters 50 | sed "s/^/ctas148 /"
echo done
