#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/sweep11.log 2>&1
for V in 0 5 6 2; do for C in c3 c3n8 c4; do
  LAM_GQA_VARIANT=$V timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 --P 128 | sed "s/^/v$V /"
done; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.log 2>&1
echo done
