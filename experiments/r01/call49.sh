#!/bin/bash
# MHA (G=1) on the tensor-core kernel vs the SIMT kernel, same box: kernel-only and bench (clocks)
mkdir -p gpurun_out
exec > gpurun_out/call49.log 2>&1
for R in 1 2; do
  PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/simt /"
  LAM_MHA_MMA=1 PYTHONPATH=$PWD timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 --iters 30 2>&1 | grep -v Warn | sed "s/^/mma /"
done
timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | sed "s/^/simt /"
LAM_MHA_MMA=1 timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | sed "s/^/mma /"
timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | sed "s/^/simt /"
LAM_MHA_MMA=1 timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | sed "s/^/mma /"
