#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
exec > gpurun_out/sweep12.log 2>&1
for R in 1 2; do
for F in 0 4; do
  for C in c2 c3 c3n8 c4 c1; do
    LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 | sed "s/^/f$F /"
  done
  LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c3 --splits 2048,1024 | sed "s/^/f$F /"
done
done
