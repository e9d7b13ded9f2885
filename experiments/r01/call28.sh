#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
exec > gpurun_out/sweep19.log 2>&1
for F in 0 4; do
  LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c5 --splits 0 | sed "s/^/f$F /"
  LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c3 --splits 0 | sed "s/^/f$F /"
  LAM_DECODE_FLAGS=$F timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 | sed "s/^/f$F /"
done
