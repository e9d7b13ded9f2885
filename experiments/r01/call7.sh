#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
exec > gpurun_out/sweep5.log 2>&1
for I in 1 2 4 8; do
  for C in c3 c3n8 c4 c2 c1; do
  LAM_ITEMS_PER_CTA=$I timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 | sed "s/^/i$I /"
  done
done


echo done
