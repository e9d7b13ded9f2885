#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
exec > gpurun_out/sweep2.log 2>&1
for V in 0 1 3; do for I in 1 2 4 8; do
  LAM_GQA_VARIANT=$V LAM_ITEMS_PER_CTA=$I timeout 300 python scripts/exp_decode.py --cfg c3 --splits 0 | sed "s/^/v$V i$I /"
done; done
for V in 0 1 2 3; do for I in 1 2 4 8; do
  LAM_SIMT_VARIANT=$V LAM_ITEMS_PER_CTA=$I timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 | sed "s/^/v$V i$I /"
done; done
for I in 1 2 4 8; do
  LAM_ITEMS_PER_CTA=$I timeout 300 python scripts/exp_decode.py --cfg c3n8 --splits 0 | sed "s/^/v0 i$I /"
  LAM_ITEMS_PER_CTA=$I timeout 300 python scripts/exp_decode.py --cfg c4 --splits 0 | sed "s/^/v0 i$I /"
done
for V in 0 1 2 3; do for I in 1 2 4 8; do
  LAM_SIMT_VARIANT=$V LAM_ITEMS_PER_CTA=$I timeout 300 python scripts/exp_decode.py --cfg c1 --splits 0 --iters 50 | sed "s/^/v$V i$I /"
done; done
echo done
