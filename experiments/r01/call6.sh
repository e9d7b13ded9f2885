#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
exec > gpurun_out/sweep4.log 2>&1
for PR in 3 0 2; do for I in 1 2 4 8; do
  LAM_TMAP_PROMOTION=$PR LAM_ITEMS_PER_CTA=$I timeout 300 python scripts/exp_decode.py --cfg c3 --splits 0 | sed "s/^/pr$PR i$I /"
done; done
for I in 1 2 4 8 16; do
  LAM_ITEMS_PER_CTA=$I timeout 300 python scripts/exp_decode.py --cfg c3n8 --splits 0 | sed "s/^/i$I /"
  LAM_ITEMS_PER_CTA=$I timeout 300 python scripts/exp_decode.py --cfg c4 --splits 0 | sed "s/^/i$I /"
  LAM_ITEMS_PER_CTA=$I timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 | sed "s/^/i$I /"
  LAM_ITEMS_PER_CTA=$I timeout 300 python scripts/exp_decode.py --cfg c1 --splits 0 --iters 50 | sed "s/^/i$I /"
done
for V in 4; do LAM_SIMT_VARIANT=$V timeout 300 python scripts/exp_decode.py --cfg c2 --splits 0 | sed "s/^/v$V /"; done
echo done
