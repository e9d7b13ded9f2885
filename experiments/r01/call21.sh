#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
exec > gpurun_out/sweep13.log 2>&1
for C in c2 c3 c3n8 c4 c4n8 c1; do
  timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 | sed "s/^/auto /"
done
timeout 300 python scripts/exp_decode.py --cfg c3 --splits 2048,1024 | sed "s/^/force /"
timeout 300 python scripts/exp_decode.py --cfg c3n8 --splits 4096,1024 | sed "s/^/force /"
timeout 300 python scripts/exp_decode.py --cfg c4 --splits 32768,4096 | sed "s/^/force /"
LAM_DECODE_CTAS=131 timeout 300 python scripts/exp_decode.py --cfg c4 --splits 32768 | sed "s/^/ctas131 /"
