#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
exec > gpurun_out/sweep7.log 2>&1
for C in c2 c3 c3n8 c4 c4n8 c1; do
  timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 | sed "s/^/auto /"
done
for C in c3 c3n8; do timeout 300 python scripts/exp_decode.py --cfg $C --splits 2048,1024,512 ; done
timeout 300 python scripts/exp_decode.py --cfg c4 --splits 16384,8192,4096,2048
timeout 300 python scripts/exp_decode.py --cfg c2 --splits 2048,1024
timeout 300 python scripts/exp_decode.py --cfg c1 --splits 512,256 --iters 50
echo done
