#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
for WL in c2 c3; do
  timeout 900 python bench.py --workload $WL --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$WL.log 2>&1
  timeout 900 python bench.py --workload $WL --steps 10 --warmup 3 --no-cpu-baseline --separate-append --no-e2e > gpurun_out/bench_${WL}_sep.log 2>&1
done
