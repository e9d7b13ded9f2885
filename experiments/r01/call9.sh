#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for WL in c2 c3 c4 c1; do
  timeout 900 python bench.py --workload $WL --steps 10 --warmup 3 $([ $WL != c2 ] && echo --no-cpu-baseline) > gpurun_out/bench_$WL.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$WL.log
done
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
