#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 ./benchmarks/bench_attention_b200 > gpurun_out/cpp_bench.log 2>&1
for WL in c2 c3 c4 c5 c1; do
  timeout 900 python bench.py --workload $WL --steps 10 --warmup 3 $([ $WL != c2 ] && [ $WL != c1 ] && echo --no-cpu-baseline) > gpurun_out/bench_$WL.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$WL.log
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.log 2>&1
PROF_TAG=c2g PROF_KERNEL=decode_simt PROF_SKIP=32 PROF_COUNT=200 BENCH_ARGS="--steps 1 --warmup 1" ./scripts/gpu_prof.sh
PROF_TAG=c3g PROF_KERNEL=decode_gqa PROF_SKIP=80 PROF_COUNT=400 BENCH_ARGS="--workload c3 --steps 1 --warmup 1" ./scripts/gpu_prof.sh
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
