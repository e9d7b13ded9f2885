PYTEST_ARGS="-k slow" PYTEST_TIMEOUT=900 BENCH_ARGS="--steps 10 --warmup 3" ./scripts/gpu_check.sh
timeout 900 python bench.py --workload c3 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
timeout 600 python bench.py --workload c1 --steps 20 --warmup 5 > gpurun_out/bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c1.log
PROF_TAG=c2 PROF_KERNEL=decode_simt PROF_SKIP=32 BENCH_ARGS="--steps 2 --warmup 1" ./scripts/gpu_prof.sh
