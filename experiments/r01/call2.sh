#!/bin/bash
mkdir -p gpurun_out
PROF_TAG=c3 PROF_KERNEL=decode_gqa PROF_SKIP=160 PROF_COUNT=400 BENCH_ARGS="--workload c3 --steps 1 --warmup 2" ./scripts/gpu_prof.sh
PROF_TAG=c1 PROF_KERNEL=decode_simt PROF_SKIP=10 PROF_COUNT=100 BENCH_ARGS="--workload c1 --steps 10 --warmup 5" ./scripts/gpu_prof.sh
