#!/bin/bash
# ncu evidence for the final committed kernels (after the tensor-map L2-promotion change):
# launch list + one --set full capture of the decode kernel for C2 (default line) and C3.
mkdir -p gpurun_out
PROF_TAG=r01c_c2 PROF_KERNEL=decode_gqa BENCH_ARGS="--workload c2 --steps 2 --warmup 3" bash scripts/gpu_prof.sh
PROF_TAG=r01c_c3 PROF_KERNEL=decode_gqa BENCH_ARGS="--workload c3 --steps 2 --warmup 3" bash scripts/gpu_prof.sh
for T in r01c_c2 r01c_c3; do
  [ -f gpurun_out/prof_$T.ncu-rep ] && ncu -i gpurun_out/prof_$T.ncu-rep --page raw --csv > gpurun_out/ncu_${T}_raw.csv 2>/dev/null
  [ -f gpurun_out/prof_$T.ncu-rep ] && ncu -i gpurun_out/prof_$T.ncu-rep --page details --csv > gpurun_out/ncu_${T}_details.csv 2>/dev/null
done
ls -la gpurun_out
