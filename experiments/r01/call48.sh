#!/bin/bash
# after the register-cap fix + planner refit: GPU tests, smoke, bench lines, ncu of C3 and C2
mkdir -p gpurun_out
exec > gpurun_out/call48.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for W in c2 c3 c4 c5 c1; do
  timeout 600 python bench.py --workload $W > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err; echo "bench $W rc=$?"
done
PROF_TAG=r02_c3 PROF_KERNEL=decode_gqa BENCH_ARGS="--workload c3 --steps 2 --warmup 3" bash scripts/gpu_prof.sh
PROF_TAG=r02_c2 PROF_KERNEL=decode_simt BENCH_ARGS="--workload c2 --steps 2 --warmup 3" bash scripts/gpu_prof.sh
ls -la gpurun_out/
