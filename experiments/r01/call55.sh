#!/bin/bash
# current build: GPU tests, smoke, every bench line, reference arm, ncu of the default (C2) and C3
mkdir -p gpurun_out
exec > gpurun_out/call55.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for W in c2 c3 c4 c5 c1; do
  timeout 600 python bench.py --workload $W > gpurun_out/b55_$W.json 2>/dev/null; echo "bench $W rc=$?"
done
timeout 600 python bench.py --impl reference > gpurun_out/b55_ref.json 2>/dev/null; echo "ref rc=$?"
PROF_TAG=r01b_c2f PROF_KERNEL=decode_gqa BENCH_ARGS="--workload c2 --steps 2 --warmup 3" bash scripts/gpu_prof.sh
PROF_TAG=r01b_c3f PROF_KERNEL=decode_gqa BENCH_ARGS="--workload c3 --steps 2 --warmup 3" bash scripts/gpu_prof.sh
timeout 600 python bench.py > gpurun_out/b55_c2_again.json 2>/dev/null; echo "bench c2 again rc=$?"
