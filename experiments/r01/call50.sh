#!/bin/bash
# MHA on the tensor-core kernel by default: GPU tests, smoke, default bench x2, ncu of C2
mkdir -p gpurun_out
exec > gpurun_out/call50.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_c2_a.json 2>/dev/null; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>/dev/null; echo "ref rc=$?"
PROF_TAG=r01b_c2mma PROF_KERNEL=decode_gqa BENCH_ARGS="--workload c2 --steps 2 --warmup 3" bash scripts/gpu_prof.sh
timeout 600 python bench.py > gpurun_out/bench_c2_b.json 2>/dev/null; echo "bench rc=$?"
